mkdir -p gpurun_out
for wv in 0 1 2; do PCS_SORT_WIDE=$wv python tools/sort_sweep.py 1x2048 16x2048 64x2048 148x2048 16x1024 16x4096 64x4096 > gpurun_out/sortwide_$wv.log 2>&1; done
echo done
