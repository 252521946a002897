mkdir -p gpurun_out
python tools/sort_sweep.py 64x8192 40x8192 72x8192 64x16384 48x16384 48x32768 > gpurun_out/pair_off.log 2>&1
PCS_SORT_PAIR=1 python tools/sort_sweep.py 64x8192 40x8192 72x8192 64x16384 48x16384 48x32768 > gpurun_out/pair_on.log 2>&1
echo done
