mkdir -p gpurun_out
python tools/sort_sweep.py 64x8192 100x8192 64x16384 128x16384 48x32768 128x32768 16x32768 > gpurun_out/sortcta_def.log 2>&1
PCS_SORT_CTA_MIN=1 python tools/sort_sweep.py 64x8192 100x8192 64x16384 128x16384 48x32768 128x32768 16x32768 > gpurun_out/sortcta_1.log 2>&1
echo done
