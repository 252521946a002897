mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export PCS_BK_SMALL=1; else unset PCS_BK_SMALL; fi
  echo "small=$v" >> gpurun_out/bk3.log
  python tools/sort_sweep.py 256x2048 256x4096 64x2048 64x4096 148x2048 256x8192 256x16384 256x32768 >> gpurun_out/bk3.log 2>&1
done
cat gpurun_out/bk3.log
