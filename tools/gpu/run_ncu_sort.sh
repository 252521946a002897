mkdir -p gpurun_out
python tools/sort_once.py 256 16384 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:radix_cta -c 1 -o gpurun_out/sort16k -f python tools/sort_once.py 256 16384 > gpurun_out/ncu_sort16k.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:radix_cta -c 1 -o gpurun_out/sort32k -f python tools/sort_once.py 256 32768 > gpurun_out/ncu_sort32k.log 2>&1
echo done
