mkdir -p gpurun_out
for wl in cfg4 cfg3 cfg5-afps256-32768; do echo $wl; python tools/e2e_parts.py $wl; done > gpurun_out/e2e_parts.log 2>&1
echo done
