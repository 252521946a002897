mkdir -p gpurun_out
for wl in cfg3 cfg5-afps256-8192 cfg5-afps256-32768 cfg4; do python tools/e2e_probe2.py $wl; done > gpurun_out/probe.log 2>&1
echo done
