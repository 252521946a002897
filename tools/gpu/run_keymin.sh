# r02 s3: TMEM NPDU A/B -- kKeyMin argmax + blocked loop + popc writes (repo) vs
# HEAD (abtest/old); PCS_NPDU_ZT (fp64 z in TMEM) on/off; parity subset first
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "npdu or tmem or cfg4 or cfg3" > gpurun_out/keymin_gpu.log 2>&1
tail -3 gpurun_out/keymin_gpu.log
PCS_NPDU_ZT=1 timeout 900 python -m pytest tests -q -m gpu -x -k "npdu or tmem or cfg4 or cfg3" > gpurun_out/keymin_gpu_zt.log 2>&1
tail -3 gpurun_out/keymin_gpu_zt.log
timeout 1200 python tools/ab_versions.py abtest/old . cfg4 cfg3 cfg5-npdu-16384 > gpurun_out/keymin_ab.log 2>&1
cat gpurun_out/keymin_ab.log
bash tools/gpu/run_envab.sh keymin_zt PCS_NPDU_ZT "0 1" "cfg4 cfg3 cfg5-npdu-16384" > /dev/null 2>&1
cat gpurun_out/keymin_zt.log
