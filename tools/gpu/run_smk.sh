mkdir -p gpurun_out
./tools/ab_bench.sh PCS_NPDU_SMK "cfg4 cfg3 cfg5-npdu-8192 cfg5-npdu-32768" > gpurun_out/smk_ab.log 2>&1
echo done
