mkdir -p gpurun_out
(./tools/microbench/cluster_prof 2048 512; ./tools/microbench/cluster_prof 8192 2048) > gpurun_out/cprof.log 2>&1
echo done
