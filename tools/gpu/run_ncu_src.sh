# one ncu --set full capture with source-level stall sampling of the sampler
# kernel of one workload (third launch) -> gpurun_out/<tag>.ncu-rep
# usage: tools/gpu/run_ncu_src.sh TAG WORKLOAD [kernel-regex]
mkdir -p gpurun_out
tag=$1; w=$2; rx=${3:-"regex:fps_full|fps_cluster|npdu_|morton_|rows_kernel|stream_sector"}
timeout 900 ncu --set full --import-source on --clock-control none -k "$rx" -s 2 -c 1 \
  -o gpurun_out/$tag -f python bench.py --workload $w --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-workloads > gpurun_out/$tag.log 2>&1
tail -2 gpurun_out/$tag.log
