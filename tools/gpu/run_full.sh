# full GPU suite + default bench (headline + workloads) -> gpurun_out/<tag>_*
mkdir -p gpurun_out
tag=${1:-full}
timeout 1200 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/${tag}_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo done
