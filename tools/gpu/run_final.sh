# full GPU suite, default bench, the reference arm, and the ncu launch list
# of the default command (per-launch times, cold-cache, serialised)
mkdir -p gpurun_out
tag=${1:-final}
timeout 1200 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/${tag}_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --no-workloads --steps 2 --warmup 3 \
  > gpurun_out/${tag}_ncu.log 2>&1
echo done
