mkdir -p gpurun_out
python tools/cluster_ab.py > gpurun_out/cluster_ab.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/cluster_gpu.log 2>&1
echo done
