mkdir -p gpurun_out
tag=${1:-sort}
python tools/sort_sweep.py > gpurun_out/${tag}_sweep.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sort" > gpurun_out/${tag}_tests.log 2>&1
echo done
