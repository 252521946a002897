# sort parity tests + sweep: tools/gpu/run_sort.sh TAG [shapes...]
mkdir -p gpurun_out
tag=$1; shift
timeout 900 python -m pytest tests -q -m gpu -x -k "sort" > gpurun_out/${tag}_gpu.log 2>&1
tail -3 gpurun_out/${tag}_gpu.log
for v in 0 1; do
  echo "PCS_SORT_BUCKET=$v" >> gpurun_out/${tag}_sweep.log
  PCS_SORT_BUCKET=$v timeout 600 python tools/sort_sweep.py "$@" >> gpurun_out/${tag}_sweep.log 2>&1
done
cat gpurun_out/${tag}_sweep.log
