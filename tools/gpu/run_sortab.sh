mkdir -p gpurun_out
tag=${1:-sortab}
python tools/sort_sweep.py > gpurun_out/${tag}_ballot.log 2>&1
PCS_SORT_MATCH=1 python tools/sort_sweep.py > gpurun_out/${tag}_match.log 2>&1
echo done
