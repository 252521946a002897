for rep in 1 2; do
for cfg in "0 4" "1 4" "1 8" "1 9"; do
  set -- $cfg
  out=$(PCS_NPDU_F64S=$1 PCS_NPDU_TMEM_G=$2 python bench.py --workload cfg4 --steps 20 --warmup 5 --no-workloads --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
  echo "f64s=$1 G=$2 $(echo $out | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done; done
