# ncu source-level stall capture of the cfg4 TMEM NPDU kernel: the full
# 128-cloud launch (multi-wave) and a 16-cloud one-wave launch
# -> gpurun_out/npdu_src_{128,16}.ncu-rep + per-instruction CSV
mkdir -p gpurun_out
rx="regex:npdu_tmem"
timeout 900 ncu --set full --import-source on --clock-control none -k "$rx" -s 2 -c 1 \
  -o gpurun_out/npdu_src_128 -f python bench.py --workload cfg4 --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-workloads > gpurun_out/npdu_src_128.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "$rx" -s 2 -c 1 \
  -o gpurun_out/npdu_src_16 -f python tools/strong_probe.py 16 > gpurun_out/npdu_src_16.log 2>&1
for t in 128 16; do
  ncu -i gpurun_out/npdu_src_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/npdu_src_$t.sass.csv 2>&1
done
ls -la gpurun_out
