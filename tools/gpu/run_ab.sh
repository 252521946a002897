# A/B of the working tree against abtest/old (an older commit built in place)
# usage: tools/gpu/run_ab.sh TAG "wl1 wl2 ..." [pytest -k expr]
mkdir -p gpurun_out
tag=$1; wls=$2; kexpr=$3
if [ -n "$kexpr" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -k "$kexpr" > gpurun_out/${tag}_gpu.log 2>&1
  tail -3 gpurun_out/${tag}_gpu.log
fi
timeout 1200 python tools/ab_versions.py abtest/old . $wls > gpurun_out/${tag}_ab.log 2>&1
cat gpurun_out/${tag}_ab.log
