# GPU session: selected parity tests, then a shape sweep.  usage: bash scripts/gpu_quick.sh <tag> <SWEEP> <cfgs> [pytest -k expr]
tag=${1:-q}; sw=${2:-base}; cfgs=${3:-5,3,4,2}; kx=${4:-"rows or factored or batch or residency or cfg3 or cfg5"}
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -m gpu -q -p no:cacheprovider --timeout=300 -x tests/test_gpu_seg.py tests/test_gpu.py -k "$kx" \
  > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$tag.log
SWEEP=$sw timeout -s KILL 900 python scripts/shape_sweep.py $cfgs > gpurun_out/sweep_$tag.jsonl 2> gpurun_out/sweep_$tag.err; echo "sweep rc=$?"
cat gpurun_out/sweep_$tag.jsonl; tail -2 gpurun_out/sweep_$tag.err
