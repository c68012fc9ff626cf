# GPU session: selected pytest files/expressions with per-test and global timeouts, then smoke.
# usage: bash scripts/gpu_tests.sh <tag> [pytest args...]
tag=${1:-t}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout -s KILL 2400 python -m pytest -m gpu -q -p no:cacheprovider --timeout=300 --timeout_method=thread "$@" \
  > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_$tag.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke_$tag.log
