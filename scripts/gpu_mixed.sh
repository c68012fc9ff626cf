# GPU session: FACTORED DFA-window layouts -- parity (factored rows tests, cfg3/cfg5 full size), then the sweep.
tag=${1:-m}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest -m gpu -q -p no:cacheprovider --timeout=300 -x \
  tests/test_gpu_seg.py -k "rows_hot_factored or rows_private" tests/test_gpu.py -k "cfg3 or cfg5 or factored or residency" \
  > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$tag.log
SWEEP=mixed timeout -s KILL 900 python scripts/shape_sweep.py 5,3 > gpurun_out/sweep_$tag.jsonl 2> gpurun_out/sweep_$tag.err; echo "sweep rc=$?"
cat gpurun_out/sweep_$tag.jsonl
