# One GPU session: gpu tests, smoke, bench (default + --all), ncu launch list
# and one full capture of the top kernel per config.
# usage: bash scripts/gpu_round.sh <tag> [configs for ncu]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
timeout 900 python bench.py --all --steps 300 --no-cpu > gpurun_out/bench_all_$tag.json 2> gpurun_out/bench_all_$tag.err; echo "bench-all rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo "bench-ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu"
$CMD > gpurun_out/plain_launch_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD \
  > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu-launch rc=$?"
for c in ${2:-2}; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu"
  $CMD > gpurun_out/plain_full_${tag}_cfg$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 3 -c 1 -o gpurun_out/full_${tag}_cfg$c $CMD \
    > gpurun_out/ncu_full_${tag}_cfg$c.log 2>&1; echo "ncu-full cfg$c rc=$?"
done
