# One GPU session: gpu tests, smoke, bench (default + --all --spec), ncu launch
# list and one full capture of the top kernel per config.  The .ncu-rep files
# stay on the box (/tmp/ncu); their raw and details pages come back as text
# (gpurun returns at most 64 MiB of gpurun_out/).
# usage: bash scripts/gpu_round.sh <tag> [configs for ncu]
tag=${1:-r1}
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
timeout 900 python bench.py --all --spec --steps 300 --no-cpu > gpurun_out/bench_all_$tag.json 2> gpurun_out/bench_all_$tag.err; echo "bench-all rc=$?"
timeout 900 python bench.py --config 5 --steps 20 --no-cpu > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err; echo "bench-c5 rc=$?"
timeout 900 python bench.py --rn --steps 100 --no-cpu --e2e-steps 1 > gpurun_out/bench_rn_$tag.json 2> gpurun_out/bench_rn_$tag.err; echo "bench-rn rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo "bench-ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu"
$CMD > gpurun_out/plain_launch_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD \
  > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu-launch rc=$?"
for c in ${2:-2}; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu"
  $CMD > gpurun_out/plain_full_${tag}_cfg$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 3 -c 1 -o /tmp/ncu/full_${tag}_cfg$c $CMD \
    > gpurun_out/ncu_full_${tag}_cfg$c.log 2>&1; echo "ncu-full cfg$c rc=$?"
  ncu -i /tmp/ncu/full_${tag}_cfg$c.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${tag}_cfg$c.csv 2>/dev/null
  ncu -i /tmp/ncu/full_${tag}_cfg$c.ncu-rep --page details > gpurun_out/ncu_details_${tag}_cfg$c.txt 2>/dev/null
done
