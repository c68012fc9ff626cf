# Round-2 measurement session (re-run per milestone): default bench line, reference arm, ncu launch
# list of a short bench command, ncu --set full of one k_scan_tma launch per
# config, and the phase stamps.  usage: bash scripts/gpu_round2.sh <tag> ["2 3 5"]
tag=${1:-r2b}; cfgs=${2:-"2 3 4 5"}
mkdir -p gpurun_out /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout -s KILL 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu --no-nsfa --no-lazy --single-reps 3"
timeout -s KILL 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launch list rc=$?"
for c in $cfgs; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tma -s 3 -c 1 \
     -o /tmp/ncu/${tag}_cfg$c python scripts/one_launch.py $c > gpurun_out/${tag}_ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_raw_cfg$c.csv 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page details > gpurun_out/${tag}_ncu_details_cfg$c.txt 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page source --csv > gpurun_out/${tag}_ncu_source_cfg$c.csv 2>/dev/null
done
timeout -s KILL 900 python scripts/stamps.py 2,3,4,5 > gpurun_out/${tag}_stamps.txt 2>&1; echo "stamps rc=$?"
