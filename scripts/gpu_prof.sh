# GPU session: stamps (diag library) and ncu captures of the scan kernel.
# usage: bash scripts/gpu_prof.sh <tag> <configs for ncu, e.g. "2 5">
tag=${1:-p}; cfgs=${2:-"2 5"}
mkdir -p gpurun_out /tmp/ncu
timeout -s KILL 900 python scripts/stamps.py 2,3,4,5 > gpurun_out/stamps_$tag.txt 2>&1; echo "stamps rc=$?"
for c in $cfgs; do
  timeout -s KILL 600 python scripts/one_launch.py $c > gpurun_out/plain_$tag_$c.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tma -s 3 -c 1 \
     -o /tmp/ncu/${tag}_cfg$c python scripts/one_launch.py $c > gpurun_out/ncu_${tag}_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${tag}_cfg$c.csv 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page details > gpurun_out/ncu_details_${tag}_cfg$c.txt 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page source --csv > gpurun_out/ncu_source_${tag}_cfg$c.csv 2>/dev/null
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}_cfg5.csv python scripts/one_launch.py 5 5 > gpurun_out/ncu_launch_$tag.log 2>&1; echo "launch list rc=$?"
