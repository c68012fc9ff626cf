# ncu --set full of one k_scan_tma launch per config; raw + details pages back in gpurun_out.
# usage: bash scripts/gpu_ncu2.sh <tag> "5 4"
tag=${1:-n}; cfgs=${2:-"5 4"}
mkdir -p gpurun_out /tmp/ncu
for c in $cfgs; do
  timeout -s KILL 600 python scripts/one_launch.py $c > gpurun_out/${tag}_plain_cfg$c.log 2>&1; echo "plain cfg$c rc=$?"
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tma -s 3 -c 1 \
     -o /tmp/ncu/${tag}_cfg$c python scripts/one_launch.py $c > gpurun_out/${tag}_ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_raw_cfg$c.csv 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page details > gpurun_out/${tag}_ncu_details_cfg$c.txt 2>/dev/null
  ncu -i /tmp/ncu/${tag}_cfg$c.ncu-rep --page source --csv > gpurun_out/${tag}_ncu_source_cfg$c.csv 2>/dev/null
done
