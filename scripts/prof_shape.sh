# usage: bash scripts/prof_shape.sh <config> <tag> <SFA_TMA_CONFIG>   -> gpurun_out/prof_<tag>.ncu-rep
c=$1; tag=$2; export SFA_TMA_CONFIG=$3
mkdir -p gpurun_out
CMD="python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 1 --no-cpu"
$CMD > gpurun_out/plain_$tag.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 3 -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1
echo "prof $tag rc=$?"
