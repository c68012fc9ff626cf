tag=${1:-st}; cfgs=${2:-2,3,4,5}
mkdir -p gpurun_out
timeout -s KILL 900 python scripts/stamps.py $cfgs > gpurun_out/stamps_$tag.txt 2>&1; echo "stamps rc=$?"
cat gpurun_out/stamps_$tag.txt | grep -v "^\s*$" | tail -80
