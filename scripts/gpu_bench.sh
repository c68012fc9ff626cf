# GPU session: the default bench line, then (optional) an ncu launch list and a full capture.
# usage: bash scripts/gpu_bench.sh <tag> [bench args...]
tag=${1:-b}; shift
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_$tag.err
