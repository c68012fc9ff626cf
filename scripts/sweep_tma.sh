# usage: bash scripts/sweep_tma.sh <tag> "<configs>" "<shapes>"
# Times bench.py per forced TMA shape (SFA_TMA_CONFIG="K,ROWB,ring,pf,promo"),
# then one ncu metrics pass per shape (DRAM bytes and duration of k_scan_tma).
tag=$1
mkdir -p gpurun_out
out=gpurun_out/sweep_$tag.log
for c in ${2:-2 4}; do
for shape in ${3:-""}; do
  SFA_TMA_CONFIG=$shape timeout 120 python bench.py --config $c --steps 300 --warmup 5 --no-cpu --e2e-steps 1 > /tmp/sw.json 2>/tmp/sw.err
  rc=$?
  python - "$c" "$shape" "$rc" >> $out <<'PY'
import json,sys
c,shape,rc=sys.argv[1:]
try:
    d=json.loads(open('/tmp/sw.json').read().strip().splitlines()[-1])
    print(f"cfg{c} shape={shape} {d['value']:.1f} GB/s sm={d['clocks']['sm_mhz']} res={d['config']['residency']}", flush=True)
except Exception as e:
    print(f"cfg{c} shape={shape} rc={rc} FAILED", open('/tmp/sw.err').read()[-300:])
PY
done; done
for c in ${2:-2 4}; do
for shape in ${3:-""}; do
  SFA_TMA_CONFIG=$shape timeout 200 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:k_scan_tma -s 3 -c 1 --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>/dev/null \
    | grep -E '"(dram__bytes_read.sum|gpu__time_duration.sum|l1tex__data_bank|smsp__inst_executed.sum)"' \
    | awk -F'","' -v s="cfg$c shape=$shape" '{printf "%s %s %s %s\n", s, $(NF-2), $(NF-1), $NF}' >> $out
done; done
echo done >> $out
