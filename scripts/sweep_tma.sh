# usage: bash scripts/sweep_tma.sh "<configs>" "<shapes>"   (writes gpurun_out/sweep.log)
mkdir -p gpurun_out
for c in ${1:-2 4}; do
for shape in ${2:-"" 1,32,0 2,32,0 2,16,0 1,16,0}; do
  SFA_TMA_CONFIG=$shape timeout 120 python bench.py --config $c --steps 300 --warmup 5 --no-cpu --e2e-steps 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cfg$c', 'shape=$shape', round(d['value'],1), 'GB/s', d['clocks']['sm_mhz'], d['config']['residency'], 'e2e', round(d['e2e']['value'],1))
    elif 'rror' in l or 'wrong' in l: print('cfg$c shape=$shape', l.strip()[:200])
"
done; done >> gpurun_out/sweep.log 2>&1
