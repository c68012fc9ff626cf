# residency / DFA-copy sweep for configs 3 and 4 (diagnostic)
mkdir -p gpurun_out
B="python bench.py --steps 100 --no-cpu --e2e-steps 1"
for c in 4; do
  echo "cfg$c auto:"; $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['config']['residency'])"
  echo "cfg$c hot:";  $B --config $c --residency 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['config']['residency'])"
done
for r in 16 8; do
  echo "cfg3 dfa copies $r:"; SFA_DFA_COPIES=$r $B --config 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['config']['residency'])"
done
for h in 512 2048; do
  echo "cfg3 hot rows $h:"; SFA_HOT_ROWS=$h $B --config 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['config']['residency'])"
done
