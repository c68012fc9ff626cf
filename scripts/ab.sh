# A/B of two builds on one box: libsfa_old.so against libsfa.so, alternating.  usage: bash scripts/ab.sh [rounds]
for r in $(seq 1 ${1:-2}); do
  for which in old new; do
    lib=paper_1405_0562_b200/_lib/libsfa.so; [ $which = old ] && lib=paper_1405_0562_b200/_lib/libsfa_old.so
    SFA_LIB=$PWD/$lib timeout -s KILL 600 python bench.py --steps 40 --no-cpu --no-nsfa --no-lazy --e2e-steps 0 --single-reps 5 \
      > gpurun_out/ab_${which}_$r.json 2> gpurun_out/ab_${which}_$r.err
    echo "== $which $r"; python scripts/q.py gpurun_out/ab_${which}_$r.json | tr '\n' ' '; echo
  done
done
