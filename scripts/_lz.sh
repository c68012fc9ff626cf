bash scripts/gpu_tests.sh lz tests/test_lazy.py
timeout 600 python scripts/lazy_probe.py > gpurun_out/lazy_probe.txt 2>&1; echo probe rc=$?
cat gpurun_out/lazy_probe.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lazy_launches.csv \
  python scripts/lazy_probe.py 1024 1 > gpurun_out/lazy_ncu.log 2>&1; echo ncu rc=$?
