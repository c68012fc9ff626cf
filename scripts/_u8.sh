timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_gpu_seg.py -k "u8 or factored or hot" > gpurun_out/u8_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/u8_tests.log
SWEEP=factored timeout 900 python scripts/shape_sweep.py 5,3 > gpurun_out/u8_sweep.txt 2>&1; echo sweep rc=$?
cat gpurun_out/u8_sweep.txt
