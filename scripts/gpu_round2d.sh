# Round-2c session: the whole -m gpu suite + smoke, then the measurement set of gpu_round2b.sh.
bash scripts/gpu_tests.sh r2d
bash scripts/gpu_round2b.sh r2d "2 3 4 5"
