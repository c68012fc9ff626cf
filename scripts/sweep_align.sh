mkdir -p gpurun_out
for c in 2 3 4; do for a in 256 64 32; do
  echo "cfg$c align $a: $(SFA_ROW_ALIGN=$a python scripts/diag_scan.py $c 1024 100 2>&1 | grep cfg)"
done; done
SFA_DEBUG_STAMPS=1 python scripts/diag_scan.py 3 1024 2 2>&1 | grep stamps | tail -5
SFA_DEBUG_STAMPS=1 python scripts/diag_scan.py 4 1024 2 2>&1 | grep stamps | tail -5
