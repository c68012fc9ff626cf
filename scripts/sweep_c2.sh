for a in 128 64; do
 for tc in "" "1,64,0"; do
  echo "align $a tma '$tc': $(SFA_ROW_ALIGN=$a SFA_TMA_CONFIG=$tc python scripts/diag_scan.py 2 256,1024 300 2>&1 | grep cfg | tr '\n' ' ')"
 done
done
for c in 3 4; do echo "cfg$c align 128: $(SFA_ROW_ALIGN=128 python scripts/diag_scan.py $c 1024 100 2>&1 | grep cfg)"; done
