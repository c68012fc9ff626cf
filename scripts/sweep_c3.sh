for h in 3000 512 256; do for tc in "" "1,32,0" "1,32,3" "1,16,4"; do
  echo "hot $h tma '$tc': $(SFA_HOT_ROWS=$h SFA_TMA_CONFIG=$tc python scripts/diag_scan.py 3 1024 100 2>&1 | grep cfg)"
done; done
