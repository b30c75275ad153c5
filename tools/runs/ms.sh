for m in 1 2 3 4; do echo "== MSTRIP $m"; TQR_MSTRIP=$m timeout 300 python tools/quick_time.py $1; done
