T=greedy,fibonacci,flat,plasma:5,plasma:10
for cfg in "TQR_WS=32" "TQR_WS=64" "TQR_WS=16" "TQR_SPLIT=0"; do
  echo "== $cfg"; env $cfg python tools/quick_time.py 40 10 200 32 $T 2>&1 | sed "s/ (all.*//"
done
