T=greedy,fibonacci,flat,plasma:5,plasma:10
for cfg in "TQR_PRIO=0" "TQR_PRIO=1" "TQR_PRIO=2" "TQR_PRIO=3" "TQR_LEVELS=8" "TQR_LEVELS=4" "TQR_LOOKAHEAD=0" "TQR_TMA=1"; do
  echo "== $cfg"; env $cfg python tools/quick_time.py 40 10 200 32 $T 2>&1 | sed "s/ (all.*//"
done
