T=greedy,fibonacci,flat,plasma:5,plasma:10
for cfg in "TQR_CHAIN_SPIN=0" "TQR_CHAIN_SPIN=8" "TQR_CHAIN_SPIN=32" "TQR_CHAIN_SPIN=64" "TQR_CHAIN_SPIN=256"; do
  echo "== $cfg"; env $cfg python tools/quick_time.py 40 10 200 32 $T 2>&1 | sed "s/ (all.*//"
done
