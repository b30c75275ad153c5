# A/B of the UNMQR+TTMQR fusion (TQR_FUSE) on configs[2] and configs[1] TT trees
for f in 0 1 0 1; do
  echo "== TQR_FUSE=$f"
  TQR_FUSE=$f timeout 300 python tools/quick_time.py 40 40 200 32 greedy,fibonacci,flat
  TQR_FUSE=$f timeout 300 python tools/quick_time.py 40 10 200 32 greedy,flat,plasma:10
done
