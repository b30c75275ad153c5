C="greedy:1:TT,flat:1:TS"
for m in 2 3 4; do
  echo "== TQR_MSTRIP=$m"
  TQR_MSTRIP=$m timeout 300 python tools/quick_time.py 40 40 200 32 $C | cut -c1-70
done
TQR_MSTRIP=2 timeout 300 python tools/quick_time.py 40 10 200 32 greedy:1:TT,flat:1:TS | cut -c1-70
TQR_MSTRIP=3 timeout 300 python tools/quick_time.py 40 10 200 32 greedy:1:TT,flat:1:TS | cut -c1-70
