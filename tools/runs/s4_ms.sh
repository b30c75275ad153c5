# session 4: strips per update task (TQR_MSTRIP) over the six configs[2] bench cases
C="greedy:1:TT,fibonacci:1:TT,flat:1:TT,greedy:1:TS,fibonacci:1:TS,flat:1:TS"
for m in 2 3 4 5; do
  echo "== TQR_MSTRIP=$m"
  TQR_MSTRIP=$m timeout 300 python tools/quick_time.py 40 40 200 32 $C
done
