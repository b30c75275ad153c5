TQR_LIB=tools/variants/H.so TQR_TMA=0 timeout 60 python tools/runs/dbg.py 3 3 96 greedy TT 2>&1 | grep -v "^$" | sort | uniq -c | sort -rn | head -20
