T=greedy,fibonacci,flat,plasma:5,plasma:10
python tools/quick_time.py 40 10 200 32 $T 2>&1 | sed "s/ (all.*//"
