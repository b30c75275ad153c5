# session 4: configs[3] one-GPU local factorization by tree and kernel family
timeout 600 python tools/quick_time.py 2048 16 256 32 greedy:1:TT,greedy:1:TS,fibonacci:1:TS,flat:1:TS,plasma:16:TS,plasma:64:TS
