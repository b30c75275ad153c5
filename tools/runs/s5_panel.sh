# session 5: 8-lane-group panel layout — parity first, then panel_bench and the bench cases
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -5
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DTQR_PROF=1 -o /tmp/panel_bench tools/panel_bench.cu && timeout 60 /tmp/panel_bench
C="greedy:1:TT,fibonacci:1:TT,flat:1:TT,greedy:1:TS,fibonacci:1:TS,flat:1:TS"
timeout 300 python tools/quick_time.py 40 40 200 32 $C
timeout 300 python tools/quick_time.py 40 10 200 32 greedy:1:TT,flat:1:TS,plasma:10:TS
timeout 300 python tools/quick_time.py 2048 16 256 32 greedy:1:TS,flat:1:TS
