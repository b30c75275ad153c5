timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest2.log 2>&1; tail -3 gpurun_out/gputest2.log
timeout 300 python tools/quick_time.py 40 40 200 32 greedy,fibonacci > gpurun_out/qt2.txt 2>&1
TQR_CLAIM_AHEAD=0 timeout 300 python tools/quick_time.py 40 40 200 32 greedy >> gpurun_out/qt2.txt 2>&1
timeout 300 python tools/quick_time.py 40 10 200 32 greedy,flat >> gpurun_out/qt2.txt 2>&1
timeout 300 python tools/trace_report.py 40 40 200 32 greedy > gpurun_out/trace2_cfg2.txt 2>&1
cat gpurun_out/qt2.txt
