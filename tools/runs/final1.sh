set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_f1.log 2>&1; tail -2 gpurun_out/gputest_f1.log
python tools/quick_time.py 40 40 200 32 greedy,flat 2>&1 | sed 's/(all.*//'
python tools/quick_time.py 40 10 200 32 greedy,flat 2>&1 | sed 's/(all.*//'
timeout 900 python bench.py > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err; tail -c 300 gpurun_out/bench_f1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_f1.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tqr_persistent -c 12 -o gpurun_out/full_square_f1 -f python tools/ncu_one.py > gpurun_out/ncu_full_sq.log 2>&1; echo full rc=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tqr_persistent -c 2 --csv --log-file gpurun_out/tall_dram_f1.csv python tools/ncu_one.py 2048 16 256 greedy:1:TT > gpurun_out/ncu_tall.log 2>&1; echo tall rc=$?
