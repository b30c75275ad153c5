# session 4: TS-family tall path tests, bench, ncu traffic of configs[3] greedy TS
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tall or distributed_apply" > gpurun_out/s4c_tests.log 2>&1; echo rc=$? >> gpurun_out/s4c_tests.log
python bench.py > gpurun_out/s4c_bench.json 2> gpurun_out/s4c_bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tqr_persistent -c 2 --csv python tools/ncu_one.py 2048 16 256 greedy:1:TS > gpurun_out/s4c_ncu_tall_ts.csv 2>&1
