# session 4: phase-2 k-step skip A/B + parity subset + panel kernel ncu (HBM GB/s)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "production or schedule or apply or fused" > gpurun_out/s4b_tests.log 2>&1; echo rc=$? >> gpurun_out/s4b_tests.log
bash tools/runs/ab.sh "head p2skip head p2skip" "40 40 200 32 greedy,flat" > gpurun_out/s4b_ab.txt 2>&1
bash tools/runs/ab.sh "head p2skip" "40 10 200 32 greedy,flat" >> gpurun_out/s4b_ab.txt 2>&1
./tools/panel_bench > gpurun_out/s4b_panel_bench.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_shared_ld.sum --clock-control none --csv ./tools/panel_bench > gpurun_out/s4b_panel_ncu.csv 2>&1
