set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/strip_bench tools/strip_bench.cu -lcuda > gpurun_out/sb_build.log 2>&1
timeout 120 ./tools/strip_bench > gpurun_out/strip_bench.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/trace_report.py 40 40 200 32 greedy > gpurun_out/trace_cfg2_greedy.txt 2>&1
timeout 300 python tools/trace_report.py 40 40 200 32 greedy:1:TS > gpurun_out/trace_cfg2_greedyTS.txt 2>&1
