timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; tail -2 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 250 gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
timeout 900 python bench.py --workload qsweep --steps 2 --warmup 1 > gpurun_out/qsweep_final.json 2> gpurun_out/qsweep.err; tail -c 200 gpurun_out/qsweep_final.json
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > gpurun_out/bench_cfg1_final.json 2> gpurun_out/cfg1.err; tail -c 200 gpurun_out/bench_cfg1_final.json
