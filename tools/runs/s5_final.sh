# session 5: final-state verification (fresh build in a re-created container)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo rc=$?; tail -c 3000 gpurun_out/s5_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5_bench_ref.json 2> gpurun_out/s5_bench_ref.err; echo rc=$?; cat gpurun_out/s5_bench_ref.json
