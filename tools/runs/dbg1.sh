timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2; echo smoke rc=$?
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "factor_parity_small and greedy" 2>&1 | tail -3
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "production_tiles" 2>&1 | tail -3
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/strip_bench tools/strip_bench.cu -lcuda && timeout 60 ./tools/strip_bench; echo sb rc=$?
