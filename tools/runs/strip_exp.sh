for e in 0 512; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -DTQR_EXP=$e -o tools/strip_bench_e$e tools/strip_bench.cu -lcuda &
done; wait
for e in 0 512; do echo "== EXP $e"; ./tools/strip_bench_e$e | grep "tma=1 ctas=148"; done
