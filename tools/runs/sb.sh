# strip bench of the in-tree header with extra -D flags: tools/runs/sb.sh "-DTQR_STAGGER=0" ...
i=0
for f in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include $f -o tools/strip_bench_v$i tools/strip_bench.cu -lcuda &
  i=$((i+1))
done; wait
i=0
for f in "$@"; do echo "== $f"; ./tools/strip_bench_v$i | grep "tma=1 ctas=148"; i=$((i+1)); done
