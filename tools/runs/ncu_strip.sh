nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/strip_bench tools/strip_bench.cu -lcuda
./tools/strip_bench > gpurun_out/strip_bench_now.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_strip -s 5 -c 1 -o gpurun_out/strip_un -f ./tools/strip_bench > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_strip -s 15 -c 1 -o gpurun_out/strip_tt -f ./tools/strip_bench > /dev/null 2>&1
ls -la gpurun_out
