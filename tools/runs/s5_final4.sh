# session 5 closing run (final build incl. per-k-step W2 fragment loads): GPU suite, smoke, bench, reference arm, launch list
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5h_gputest.log 2>&1; echo rc=$? >> gpurun_out/s5h_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5h_smoke.log 2>&1; echo rc=$? >> gpurun_out/s5h_smoke.log
python bench.py > gpurun_out/s5h_bench.json 2> gpurun_out/s5h_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s5h_bench_ref.json 2> gpurun_out/s5h_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5h_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s5h_ncu_bench.log 2>&1
mkdir -p /tmp/ncu
args=""
for c in greedy:1:TT fibonacci:1:TT flat:1:TT greedy:1:TS fibonacci:1:TS flat:1:TS; do
  n=$(echo $c | tr ':' '_')
  timeout 600 ncu --set full --import-source off --clock-control none -k regex:tqr_persistent --launch-skip 1 -c 1 -f -o /tmp/ncu/$n python tools/ncu_one.py 40 40 200 $c > gpurun_out/s5h_ncu_$n.log 2>&1
  args="$args $c=/tmp/ncu/$n.ncu-rep"
done
python tools/ncu_cases.py gpurun_out/s5h_ncu_cases.json "ncu --set full --clock-control none -k regex:tqr_persistent --launch-skip 1 -c 1 python tools/ncu_one.py 40 40 200 <case> (configs[2], one report per bench.py case, the measured launch after one warm-up)" $args > gpurun_out/s5h_ncu_cases.log 2>&1
timeout 600 python bench.py --workload cfg1 --no-cpu-baseline > gpurun_out/s5h_bench_cfg1.json 2> gpurun_out/s5h_cfg1.err
