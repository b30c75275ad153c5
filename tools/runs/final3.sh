timeout 900 ncu --set full --import-source on --clock-control none -k regex:tqr_persistent -c 12 -o /tmp/full_square_f1 -f python tools/ncu_one.py > gpurun_out/ncu_full_sq.log 2>&1; echo full rc=$?
python tools/ncu_summary.py /tmp/full_square_f1.ncu-rep gpurun_out/ncu_full_summary_square.json "ncu --set full --import-source on --clock-control none -k regex:tqr_persistent -c 12 python tools/ncu_one.py (configs[2]: the six bench.py cases, warm-up + measured launch each; per-launch figures = mean over the 6 measured launches)" 2
ncu -i /tmp/full_square_f1.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
ks=[k for k in h if ('dram__bytes' in k and k.endswith('.sum')) or k in ('gpu__time_duration.sum','sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__inst_executed_pipe_fp64.sum')]
print(ks)
for r in rows[2:]:
    if len(r)==len(h): d=dict(zip(h,r)); print([d[k] for k in ks])
" > gpurun_out/ncu_square_per_launch.txt
