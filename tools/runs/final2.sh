timeout 900 python bench.py > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err; tail -c 200 gpurun_out/bench_f1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_f1.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tqr_persistent -c 12 -o /tmp/full_square_f1 -f python tools/ncu_one.py > gpurun_out/ncu_full_sq.log 2>&1; echo full rc=$?
python tools/ncu_summary.py /tmp/full_square_f1.ncu-rep gpurun_out/ncu_full_summary_square.json "ncu --set full --clock-control none -k regex:tqr_persistent -c 12 python tools/ncu_one.py (configs[2], six cases, measured launches)" 2 > /dev/null
python tools/ncu_lines.py /tmp/full_square_f1.ncu-rep 40 > gpurun_out/ncu_lines_square.txt 2>&1
ncu -i /tmp/full_square_f1.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null; python - <<'PY' > gpurun_out/ncu_stalls_square.txt
import csv
rows=list(csv.reader(open('/tmp/raw.csv')))
h=rows[0]
for r in rows[2:]:
    if len(r)!=len(h): continue
    d=dict(zip(h,r))
    st={k:float(v.replace(',','')) for k,v in d.items() if 'pcsamp_warps_issue_stalled' in k and 'not_issued' not in k}
    tot=sum(st.values()) or 1
    top=sorted(st.items(),key=lambda x:-x[1])[:8]
    print(d.get('gpu__time_duration.sum'), ' '.join(f"{k.split('stalled_')[1]}={100*v/tot:.1f}%" for k,v in top))
PY
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tqr_persistent -c 2 --csv --log-file gpurun_out/tall_dram_f1.csv python tools/ncu_one.py 2048 16 256 greedy:1:TT > gpurun_out/ncu_tall.log 2>&1; echo tall rc=$?
du -sh gpurun_out
