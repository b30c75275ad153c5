TQR_LIB=tools/variants/wpv.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "production or schedule or apply_parity or fused" > gpurun_out/s4w_tests.log 2>&1; echo rc=$? >> gpurun_out/s4w_tests.log
bash tools/runs/ab.sh "base wpv base wpv" "40 40 200 32 greedy:1:TT,flat:1:TS" > gpurun_out/s4w_ab.txt 2>&1
bash tools/runs/ab.sh "base wpv" "40 10 200 32 greedy:1:TT,flat:1:TT" >> gpurun_out/s4w_ab.txt 2>&1
