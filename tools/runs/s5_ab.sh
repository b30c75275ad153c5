# session 5: A/B of a variant library against the default build (configs[2] and configs[1])
V=$1
C="greedy:1:TT,flat:1:TS"
for lib in "" tools/variants/$V.so "" tools/variants/$V.so; do
  echo "== lib=${lib:-default}"
  TQR_LIB=$lib timeout 300 python tools/quick_time.py 40 40 200 32 $C | cut -c1-70
done
echo "== parity of the variant"
TQR_LIB=tools/variants/$V.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
