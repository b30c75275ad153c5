# A/B of library variants: tools/runs/ab.sh "A B C" "p q nb ib trees"
for v in $1; do
  echo "== $v"
  TQR_LIB=tools/variants/$v.so timeout 300 python tools/quick_time.py $2
done
