# 64-bin exhaustive variants (SALVOX_KB65 = quad | tmem | kb) at C2, two rounds
for r in 1 2; do for v in quad tmem kb; do
  SALVOX_KB65=$v timeout 300 python tools/bench_exh_configs.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', round(d['C2 256^3 64 bins']['ms'],2))"
done; done
