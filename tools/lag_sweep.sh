for L in ${LAGS:-0 10000 20000 30000}; do
  SALVOX_KB_LAG=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/lag.log 2>&1
  python - $L <<'P'
import json, sys
for l in open('gpurun_out/lag.log'):
    if l.startswith('{'):
        d=json.loads(l); print('lag', sys.argv[1], 'kb_ms', round(d['roofline']['kb_ms_per_launch'],2))
P
done
