timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/pr.log 2>&1
python - <<'P'
import json
for l in open('gpurun_out/pr.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('kb_ms', r['kb_ms_per_launch'], 'frac', r['frac'], 'peak', r['peak'], 'prmt', r['atoms_prmt_walk_peak'], 'pair', r['pair_peak'])
P
tail -3 gpurun_out/pr.log | grep -i error
