# A/B of exhaustive kernel variants on one B200: parity suites under each
# variant in $VARIANTS (default "4"), then the C2 bench step for 3 and each.
VARIANTS=${VARIANTS:-4}
for v in $VARIANTS; do
  SALVOX_KB_VARIANT=$v timeout 600 python -m pytest -q -m gpu tests/test_gpu_exhaustive.py tests/test_golden.py -k "exh or square or squares or histograms or slabs or scales or range" -x > gpurun_out/ab_tests_$v.log 2>&1; echo "variant $v tests: $(tail -1 gpurun_out/ab_tests_$v.log)"
done
for v in 3 $VARIANTS; do
  SALVOX_KB_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/ab_bench_$v.log 2>&1
  python - $v <<'P'
import json, sys
for l in open(f'gpurun_out/ab_bench_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d=json.loads(l); print('variant', sys.argv[1], 'kb_ms', round(d['roofline']['kb_ms_per_launch'],2), 'ms/step', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
P
done
