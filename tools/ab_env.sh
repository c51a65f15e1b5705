# A/B of environment knobs of the exhaustive path on one B200: the exhaustive
# parity suites under each setting in $ENVS (space-separated NAME=VALUE, use
# commas to set several at once), then the C2 bench step for each, alternating
# over $ROUNDS rounds (GPU clocks drift; compare within a round).
ENVS=${ENVS:-"SALVOX_KB_VB=1 SALVOX_KB_VB=2"}
ROUNDS=${ROUNDS:-2}
for e in $ENVS; do
  [ "${SKIP_TESTS:-0}" = 1 ] && break
  env ${e//,/ } timeout 600 python -m pytest -q -m gpu tests/test_gpu_exhaustive.py tests/test_golden.py tests/test_gpu_reference.py -k "exh or square or squares or histograms or slabs or scales or range" -x -p no:cacheprovider > gpurun_out/abe_tests.log 2>&1; echo "$e tests: $(tail -1 gpurun_out/abe_tests.log)"
done
for r in $(seq $ROUNDS); do
  for e in $ENVS; do
    env ${e//,/ } timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/abe_bench.log 2>&1
    python - "$e" <<'P'
import json, sys
for l in open('gpurun_out/abe_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], 'kb_ms', round(d['roofline']['kb_ms_per_launch'],2), 'ms/step', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3), 'e2e_ms', round(d['e2e'].get('ms_per_step', 0),2), 'clk', d['clocks']['sm_mhz'])
P
  done
done
