export SALVOX_KB_VARIANT=${SALVOX_KB_VARIANT:-3}
timeout 600 python -m pytest -q -m gpu tests/test_gpu_exhaustive.py tests/test_golden.py -k "exh or square or squares or histograms or slabs or scales or range" -x > gpurun_out/q3_tests.log 2>&1; tail -1 gpurun_out/q3_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/q3_bench.log 2>&1
python - <<'P'
import json
for l in open('gpurun_out/q3_bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('kb_ms', d['roofline']['kb_ms_per_launch'], 'ms/step', d['ms_per_step'])
P
if [ "${NCU:-0}" = 1 ]; then timeout 600 ncu --section WarpStateStats --section SchedulerStats --section InstructionStats --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none --kernel-name regex:kb_quad_kernel --launch-skip 1 --launch-count 1 --section SourceCounters --import-source on -o gpurun_out/quad6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-seed-grid > gpurun_out/quad6_ncu.log 2>&1; tail -1 gpurun_out/quad6_ncu.log; fi
