# One ncu capture of the exhaustive kernel (variant $SALVOX_KB_VARIANT) on the C2 bench step.
v=${SALVOX_KB_VARIANT:-3}
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:kb_quad_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/kb_v$v python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-seed-grid > gpurun_out/kb_v${v}_ncu.log 2>&1; tail -2 gpurun_out/kb_v${v}_ncu.log
