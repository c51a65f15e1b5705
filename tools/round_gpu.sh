# one gpurun call: full GPU suite, bench line, launch list, one full ncu capture of the top kernel
set -u
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:kb_quad_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/kb_quad_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-seed-grid > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
