# ncu --set full of the seek kernels (one launch each) + the reference arm line.
for cfg in ${CFGS:-"C3:shift_cta_kernel" "C1:shift_kernel" "C1:ascent_kernel" "PAPER MR:abmsod_cta_kernel"}; do
  name=${cfg%%:*}; kern=${cfg##*:}; tag=$(echo "$name-$kern" | tr ' ' '_')
  timeout 600 ncu --set full --clock-control none --kernel-name regex:$kern --launch-skip 1 --launch-count 1 -o gpurun_out/seek_$tag python tools/bench_seek.py --c5 0 --only "$name" > gpurun_out/seek_$tag.log 2>&1; echo "$name rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.jsonl 2> gpurun_out/ref.err; echo "ref rc=$?"
