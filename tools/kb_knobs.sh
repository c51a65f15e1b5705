# Profiling knobs of the exhaustive kernel: rebuild the library with each EXTRA
# flag set in $KNOBS (a scratch copy of csrc/), time the C2 bench step, restore.
KNOBS=${KNOBS:-"-DKB_SKIP_MATH -DKB_SKIP_BOUNDARY"}
LIB=$PWD/paper_1310_6736_b200/libsalvox_b200.so
cp $LIB /tmp/lib_orig.so
for k in $KNOBS; do
  K=paper_1310_6736_b200/csrc_knob; rm -rf $K && cp -r paper_1310_6736_b200/csrc $K && rm -f $K/*.o
  make -s -C $K EXTRA="$k" OUT=$LIB > /tmp/kbk_build.log 2>&1 || { echo "build $k failed"; tail /tmp/kbk_build.log; continue; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/knob.log 2>&1
  python - "$k" <<'P'
import json, sys
for l in open('gpurun_out/knob.log'):
    if l.startswith('{'):
        d=json.loads(l); print('knob', sys.argv[1], 'kb_ms', round(d['roofline']['kb_ms_per_launch'],2), 'ms/step', round(d['ms_per_step'],2))
P
done
cp /tmp/lib_orig.so $LIB
rm -rf paper_1310_6736_b200/csrc_knob
