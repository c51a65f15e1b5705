# Build knobs for the 64-bin exhaustive kernel: rebuild with each EXTRA flag in
# $KNOBS (scratch copy of csrc/), time C2 at 64 bins (tools/bench_exh_configs.py), restore.
KNOBS=${KNOBS:-"-DKB_SKIP_BOUNDARY"}
LIB=$PWD/paper_1310_6736_b200/libsalvox_b200.so
cp $LIB /tmp/lib_orig.so
for k in $KNOBS; do
  K=paper_1310_6736_b200/csrc_knob; rm -rf $K && cp -r paper_1310_6736_b200/csrc $K && rm -f $K/*.o
  make -s -C $K EXTRA="$k" OUT=$LIB > /tmp/k65_build.log 2>&1 || { echo "build $k failed"; tail -3 /tmp/k65_build.log; continue; }
  timeout 300 python tools/bench_exh_configs.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('knob $k', round(d['C2 256^3 64 bins']['ms'],2), 'ms (32 bins:', round(d['C2 256^3 32 bins']['ms'],2), ')')"
done
cp /tmp/lib_orig.so $LIB
rm -rf paper_1310_6736_b200/csrc_knob
