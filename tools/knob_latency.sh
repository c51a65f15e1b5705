LIB=$PWD/paper_1310_6736_b200/libsalvox_b200.so
cp $LIB /tmp/lib_orig.so
timeout 300 python tools/c3_longest.py
for k in ${KNOBS:--DSEEK_DOUBLE_CHAINS}; do
  K=paper_1310_6736_b200/csrc_knob; rm -rf $K && cp -r paper_1310_6736_b200/csrc $K && rm -f $K/*.o
  make -s -C $K EXTRA="$k" OUT=$LIB > /tmp/kbk_build.log 2>&1 || { echo "build $k failed"; tail -3 /tmp/kbk_build.log; continue; }
  echo "knob $k: $(timeout 300 python tools/c3_longest.py)"
  timeout 300 python tools/bench_seek.py --c5 0 --only "C3" | cut -c1-100
done
cp /tmp/lib_orig.so $LIB
rm -rf paper_1310_6736_b200/csrc_knob
