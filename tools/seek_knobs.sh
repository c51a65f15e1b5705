# Seek-kernel build knobs: rebuild with each EXTRA flag in $KNOBS (a scratch copy
# of csrc/), run the seek parity suites and time C3 / paper shapes, restore.
KNOBS=${KNOBS:-"-DCTA_MINB=1 -DCTA_MINB=6"}
LIB=$PWD/paper_1310_6736_b200/libsalvox_b200.so
cp $LIB /tmp/lib_orig.so
for k in $KNOBS; do
  K=paper_1310_6736_b200/csrc_knob; rm -rf $K && cp -r paper_1310_6736_b200/csrc $K && rm -f $K/*.o
  make -s -C $K EXTRA="$k" OUT=$LIB > /tmp/kbk_build.log 2>&1 || { echo "build $k failed"; tail /tmp/kbk_build.log; continue; }
  grep -A2 "shift_cta_kernel" $K/seek.ptxas.log | grep -m1 registers
  timeout 600 python -m pytest -q -m gpu tests/test_gpu_seek.py tests/test_gpu_abmsod.py -x > gpurun_out/seekk_tests.log 2>&1; echo "knob $k tests: $(tail -1 gpurun_out/seekk_tests.log)"
  timeout 600 python tools/bench_seek.py --c5 0 --only "${ONLY:-}" > gpurun_out/seekk.log 2>&1; echo "knob $k"; cut -c1-160 gpurun_out/seekk.log
done
cp /tmp/lib_orig.so $LIB
rm -rf paper_1310_6736_b200/csrc_knob
