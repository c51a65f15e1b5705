# Maxima-pass knobs: rebuild with each EXTRA flag in $KNOBS (scratch copy of
# csrc/), print maxima_tile_kernel's ncu durations on the C2 bench step, restore.
KNOBS=${KNOBS:-"-DMX_Z=16 -DMX_Z=8"}
LIB=$PWD/paper_1310_6736_b200/libsalvox_b200.so
cp $LIB /tmp/lib_orig.so
for k in $KNOBS; do
  K=paper_1310_6736_b200/csrc_knob; rm -rf $K && cp -r paper_1310_6736_b200/csrc $K && rm -f $K/*.o
  make -s -C $K EXTRA="$k" OUT=$LIB > /tmp/mxk_build.log 2>&1 || { echo "build $k failed"; tail /tmp/mxk_build.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:maxima_tile --csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-seed-grid > gpurun_out/mxk.csv 2>/dev/null
  echo "knob $k maxima_tile_kernel us: $(grep maxima_tile gpurun_out/mxk.csv | awk -F'","' '{gsub(/"/,"",$NF); printf "%.1f ", $NF/1000}')"
done
cp /tmp/lib_orig.so $LIB
rm -rf paper_1310_6736_b200/csrc_knob
