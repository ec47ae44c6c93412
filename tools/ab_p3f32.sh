cp paper_1907_06191_b200/libdgdiff.so /tmp/libdgdiff_keep.so
for rep in 1 2; do
for v in "$@"; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  echo "$v: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --degree 3 --precision 32 --nsteps 4 --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
done
done
cp /tmp/libdgdiff_keep.so paper_1907_06191_b200/libdgdiff.so
