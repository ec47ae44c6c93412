# A/B prebuilt library variants on c5 Q1/Q2 fp64: bash tools/ab_q.sh v1 v2 ...
cp paper_1907_06191_b200/libdgdiff.so /tmp/libdgdiff_keep.so
for rep in 1 2; do
for v in "$@"; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  for d in 2 1; do
  echo "$v Q$d: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --degree $d --element 1 --nsteps 8 --reps 2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
done
cp /tmp/libdgdiff_keep.so paper_1907_06191_b200/libdgdiff.so
