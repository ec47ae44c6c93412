# A/B for the quad / P3 ring configs on c5 (64 sources)
run() { echo "$1 [$2] $3: $(eval $3 DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --nsteps 2 --reps 1 $2 2>&1 | grep '\[dgdiff\]' | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"; }
for rep in 1 2; do
  for v in qfull qnc; do
    cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
    for c in "--degree 2 --element 1" "--degree 1 --element 1" "--degree 3"; do
      run $v "$c" ""
      [ $v = qfull ] && run $v "$c" "DGDIFF_RING=72,0"
    done
  done
done
