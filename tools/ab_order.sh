# A/B of the MAC issue order on every element type
for rep in 1 2; do
for v in rowmajor colmajor; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  for c in "--config c4 --sources 256" "--config c5 --sources 64 --degree 2" "--config c5 --sources 64 --degree 3" "--config c5 --sources 64 --degree 2 --element 1" "--config c4 --sources 512 --precision 32"; do
    echo "$v [$c]: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --nsteps 2 --reps 1 $c 2>&1 | grep '\[dgdiff\]' | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
done
