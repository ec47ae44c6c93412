# A/B of prebuilt variants on the P2 workloads: bash tools/ab_p2.sh v1 v2 ...
for rep in 1 2; do
for v in "$@"; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  for c in "--config c2 --sources 1024 --degree 2" "--config c5 --sources 256 --degree 2" "--config c5 --sources 512 --degree 2 --precision 32"; do
    echo "$v [$c]: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --nsteps 2 --reps 1 $c 2>&1 | grep '\[dgdiff\]' | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
done
