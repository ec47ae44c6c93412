# A/B of prebuilt fp32 variants: bash tools/ab32.sh v1 v2 ...
for rep in 1 2; do
for v in "$@"; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  for c in "--config c4 --sources 512" "--config c2 --sources 1024" "--config c2 --sources 1024 --degree 2"; do
    echo "$v [$c]: $(DGDIFF_STAGE_DETAIL=1 timeout 60 python tools/prof_stage.py --precision 32 --nsteps 2 --reps 1 $c 2>&1 | grep '\[dgdiff\]' | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
done
