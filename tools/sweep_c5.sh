# c5 P2 stage-1 ring sweep: ring-1 depth (DGDIFF_RING=n1,0) and lookahead (DGDIFF_AHEAD=a,n)
for r in "" "40,0" "73,0"; do
  for ah in "" "0,8" "0,12"; do
    echo "ring=$r ahead=$ah: $(DGDIFF_RING=$r DGDIFF_AHEAD=$ah DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --degree 2 --nsteps 2 --reps 1 2>&1 | grep '\[dgdiff\]' | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"
  done
done
