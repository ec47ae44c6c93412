for ah in 4,4 6,6 8,8 10,10 12,12 15,15; do
  for cfg in "" "--config c2 --sources 1024"; do
    echo "AHEAD=$ah $cfg"
    DGDIFF_AHEAD=$ah DGDIFF_STAGE_DETAIL=1 timeout 60 python tools/prof_stage.py --kernel 0 --nsteps 2 --reps 2 $cfg 2>&1 | grep "stage" | tail -3 | tr '\n' ' '
    echo
  done
done
