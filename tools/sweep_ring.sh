# A/B of ring capacity / lookahead within one GPU session (stage times per variant)
run() { echo "$1 $2 :: $(env $1 DGDIFF_STAGE_DETAIL=1 timeout 60 python tools/prof_stage.py --kernel 0 --nsteps 2 --reps 2 $2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"; }
for rep in 1 2; do
for v in "DGDIFF_RING=40,0" "DGDIFF_RING=56,0" "DGDIFF_RING=0,0" "DGDIFF_AHEAD=15,6" "DGDIFF_AHEAD=15,10"; do
  run "$v" ""
done
done
for v in "DGDIFF_RING=40,0" "DGDIFF_RING=0,0"; do run "$v" "--config c2 --sources 1024"; done
