run() { echo "$1 $2 :: $(env $1 DGDIFF_STAGE_DETAIL=1 timeout 60 python tools/prof_stage.py --kernel 0 --nsteps 2 --reps 2 $2 2>&1 | grep '\[dgdiff\]' | tail -3 | sed 's/\[dgdiff\] //g' | tr '\n' ' ')"; }
for v in "DGDIFF_STAGGER=0" "DGDIFF_STAGGER=4096" "DGDIFF_STAGGER=65536" "DGDIFF_STAGGER=1048576" "DGDIFF_STAGGER=7340288" "DGDIFF_RING=40,0"; do run "$v" ""; done
for v in "DGDIFF_STAGGER=7340288 DGDIFF_RING=40,0" "DGDIFF_STAGGER=65536 DGDIFF_RING=40,0"; do run "$v" ""; done
