for pad in 0 40000 90000; do
  for cfg in "" "--config c2 --sources 1024"; do
    echo "PAD=$pad $cfg: $(DGDIFF_SMEM_PAD=$pad DGDIFF_STAGE_DETAIL=1 timeout 60 python tools/prof_stage.py --kernel 0 --nsteps 2 --reps 2 $cfg 2>&1 | grep '\[dgdiff\]' | tail -3 | tr '\n' ' ')"
  done
done
