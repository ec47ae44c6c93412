cp paper_1907_06191_b200/libdgdiff.so /tmp/keep.so
for v in base fake base fake; do
cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
echo "$v: $(DGDIFF_STAGE_DETAIL=1 timeout 120 python tools/prof_stage.py --config c5 --sources 64 --degree 3 --nsteps 1 --reps 3 2>&1 | grep -i '\[dgdiff\]\|error' | tail -3 | tr '\n' ' ')"
done
cp /tmp/keep.so paper_1907_06191_b200/libdgdiff.so
