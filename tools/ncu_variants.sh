# ncu --set full of one stage-1 and one alpha-stage launch for the P2, P3 and Q2
# ring kernels on the c5 substrate (64 sources); run each command once without
# ncu first (the recipe's rule)
set -e
mkdir -p gpurun_out
for v in "--degree 2" "--degree 3" "--degree 2 --element 1"; do
  timeout 120 python tools/prof_stage.py --config c5 --sources 64 --nsteps 1 --reps 1 $v > /dev/null
done
i=0
for v in "--degree 2" "--degree 3" "--degree 2 --element 1"; do
  i=$((i+1))
  timeout 900 ncu --set full --clock-control none -k regex:k_stage_ring -c 2 -o gpurun_out/var$i \
    python tools/prof_stage.py --config c5 --sources 64 --nsteps 1 --reps 1 $v > gpurun_out/ncu_var$i.log 2>&1
  tail -1 gpurun_out/ncu_var$i.log
done
