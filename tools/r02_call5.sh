#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "k3d" > gpurun_out/pytest_k3d.log 2>&1
timeout 600 python tools/try_pair.py 0,5 > gpurun_out/try_pair.log 2>&1
for w in 6,5 7,5 7,6 8,6 9,7 10,6; do for pf in 0 4 8; do
  echo "warps $w pf $pf: $(DGDIFF_TUNING_LIB=1 DGDIFF_PAIR_WARPS=$w DGDIFF_PAIR_PF=$pf PAIR_CASES=c4_p1_fp64 timeout 300 python tools/try_pair.py 5 2>&1 | tail -1)" >> gpurun_out/pair_sweep.log
done; done
tail -3 gpurun_out/pytest_k3d.log; cat gpurun_out/try_pair.log gpurun_out/pair_sweep.log
