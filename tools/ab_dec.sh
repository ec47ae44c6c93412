# K3b role-count A/B on the c4 chunk (ms per step) + parity spot check
for v in dec544 decpf; do
  cp scratch_libs/libdgdiff_$v.so paper_1907_06191_b200/libdgdiff.so
  echo "$v: $(timeout 300 python tools/try_dec.py 2>&1 | grep -E 'ts 3|rand' | tr '\n' ' ')"
done
