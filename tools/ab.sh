#!/bin/bash
# A/B of experiment builds (tools/build_var.py): tools/ab.sh V [V ...]
# per variant: result digest (tools/ab_check.py) + the C5 launch sequence.
L=paper_0810_3203_b200/lib
cp $L/libcftft_b200.so $L/keep.so
for v in "$@"; do
  cp $L/var_$v.so $L/libcftft_b200.so
  echo "=== variant $v"
  timeout 300 python tools/ab_check.py 2>&1 | tail -1
  timeout 300 python tools/launch_seq.py C5 4 2>&1 | grep -v "wave_kernel\|0.0[0-9][0-9] ms"
done
cp $L/keep.so $L/libcftft_b200.so
