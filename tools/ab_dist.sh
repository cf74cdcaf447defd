#!/bin/bash
# A/B of experiment builds on the multi-GPU path (one rank): tools/ab_dist.sh V [V ...]
L=paper_0810_3203_b200/lib
cp $L/libcftft_b200.so $L/keep.so
for v in "$@"; do
  cp $L/var_$v.so $L/libcftft_b200.so
  echo "=== variant $v"
  timeout 300 python tools/ab_check.py 2>&1 | tail -1
  timeout 300 python tools/launch_seq.py C5 4 2>&1 | grep "launches"
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k native_dist 2>&1 | tail -3
  timeout 600 python bench.py --force-dist --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1
done
cp $L/keep.so $L/libcftft_b200.so
