#!/bin/bash
# tools/exp_loop.sh CFG "ENV=.." ... : steady-state TFT/ITFT per option set (random data)
cfg=$1; shift
for v in "$@"; do
  [ "$v" = "-" ] && v=""
  echo "[$v]"; env $v timeout 300 python tools/loop_time.py $cfg 2>&1 | grep random
done
