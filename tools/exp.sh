#!/bin/bash
# quick A/B of engine options on bench lines: tools/exp.sh "ENV=.. ENV2=.." ... -- C5 C2
opts=(); while [ "$1" != "--" ] && [ -n "$1" ]; do opts+=("$1"); shift; done; shift
for cfg in "$@"; do
  for v in "${opts[@]}"; do
    [ "$v" = "-" ] && v=""
    echo -n "[$v] "; env $v BENCH_ARGS="" timeout 200 bash tools/benchline.sh $cfg 2>&1 | tail -1
  done
done
