#!/bin/bash
# one ncu --set full capture of launch number SKIP of kernel REGEX in one C5 transform:
# tools/prof_wave.sh TAG tft|itft REGEX SKIP
TAG=$1; WHICH=$2; RX=$3; SKIP=$4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c 1 -f -o gpurun_out/full_$TAG \
  python tools/prof_one.py C5 $WHICH > gpurun_out/ncu_f_$TAG.log 2>&1; echo ncu-full-$TAG=$?
