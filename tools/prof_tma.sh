#!/bin/bash
# ncu of the C5 TFT TMA waves: launch list + one full capture + stall summary.
# usage: tools/prof_tma.sh TAG [SKIP]
TAG=$1; SKIP=${2:-1}
bash tools/prof_waves.sh $TAG 1 tft coset_tma $SKIP
python tools/launch_summary.py gpurun_out/launches_$TAG.csv
python tools/ncu_stalls.py gpurun_out/full_$TAG.ncu-rep
ncu -i gpurun_out/full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$TAG.csv 2>/dev/null
