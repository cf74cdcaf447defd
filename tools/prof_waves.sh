#!/bin/bash
# ncu of one C5 transform under a given engine mode: launch list with DRAM
# bytes, and one --set full capture of launch number SKIP of kernel REGEX.
# usage: tools/prof_waves.sh TAG WIDE [tft|itft] [REGEX] [SKIP]
TAG=$1; WIDE=$2; WHICH=${3:-tft}; RX=${4:-coset_tma}; SKIP=${5:-1}
export CFTFT_WIDE=$WIDE
python tools/prof_one.py C5 $WHICH > gpurun_out/p_$TAG.log 2>&1 || { echo plain-failed; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum \
  --clock-control none -k regex:"coset|leaf|fold" --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_one.py C5 $WHICH \
  > gpurun_out/ncu_l_$TAG.log 2>&1; echo ncu-list=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SKIP -c 1 -f -o gpurun_out/full_$TAG \
  python tools/prof_one.py C5 $WHICH > gpurun_out/ncu_f_$TAG.log 2>&1; echo ncu-full=$?
