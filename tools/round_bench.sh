#!/bin/bash
# Full measurement pass on one GPU: bench lines (C5 default + C2 + C4), the
# reference arm, the ncu launch list of the bench command, DRAM traffic of the
# leaf kernels, one ncu --set full capture of the C5 TFT leaf kernel.
# usage: tools/round_bench.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench C5 rc=$?"
tail -1 gpurun_out/bench_${TAG}_c5.json
for c in C2 C4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$c.json 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${TAG}_$c.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_${TAG}.json 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/ref_${TAG}.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "ncu launches rc=$?"
for w in tft itft; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"leaf_kernel|coset_wave|fold" --csv --log-file gpurun_out/traffic_${TAG}_c5_$w.csv python tools/prof_one.py C5 $w \
    > gpurun_out/ncu_traffic_${TAG}_$w.log 2>&1; echo "ncu traffic $w rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coset_wave -s 3 -c 1 -f -o gpurun_out/full_${TAG}_c5tft_unal \
  python tools/prof_one.py C5 tft > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coset_wave -c 1 -f -o gpurun_out/full_${TAG}_c5tft_wave \
  python tools/prof_one.py C5 tft > gpurun_out/ncu_full_wave_${TAG}.log 2>&1; echo "ncu full wave rc=$?"
