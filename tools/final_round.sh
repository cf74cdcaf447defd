#!/bin/bash
# Full measurement pass on one B200 (everything lands in gpurun_out/, TAG-named):
# GPU test suite, bench lines (C5 default with e2e + CPU baselines, reference arm,
# C1 C2 C4 G, the multi-GPU path on one rank), multiplication pipeline times,
# the ncu launch list of the bench command, per-launch DRAM traffic of one
# TFT + one ITFT, and ncu --set full captures of the dominant kernel
# (the unaligned TFT pass and the ITFT's truncated column wave).
# usage: tools/final_round.sh TAG
TAG=${1:-run}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu_$TAG.log
timeout 900 python bench.py > $O/bench_${TAG}_c5.json 2> $O/bench_${TAG}_c5.err; echo "bench C5 rc=$?"; tail -1 $O/bench_${TAG}_c5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_$TAG.json 2> $O/ref_$TAG.err; echo "ref rc=$?"; tail -1 $O/ref_$TAG.json
for c in C1 C2 C4 G; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err; echo "bench $c rc=$?"
  tail -1 $O/bench_${TAG}_$c.json
done
timeout 600 python bench.py --force-dist --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_${TAG}_dist.json 2> $O/bench_${TAG}_dist.err; echo "bench dist rc=$?"
tail -1 $O/bench_${TAG}_dist.json
timeout 600 python tools/mul_times.py > $O/mul_times_$TAG.txt 2>&1; echo "mul_times rc=$?"; tail -4 $O/mul_times_$TAG.txt
timeout 300 python tools/launch_seq.py C5 4 > $O/seq_c5_$TAG.txt 2>&1; cat $O/seq_c5_$TAG.txt
timeout 300 python tools/c1_time.py > $O/c1_time_$TAG.txt 2>&1; tail -3 $O/c1_time_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_${TAG}_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
for w in tft itft; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"coset|leaf|fold|rotate|copy" --csv --log-file $O/traffic_${TAG}_c5_$w.csv python tools/prof_one.py C5 $w \
    > $O/ncu_traffic_${TAG}_$w.log 2>&1; echo "ncu traffic $w rc=$?"
done
bash tools/prof_wave.sh ${TAG}_tft2 tft coset_tma 1
bash tools/prof_wave.sh ${TAG}_itft_last itft coset_tma 4
bash tools/prof_wave.sh ${TAG}_fold tft cs_fold 0
