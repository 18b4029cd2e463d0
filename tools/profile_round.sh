#!/bin/bash
# Evidence pass: bench line, ncu launch list, full captures of K1 (reach) and K2 (min-path),
# and the random-gather roofline probe. Usage: gpurun -- bash tools/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_peak tools/gather_peak.cu && ./tools/gather_peak > gpurun_out/gather_peak_$TAG.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 6 -c 1 \
  -o gpurun_out/prof_k1_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 14 -c 1 \
  -o gpurun_out/prof_k2_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 exit $?"
