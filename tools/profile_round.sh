#!/bin/bash
# Evidence pass: bench line, ncu launch lists (unsharded and --force-shard),
# full captures of K1 (reach, C5 insertion batch 6), K2 (min-path, deletion
# batch 14) and k_del_flow, their summaries, and the random-gather probe.
# Usage: gpurun -- bash tools/profile_round.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_peak tools/gather_peak.cu && ./tools/gather_peak > gpurun_out/gather_peak_$TAG.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?"
for mode in c5 shard; do
  extra=""; [ $mode = shard ] && extra="--force-shard"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/ncu_${mode}_launches_$TAG.csv python bench.py $extra --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "launches $mode exit $?"
  python tools/ncu_launch_summary.py gpurun_out/ncu_${mode}_launches_$TAG.csv 45 > gpurun_out/ncu_launches_${TAG}_$mode.txt
done
cap() {  # REGEX SKIP NAME
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
    -o gpurun_out/prof_$3_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "$3 exit $?"
}
cap k_walk 26 k1   # the 2nd replay (the 1st runs the instrumented kernels)
cap k_walk 34 k2
cap k_del_flow 6 flow
python tools/ncu_summary.py gpurun_out/prof_k1_$TAG.ncu-rep gpurun_out/prof_k2_$TAG.ncu-rep \
  gpurun_out/prof_flow_$TAG.ncu-rep > gpurun_out/ncu_summary_$TAG.txt 2>&1
