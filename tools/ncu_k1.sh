#!/bin/bash
# One full ncu capture of the first C5 reach-walk launch (K1): bash tools/ncu_k1.sh TAG
TAG=${1:-k1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 0 -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?"
