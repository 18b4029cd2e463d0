#!/bin/bash
# Full ncu captures of the per-batch prepare and commit kernels (C5, one launch each,
# late in the warm-up replay). Usage: gpurun -- bash tools/ncu_commit.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
for k in "k_prep<0>:k_prep:6" "k_del_flow:k_del_flow:6" "k_prep<1>:k_prep:16"; do
  IFS=: read name rx skip <<< "$k"
  tag=$(echo $name | tr -d '<>')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
    -o gpurun_out/prof_${tag}_$TAG -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "$name exit $?"
done
