#!/bin/bash
# Bench the working tree and each _ab/VARIANT alternately (ROUNDS rounds):
# bash tools/ab_run.sh TAG ROUNDS VARIANT...   -> gpurun_out/ab_TAG_<variant>_<round>.json
TAG=$1; ROUNDS=$2; shift 2
mkdir -p gpurun_out
for r in $(seq 1 $ROUNDS); do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_${TAG}_main_$r.json 2>/dev/null; echo "main $r $?"
  for v in "$@"; do
    (cd _ab/$v && timeout 600 python bench.py --no-cpu-baseline > ../../gpurun_out/ab_${TAG}_${v}_$r.json 2>/dev/null); echo "$v $r $?"
  done
done
python tools/ab_table.py gpurun_out/ab_${TAG}_*.json
