#!/bin/bash
# One full ncu capture: bash tools/ncu_one.sh REGEX SKIP OUTNAME
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
  -o gpurun_out/$3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo "$3 exit $?"
