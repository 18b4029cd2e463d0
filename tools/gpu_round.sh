#!/bin/bash
# One gpurun pass: GPU tests, then bench lines (C5 default, C4, sharded path).
# Usage: gpurun --timeout 3000 -- bash tools/gpu_round.sh TAG [pytest-args...]
TAG=${1:-r2}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench c5 exit $?"
timeout 600 python bench.py --config C4 > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err; echo "bench c4 exit $?"
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_${TAG}_shard.json 2> gpurun_out/bench_${TAG}_shard.err; echo "bench shard exit $?"
