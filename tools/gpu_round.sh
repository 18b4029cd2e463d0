#!/bin/bash
# One gpurun pass: the GPU test suite, smoke(), then bench lines (C5 with the
# CPU baseline, the reference arm, C4, the sharded path over both transports).
# Usage: gpurun --timeout 3600 -- bash tools/gpu_round.sh TAG [pytest-args...]
TAG=${1:-r2}; shift
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?"
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "bench ref exit $?"
timeout 900 python bench.py --config C4 > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err; echo "bench c4 exit $?"
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_${TAG}_shard_peer.json 2> gpurun_out/bench_${TAG}_shard_peer.err; echo "bench shard peer exit $?"
timeout 600 python bench.py --force-shard --no-cpu-baseline --transport collective > gpurun_out/bench_${TAG}_shard_coll.json 2> gpurun_out/bench_${TAG}_shard_coll.err; echo "bench shard collective exit $?"
python tools/ab_table.py gpurun_out/bench_${TAG}_*.json
