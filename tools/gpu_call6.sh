mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/pytest_gpu_r2f_shard.log 2>&1; echo "pytest shard exit $?"; tail -n 15 gpurun_out/pytest_gpu_r2f_shard.log
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2f_shard_peer.json 2> gpurun_out/bench_r2f_shard_peer.err; echo "bench shard peer exit $?"; tail -n 3 gpurun_out/bench_r2f_shard_peer.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2f_c5.json 2>/dev/null; echo "bench c5 $?"
DYG_REACH_SPLIT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2f_c5_nosplit.json 2>/dev/null; echo "bench c5 nosplit $?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2f_c5_b.json 2>/dev/null; echo "bench c5 $?"
DYG_REACH_SPLIT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2f_c5_nosplit_b.json 2>/dev/null; echo "bench c5 nosplit $?"
python tools/ab_table.py gpurun_out/bench_r2f_*.json
