mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_shard.py -m gpu -q > gpurun_out/pytest_gpu_r2g_shard.log 2>&1; echo "pytest shard exit $?"; tail -n 3 gpurun_out/pytest_gpu_r2g_shard.log
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2g_shard_peer.json 2> /dev/null; echo "bench shard peer exit $?"
python tools/ab_table.py gpurun_out/bench_r2g_shard_peer.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_shard_launches.csv python bench.py --force-shard --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/ncu_c5_launches.csv python bench.py --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu $?"
