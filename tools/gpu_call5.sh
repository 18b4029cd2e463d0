mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_walks.py tests/test_gpu_replay.py tests/test_gpu_c5.py -m gpu -x -q > gpurun_out/pytest_gpu_r2e.log 2>&1; echo "pytest exit $?"; tail -n 2 gpurun_out/pytest_gpu_r2e.log
bash tools/ab_run.sh k1b 2 k1_3blk
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2e_shard.json 2> gpurun_out/bench_r2e_shard.err; echo "bench shard exit $?"
timeout 900 python bench.py --config C4 > gpurun_out/bench_r2e_c4.json 2> gpurun_out/bench_r2e_c4.err; echo "bench c4 exit $?"
python tools/ab_table.py gpurun_out/bench_r2e_shard.json gpurun_out/bench_r2e_c4.json
