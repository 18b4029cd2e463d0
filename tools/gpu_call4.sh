mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2d.log 2>&1; echo "pytest exit $?"; grep -E "FAILED|ERROR|passed|failed" gpurun_out/pytest_gpu_r2d.log | tail -8
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2d_shard.json 2> gpurun_out/bench_r2d_shard.err; echo "bench shard exit $?"
python tools/ab_table.py gpurun_out/bench_r2d_shard.json
bash tools/ab_run.sh k1 2 k1_4blk tail16 tail8
