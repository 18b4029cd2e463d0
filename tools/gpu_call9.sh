mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_dist.py tests/test_gpu_replay.py -m gpu -q > gpurun_out/pytest_gpu_r2i.log 2>&1; echo "pytest exit $?"; tail -n 3 gpurun_out/pytest_gpu_r2i.log
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2i_shard_peer.json 2> /dev/null; echo "bench shard $?"
python tools/ab_table.py gpurun_out/bench_r2i_shard_peer.json
timeout 900 python tools/spectral_bench.py 512 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 6 -c 1 -o gpurun_out/prof_k1_r2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 14 -c 1 -o gpurun_out/prof_k2_r2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_del_flow -s 6 -c 1 -o gpurun_out/prof_flow_r2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "flow exit $?"
python tools/ncu_summary.py gpurun_out/prof_k1_r2.ncu-rep gpurun_out/prof_k2_r2.ncu-rep gpurun_out/prof_flow_r2.ncu-rep > gpurun_out/ncu_summary_r2.txt 2>&1; echo "summary $?"
