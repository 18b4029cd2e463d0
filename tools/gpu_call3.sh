mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2c.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu_r2c.log
SAN_TIMEOUT=900 bash tools/sanitize.sh memcheck initcheck
timeout 600 python tools/relabel_probe.py --order morton > gpurun_out/relabel_morton.json 2>gpurun_out/relabel.err; echo "relabel $?"; cat gpurun_out/relabel_morton.json
timeout 600 python tools/relabel_probe.py --order hilbert > gpurun_out/relabel_hilbert.json 2>>gpurun_out/relabel.err; echo "relabel $?"; cat gpurun_out/relabel_hilbert.json
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2c_c5.json 2> gpurun_out/bench_r2c_c5.err; echo "bench c5 exit $?"
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2c_shard.json 2> gpurun_out/bench_r2c_shard.err; echo "bench shard exit $?"
