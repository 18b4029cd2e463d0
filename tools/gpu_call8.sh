mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_spectral_kat.py -m gpu -q > gpurun_out/pytest_gpu_r2h_spec.log 2>&1; echo "pytest spectral exit $?"; tail -n 3 gpurun_out/pytest_gpu_r2h_spec.log
echo "== nd"; timeout 900 python tools/spectral_bench.py 512 2>&1 | tail -2
NOCPU=1 timeout 900 python tools/spectral_bench.py 1024 2>&1 | tail -2
echo "== metis"; DYG_ORDERING=metis NOCPU=1 timeout 900 python tools/spectral_bench.py 512 1024 2>&1 | tail -4
echo "== nd debug 512"; DYG_SPECTRAL_DEBUG=1 NOCPU=1 timeout 900 python tools/spectral_bench.py 512 2>&1 | grep -E "chol|kappa" | head -20
timeout 600 python bench.py --force-shard --no-cpu-baseline > gpurun_out/bench_r2h_shard_peer.json 2> /dev/null; echo "bench shard $?"
python tools/ab_table.py gpurun_out/bench_r2h_shard_peer.json
