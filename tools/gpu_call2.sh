mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2b.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu_r2b.log
timeout 600 python bench.py > gpurun_out/bench_r2b_c5.json 2>gpurun_out/bench_r2b_c5.err; echo "bench $?"
SAN_TIMEOUT=1500 bash tools/sanitize.sh memcheck racecheck synccheck initcheck
