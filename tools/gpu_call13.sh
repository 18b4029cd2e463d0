mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2m.log 2>&1; echo "pytest exit $?"; tail -n 3 gpurun_out/pytest_gpu_r2m.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
timeout 900 python bench.py > gpurun_out/bench_r2m_c5.json 2> gpurun_out/bench_r2m_c5.err; echo "bench c5 $?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_r2m_ref.json 2> gpurun_out/bench_r2m_ref.err; echo "bench ref $?"; cat gpurun_out/bench_r2m_ref.json | head -c 600; echo
python tools/ab_table.py gpurun_out/bench_r2m_c5.json
