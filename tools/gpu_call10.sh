mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream_gen.py -m gpu -q > gpurun_out/pytest_gpu_r2j_gen.log 2>&1; echo "pytest gen exit $?"; tail -n 15 gpurun_out/pytest_gpu_r2j_gen.log
timeout 900 python -c "
import time, sys; sys.path.insert(0,'.')
import paper_2505_02741_b200 as D
g = D.make_mesh(2048, 2048, 1); o = D.StreamGenOptions(0.25, 0.01, 10, 7, 0)
for f in (D.generate_update_stream_gpu, D.generate_update_stream, D.generate_update_stream_gpu):
    t = time.perf_counter(); s = f(g, o); print(f.__name__, len(s.events), round(time.perf_counter() - t, 3), 's', flush=True)
"
timeout 900 python bench.py > gpurun_out/bench_r2j_c5.json 2> gpurun_out/bench_r2j_c5.err; echo "bench $?"; tail -n 2 gpurun_out/bench_r2j_c5.err
python tools/ab_table.py gpurun_out/bench_r2j_c5.json
