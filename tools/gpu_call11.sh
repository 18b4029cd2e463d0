mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream_gen.py -m gpu -q > gpurun_out/pytest_gpu_r2k_gen.log 2>&1; echo "pytest gen exit $?"; tail -n 2 gpurun_out/pytest_gpu_r2k_gen.log
timeout 900 python -c "
import time, sys; sys.path.insert(0,'.')
import paper_2505_02741_b200 as D
g = D.make_mesh(2048, 2048, 1); o = D.StreamGenOptions(0.25, 0.01, 10, 7, 0)
for f in (D.generate_update_stream_gpu, D.generate_update_stream, D.generate_update_stream_gpu):
    t = time.perf_counter(); s = f(g, o); print(f.__name__, len(s.events), round(time.perf_counter() - t, 3), 's', flush=True)
"
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_l2_base_$i.json 2>/dev/null; echo "base $?"
DYG_GRAPH_DEBUG=1 DYG_L2_PERSIST_MB=40 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_l2_p40_$i.json 2>gpurun_out/ab_l2_p40.err; echo "p40 $?"; grep "L2 window" gpurun_out/ab_l2_p40.err | head -1
DYG_L2_PERSIST_MB=80 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_l2_p80_$i.json 2>/dev/null; echo "p80 $?"
done
python tools/ab_table.py gpurun_out/ab_l2_*.json
