"""generate_update_stream with the insertion sampling on the device
(dyg_generate_stream, csrc/stream_gen.cu) against the compiled reference
(stream.cpp:114-200): every event (kind, endpoints, weight bits, batch
index) identical, for sparse meshes (almost no rejected attempts), small
dense graphs (many self-loop / edge / repeat rejections: many speculative
rounds and pair-set rebuilds), the reference's errors, and the C4 shape at
full size against the host pipeline."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def same_events(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return len(a) == len(b) and all(np.array_equal(a[f], b[f]) for f in ("kind", "u", "v", "batch_index")) \
        and np.array_equal(a["weight"].view(np.uint64), b["weight"].view(np.uint64))


CASES = [
    ("mesh", 40, 50, 0.25, 0.05, 10, 7),
    ("mesh", 100, 110, 0.25, 0.01, 10, 7),   # C2 shape, locality 0
    ("grid4", 60, 60, 0.5, 0.0, 10, 3),
    ("mesh", 6, 6, 4.0, 0.2, 7, 11),          # dense: ~50% of attempts rejected
    ("mesh", 5, 5, 6.0, 0.0, 3, 5),           # near saturation
    ("grid4", 30, 30, 0.0, 0.3, 4, 2),        # deletions only
]


@pytest.mark.parametrize("kind,rows,cols,ins,dele,batches,seed", CASES)
def test_device_generator_equals_reference(oracle, dyg, kind, rows, cols, ins, dele, batches, seed):
    og = oracle.make_mesh(rows, cols, 1) if kind == "mesh" else oracle.make_grid4(rows, cols, 1)
    ref = oracle.generate_stream(og, ins, dele, batches, seed, 0)
    g = dyg.DynamicGraph.from_rows(*og.export())
    got = dyg.generate_update_stream_gpu(g, dyg.StreamGenOptions(ins, dele, batches, seed, 0))
    assert got.batch_count == ref.batch_count
    assert same_events(got.events, ref.events())


def test_device_generator_errors_match_reference(oracle, dyg):
    og = oracle.make_mesh(4, 4, 1)  # 16 vertices, 33 edges: 87 non-edges
    g = dyg.DynamicGraph.from_rows(*og.export())
    with pytest.raises(O.OracleError) as r:
        oracle.generate_stream(og, 8.0, 0.0, 2, 1, 0)  # 128 insertions > 87 non-edges
    with pytest.raises(dyg.Error) as e:
        dyg.generate_update_stream_gpu(g, dyg.StreamGenOptions(8.0, 0.0, 2, 1, 0))
    assert int(e.value.kind) == r.value.kind and str(e.value) == r.value.message
    with pytest.raises(dyg.Error) as e:
        dyg.generate_update_stream_gpu(g, dyg.StreamGenOptions(0.1, 0.0, 0, 1, 0))
    assert e.value.kind == dyg.ErrorKind.Usage and str(e.value) == "batch count must be positive"


def test_device_generator_c4_equals_host_pipeline(dyg):
    g = dyg.make_grid4(1225, 1225, 1)
    o = dyg.StreamGenOptions(0.25, 0.0, 10, 7, 0)
    host = dyg.generate_update_stream(g, o)
    dev = dyg.generate_update_stream_gpu(g, o)
    assert dev.batch_count == host.batch_count == 10
    assert same_events(dev.events, host.events)
