"""Host-side pipeline of libdyg.so (CPU only): the reference's file formats,
DynamicGraph mutation semantics and the deterministic benchmark-input
generators must reproduce the reference exactly -- including per-row order,
which every later walk depends on (SURVEY.md findings 3 and 5)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import bits, first_row_diff, same_rows


@pytest.fixture(scope="module")
def ref(oracle):
    return oracle


def test_mesh_and_sparsifier_match(ref, dyg):
    for rows, cols, seed in [(100, 100, 1), (100, 110, 1), (37, 23, 5)]:
        g1, g2 = ref.make_mesh(rows, cols, seed), dyg.make_mesh(rows, cols, seed)
        assert same_rows(g1.export(), g2.rows()), first_row_diff(g1.export(), g2.rows())
        h1 = ref.build_initial_sparsifier(g1, 0.10, seed)
        h2 = dyg.build_initial_sparsifier(g2, 0.10, seed)
        assert same_rows(h1.export(), h2.rows())


def test_grid4_and_random_graphs_match(ref, dyg):
    assert same_rows(ref.make_grid4(40, 33, 1).export(), dyg.make_grid4(40, 33, 1).rows())
    for pend in (False, True):
        a = ref.make_random_connected(300, 500, 9, 0.1, 10.0, pend)
        b = dyg.make_random_connected(300, 500, 9, 0.1, 10.0, pend)
        assert same_rows(a.export(), b.rows())


@pytest.mark.parametrize("loc,ins,dele,batches", [(0, 0.25, 0.01, 10), (3, 0.25, 0.01, 10),
                                                  (2, 0.5, 0.2, 3), (0, 0.0, 0.3, 4)])
def test_stream_generator_matches(ref, dyg, loc, ins, dele, batches):
    g1, g2 = ref.make_mesh(30, 31, 2), dyg.make_mesh(30, 31, 2)
    s1 = ref.generate_stream(g1, ins, dele, batches, 7, loc)
    s2 = dyg.generate_update_stream(g2, dyg.StreamGenOptions(ins, dele, batches, 7, loc))
    assert np.array_equal(bits(s1.events()), bits(s2.events))
    assert s1.batch_count == s2.batch_count


def test_generator_errors(dyg):
    g = dyg.make_mesh(3, 3, 1)
    with pytest.raises(dyg.Error) as e:
        dyg.generate_update_stream(g, dyg.StreamGenOptions(0.1, 0.0, 0, 1, 0))
    assert e.value.kind == dyg.ErrorKind.Usage
    with pytest.raises(dyg.Error) as e:
        dyg.generate_update_stream(g, dyg.StreamGenOptions(-1.0, 0.0, 1, 1, 0))
    assert e.value.kind == dyg.ErrorKind.Usage
    disconnected = dyg.DynamicGraph(4)
    disconnected.insert_edge(0, 1, 1.0)
    with pytest.raises(dyg.Error) as e:
        dyg.build_initial_sparsifier(disconnected, 0.1, 1)
    assert e.value.kind == dyg.ErrorKind.Data


def test_graph_mutation_fuzz_matches(ref, dyg):
    # test_graph.cpp:203-219-style random mutations; rows (order included)
    # must track the reference after every operation batch.
    rng = np.random.default_rng(4)
    a, b = ref.graph(50), dyg.DynamicGraph(50)
    for step in range(3000):
        u, v = int(rng.integers(50)), int(rng.integers(50))
        if u == v:
            continue
        if rng.random() < 0.6:
            w = float(rng.uniform(0.1, 2.0))
            a.insert(u, v, w)
            b.insert_edge(u, v, w)
        else:
            ea = eb = None
            try:
                a.delete(u, v)
            except O.OracleError as x:
                ea = x
            try:
                b.delete_edge(u, v)
            except dyg.Error as x:
                eb = x
            assert (ea is None) == (eb is None)
            if ea is not None:
                assert str(eb) == ea.message and int(eb.kind) == ea.kind
        if step % 500 == 0:
            assert same_rows(a.export(), b.rows())
    assert same_rows(a.export(), b.rows())
    assert a.edge_count == b.edge_count()


def test_graph_usage_errors(dyg):
    g = dyg.DynamicGraph(3)
    for args, kind in [((0, 0, 1.0), dyg.ErrorKind.Usage), ((0, 5, 1.0), dyg.ErrorKind.Usage),
                       ((0, 1, -1.0), dyg.ErrorKind.Usage), ((0, 1, float("inf")), dyg.ErrorKind.Usage)]:
        with pytest.raises(dyg.Error) as e:
            g.insert_edge(*args)
        assert e.value.kind == kind
    with pytest.raises(dyg.Error) as e:
        dyg.DynamicGraph(0)
    assert e.value.kind == dyg.ErrorKind.Usage


MM_CASES = {
    "symmetric_real": "%%MatrixMarket matrix coordinate real symmetric\n% c\n5 5 7\n1 1 4.0\n2 1 -1.5\n"
                      "3 2 2.25\n4 3 -0.5\n5 4 1\n5 1 3\n3 1 0.75\n",
    "general_dupes": "%%MatrixMarket matrix coordinate real general\n4 4 8\n1 2 1.0\n2 1 1.0\n"
                     "3 4 2.0\n4 3 -2.0\n2 3 0.5\n2 3 0.25\n1 4 1e-3\n4 4 9\n",
    "integer": "%%MatrixMarket matrix coordinate integer symmetric\n6 6 6\n2 1 3\n3 2 -4\n6 5 7\n"
               "5 4 1\n4 3 2\n6 1 5\n",
    "rect_header": "%%MatrixMarket matrix coordinate real general\n3 5 2\n1 5 2.0\n3 4 1.0\n",
}
MM_BAD = {
    "banner": "%%MatrixMarket matrix array real general\n2 2 1\n1 2 1\n",
    "field": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 2 1 0\n",
    "count": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 1\n",
    "range": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 4 1\n",
    "zero": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 2 0\n2 3 1\n",
    "malformed": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 x 1\n",
    "empty": "",
}


@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_matrix_market_load_matches_reference_order(tmp_path, reference, dyg, case):
    p = tmp_path / f"{case}.mtx"
    p.write_text(MM_CASES[case])
    a = reference.load_matrix_market(str(p))
    b = dyg.load_matrix_market(str(p))
    assert same_rows(a.export(), b.rows())
    # save: sorted lower triangle, %.17g -- byte-identical files
    pa, pb = tmp_path / "a.mtx", tmp_path / "b.mtx"
    a.save_matrix_market(str(pa))
    dyg.save_matrix_market(b, str(pb))
    assert pa.read_bytes() == pb.read_bytes()


@pytest.mark.parametrize("case", sorted(MM_BAD))
def test_matrix_market_errors_match(tmp_path, reference, dyg, case):
    p = tmp_path / f"{case}.mtx"
    p.write_text(MM_BAD[case])
    with pytest.raises(O.OracleError) as ea:
        reference.load_matrix_market(str(p))
    with pytest.raises(dyg.Error) as eb:
        dyg.load_matrix_market(str(p))
    assert str(eb.value) == ea.value.message and int(eb.value.kind) == ea.value.kind


def test_matrix_market_large_order(tmp_path, reference, dyg):
    # unordered_map iteration order at a realistic size fixes the rows.
    g = reference.make_mesh(60, 70, 3)
    p = tmp_path / "mesh.mtx"
    g.save_matrix_market(str(p))
    a = reference.load_matrix_market(str(p))
    b = dyg.load_matrix_market(str(p))
    assert same_rows(a.export(), b.rows())


def test_stream_file_roundtrip_matches(tmp_path, reference, dyg):
    g = reference.make_mesh(20, 20, 1)
    s = reference.generate_stream(g, 0.3, 0.05, 3, 5, 2)
    pa, pb = tmp_path / "a.txt", tmp_path / "b.txt"
    s.save(str(pa))
    ds = dyg.UpdateStream(s.events(), s.batch_count)
    dyg.save_update_stream(ds, str(pb))
    assert pa.read_bytes() == pb.read_bytes()
    back = dyg.load_update_stream(str(pa))
    ref_back = reference.load_stream(str(pa))
    assert np.array_equal(bits(back.events), bits(ref_back.events()))
    assert back.batch_count == ref_back.batch_count


@pytest.mark.parametrize("text", ["i 1 2\n", "d 1\n", "x 1 2\n", "i 1 2 3\n#batch\n\n# c\nd 4 5\n",
                                  "#batch\n#batch\n", "i 1 2 0.5\n#batch\n#batch\nd 2 3\n"])
def test_stream_parse_matches(tmp_path, reference, dyg, text):
    p = tmp_path / "s.txt"
    p.write_text(text)
    ea = eb = None
    try:
        ra = reference.load_stream(str(p))
    except O.OracleError as x:
        ea = x
    try:
        rb = dyg.load_update_stream(str(p))
    except dyg.Error as x:
        eb = x
    assert (ea is None) == (eb is None)
    if ea is None:
        assert np.array_equal(bits(ra.events()), bits(rb.events))
        assert ra.batch_count == rb.batch_count
    else:
        assert str(eb) == ea.message.replace(str(p), str(p))


def test_no_gpu_fails_loudly(dyg):
    if dyg.device_count() > 0:
        pytest.skip("a GPU is visible")
    g = dyg.make_mesh(4, 4, 1)
    h = dyg.build_initial_sparsifier(g, 0.1, 1)
    with pytest.raises(dyg.Error) as e:
        dyg.SparsifierState(g, h, dyg.SparsifierOptions(batched=True))
    assert e.value.kind == dyg.ErrorKind.Device
