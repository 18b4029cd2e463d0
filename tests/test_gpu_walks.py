"""GPU walk kernels (K1 reach, K2/K3 min-path) vs the CPU oracle, through
dyg_run_batch (the stateless twin of run_batch, walk.hpp:86-92).

Bit-exact: reached / best_estimate / steps_used / loop-erased path /
resistance must equal the oracle's for every query. Known answers re-express
proj/tests/test_walk.cpp (cited per test)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import bits, to_dyg

pytestmark = pytest.mark.gpu


def random_queries(rng, n, nq, minpath_every=3, w_lo=0.5, w_hi=1.5):
    q = np.zeros(nq, O.QUERY_DTYPE)
    for i in range(nq):
        p = int(rng.integers(n))
        t = int(rng.integers(n))
        if p == t:
            t = (t + 1) % n
        q[i] = (1 if (minpath_every and i % minpath_every == 0) else 0, p, t, 0,
                rng.uniform(w_lo, w_hi), i * 7 + 3)
    return q


def check_same(oout, opaths, dout, dpaths):
    assert np.array_equal(oout["reached"], dout["reached"])
    assert np.array_equal(oout["steps_used"], dout["steps_used"])
    assert np.array_equal(bits(oout["best_estimate"]), bits(dout["best_estimate"]))
    assert np.array_equal(oout["path_len"], dout["path_len"])
    assert np.array_equal(bits(oout["resistance"]), bits(dout["resistance"]))
    for i in range(len(oout)):
        L = int(oout["path_len"][i])
        assert np.array_equal(opaths[i, :L], dpaths[i, :L]), i


@pytest.mark.parametrize("s", [1, 4, 8, 16, 32, 3, 64])
@pytest.mark.parametrize("K", [20.0, 1e18])
def test_random_graph_batches(oracle, dyg, s, K):
    # test_walk.cpp:228-260 "batch execution matches sequential execution",
    # here GPU vs CPU, bitwise.
    g = oracle.make_random_connected(80, 120, 47)
    rng = np.random.default_rng(9)
    q = random_queries(rng, 80, 64)
    T = 100
    oout, opaths = oracle.run_batch(g, q, K, T, s, 3)
    dout, dpaths = dyg.run_batch(to_dyg(dyg, g), q, dyg.WalkConfig(K, T, s, 3))
    check_same(oout, opaths, dout, dpaths)


@pytest.mark.parametrize("T", [1, 5, 100, 300])
def test_step_caps(oracle, dyg, T):
    g = oracle.make_mesh(30, 30, 5)
    rng = np.random.default_rng(T)
    q = random_queries(rng, 900, 200, minpath_every=2)
    oout, opaths = oracle.run_batch(g, q, 50.0, T, 16, 11)
    dout, dpaths = dyg.run_batch(to_dyg(dyg, g), q, dyg.WalkConfig(50.0, T, 16, 11))
    check_same(oout, opaths, dout, dpaths)


def test_high_degree_rows_use_overflow_pool(oracle, dyg):
    # Rows longer than the 4 (H) / 10 (G) inline slab entries live in the
    # overflow pool; the sampler must walk them identically.
    g = oracle.make_random_connected(60, 900, 13)
    rng = np.random.default_rng(1)
    q = random_queries(rng, 60, 300)
    oout, opaths = oracle.run_batch(g, q, 8.0, 100, 16, 21)
    dout, dpaths = dyg.run_batch(to_dyg(dyg, g), q, dyg.WalkConfig(8.0, 100, 16, 21))
    check_same(oout, opaths, dout, dpaths)


def test_mesh_insertion_shape(oracle, dyg):
    # The C3 walk shape: reach queries on a mesh sparsifier.
    G = oracle.make_mesh(64, 64, 1)
    H = oracle.build_initial_sparsifier(G, 0.10, 1)
    rng = np.random.default_rng(3)
    q = random_queries(rng, 64 * 64, 2000, minpath_every=0)
    oout, opaths = oracle.run_batch(H, q, 100.0, 100, 16, 42)
    dout, dpaths = dyg.run_batch(to_dyg(dyg, H), q, dyg.WalkConfig(100.0, 100, 16, 42))
    check_same(oout, opaths, dout, dpaths)


def test_path_graph_known_answers(dyg):
    # test_walk.cpp:15-30: forced walk on a path reaches with R = 2.0; a
    # budget of 1.5 cuts it (BudgetExceeded, 2 steps, no reach).
    g = dyg.DynamicGraph(3)
    g.insert_edge(0, 1, 1.0)
    g.insert_edge(1, 2, 1.0)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (0, 0, 2, 0, 1.0, 0)
    out, _ = dyg.run_batch(g, q, dyg.WalkConfig(10.0, 10, 1, 1))
    assert out["reached"][0] == 1 and out["best_estimate"][0] == 2.0
    assert out["steps_used"][0] == 2
    out, _ = dyg.run_batch(g, q, dyg.WalkConfig(1.5, 10, 1, 1))
    assert out["reached"][0] == 0 and out["steps_used"][0] == 2
    out, _ = dyg.run_batch(g, q, dyg.WalkConfig(100.0, 1, 1, 1))  # step cap
    assert out["reached"][0] == 0 and out["steps_used"][0] == 1


def test_tree_paths_are_exact(dyg, oracle):
    # test_walk.cpp:65-78 / 179-194: on a path graph the min-path walk is the
    # tree path and its resistance the exact series sum.
    n = 20
    g = dyg.DynamicGraph(n)
    for v in range(n - 1):
        g.insert_edge(v, v + 1, 0.8)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (1, 2, 17, 0, 1.0, 0)
    out, paths = dyg.run_batch(g, q, dyg.WalkConfig(1e18, 100, 4, 19))
    assert out["reached"][0] == 1
    assert paths[0, : out["path_len"][0]].tolist() == list(range(2, 18))
    expect = 0.0
    for _ in range(15):
        expect += 1.0 / 0.8
    assert out["resistance"][0] == expect


def test_case_study_recovery_golden(dyg):
    # test_walk.cpp:213-226 (fixture support/case_study.hpp:16-40): delete
    # (16,17); 32 walkers, seed 2024, uid 0 recover {16,21,22,17}, R = 3.0.
    h_edges = [(25, 20), (20, 21), (21, 22), (22, 17), (17, 16), (16, 15), (15, 14), (14, 13),
               (13, 12), (12, 11), (11, 10), (10, 9), (22, 23), (23, 24), (17, 18), (18, 19),
               (19, 0), (0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 8), (8, 9)]
    g = dyg.DynamicGraph(26)
    for u, v in h_edges + [(24, 25), (16, 21), (3, 7)]:
        g.insert_edge(u, v, 1.0)
    g.delete_edge(16, 17)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (1, 16, 17, 0, 1.0, 0)
    out, paths = dyg.run_batch(g, q, dyg.WalkConfig(1e18, 100, 32, 2024))
    assert out["reached"][0] == 1
    assert paths[0, : out["path_len"][0]].tolist() == [16, 21, 22, 17]
    assert out["resistance"][0] == 3.0


def test_usage_errors(dyg):
    # walk.cpp:43-48: p == q and isolated starts are usage errors.
    g = dyg.DynamicGraph(4)
    g.insert_edge(0, 1, 1.0)
    q = np.zeros(1, O.QUERY_DTYPE)
    q[0] = (0, 1, 1, 0, 1.0, 0)
    with pytest.raises(dyg.Error) as e:
        dyg.run_batch(g, q, dyg.WalkConfig())
    assert e.value.kind == dyg.ErrorKind.Usage
    q[0] = (0, 3, 1, 0, 1.0, 0)
    with pytest.raises(dyg.Error) as e:
        dyg.run_batch(g, q, dyg.WalkConfig())
    assert "isolated" in str(e.value)
