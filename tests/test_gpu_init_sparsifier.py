"""the initial sparsifier builder on the device
(dyg_build_initial_sparsifier) must build H exactly as the reference's
build_initial_sparsifier (sparsifier.cpp:105-159): the same rows, in the same
order, with the same weight bits -- checked against the compiled reference
(or its restatement) and the host pipeline."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.parity import same_rows, to_dyg

pytestmark = pytest.mark.gpu


def _gpu_rows(dyg, g, target, seed):
    h = dyg.build_initial_sparsifier_gpu(to_dyg(dyg, g), target, seed)
    return h.rows()


@pytest.mark.parametrize("shape,target,seed", [
    ((10, 10, 1), 0.10, 1),
    ((100, 100, 1), 0.10, 1),
    ((37, 53, 7), 0.25, 3),
    ((64, 64, 2), 0.0, 5),     # tree only
    ((16, 16, 4), 10.0, 9),    # every off-tree edge
])
def test_device_builder_equals_reference_mesh(oracle, dyg, shape, target, seed):
    g = oracle.make_mesh(*shape)
    ref = oracle.build_initial_sparsifier(g, target, seed)
    assert same_rows(ref.export(), _gpu_rows(dyg, g, target, seed))


def test_device_builder_equals_reference_grid_and_ties(oracle, dyg):
    # grid4 (C4's generator) and a random connected graph with pendant
    # vertices; equal weights exercise the (u, v) tie order of the sort.
    for g in (oracle.make_grid4(40, 50, 3), oracle.make_random_connected(500, 900, 4, True)):
        for target, seed in ((0.1, 1), (0.3, 11)):
            ref = oracle.build_initial_sparsifier(g, target, seed)
            assert same_rows(ref.export(), _gpu_rows(dyg, g, target, seed))
    # Many equal weights: the (u, v) order decides the tree.
    rp, ids, w = oracle.make_mesh(30, 30, 2).export()
    g = oracle.graph(len(rp) - 1)
    for u in range(len(rp) - 1):
        for i in range(int(rp[u]), int(rp[u + 1])):
            if u < ids[i]:
                g.insert(u, int(ids[i]), float(np.round(w[i] * 2) / 2))
    ref = oracle.build_initial_sparsifier(g, 0.2, 3)
    assert same_rows(ref.export(), _gpu_rows(dyg, g, 0.2, 3))


def test_device_builder_c3_matches_host_pipeline(dyg):
    g = dyg.make_mesh(512, 512, 1)
    host = dyg.build_initial_sparsifier(g, 0.10, 1)
    dev = dyg.build_initial_sparsifier_gpu(g, 0.10, 1)
    assert same_rows(host.rows(), dev.rows())


def test_device_builder_errors(dyg):
    g = dyg.make_mesh(8, 8, 1)
    with pytest.raises(dyg.Error) as e:
        dyg.build_initial_sparsifier_gpu(g, -0.1, 1)
    assert e.value.kind == dyg.ErrorKind.Usage
    two = dyg.DynamicGraph.from_rows(np.array([0, 1, 2, 3, 4], np.uint64),
                                     np.array([1, 0, 3, 2], np.uint32),
                                     np.array([1.0, 1.0, 2.0, 2.0]))
    with pytest.raises(dyg.Error) as e:
        dyg.build_initial_sparsifier_gpu(two, 0.1, 1)
    assert e.value.kind == dyg.ErrorKind.Data
    assert str(e.value) == "graph must be connected to build a sparsifier"
