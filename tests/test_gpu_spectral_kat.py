"""The reference's own spectral known answers, re-expressed against the device
(proj/tests/test_spectral.cpp:160-232; the doctest suite itself cannot be
built here: doctest and Eigen are absent). Inputs come from the product's
generators, which equal the reference's (tests/test_host.py): the same
random_connected graphs, the same build_initial_sparsifier, the same seeds.

  * kappa(G, G) = 1 to 1e-8                              (:161-165)
  * triangle vs its spanning tree: kappa 3, lambda_min 1  (:166-175)
  * kappa >= 1 - 1e-9 on initial sparsifiers             (:176-183)
  * a disconnected sparsifier is a Data error            (:184-189)
  * dense vs iterative pencils within 1e-4, seeds 1..25  (:192-213)
  * pendant graphs pin lambda_min at 1 (1e-6), and the
    resistance ratio R_H / R_G <= lambda_max             (:215-232)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def triangle(D):
    g = D.DynamicGraph(3)
    for u, v in ((0, 1), (1, 2), (2, 0)):  # make_cycle(3, 1.0)
        g.insert_edge(u, v, 1.0)
    return g


def resistances(D, g):
    """All-pairs effective resistance from the dense pseudo-inverse (test side)."""
    rp, ids, w = g.rows()
    n = len(rp) - 1
    L = np.zeros((n, n))
    for u in range(n):
        for i in range(rp[u], rp[u + 1]):
            L[u, ids[i]] -= w[i]
            L[u, u] += w[i]
    P = np.linalg.pinv(L)
    d = np.diag(P)
    return d[:, None] + d[None, :] - 2 * P


def test_identical_graphs(dyg):
    g = dyg.make_random_connected(40, 60, 33)
    est = dyg.condition_number(g, g)
    assert est.kappa == pytest.approx(1.0, rel=1e-8)


def test_triangle_against_its_spanning_tree(dyg):
    h = dyg.DynamicGraph(3)
    h.insert_edge(0, 1, 1.0)
    h.insert_edge(1, 2, 1.0)
    est = dyg.condition_number(triangle(dyg), h)
    assert est.kappa == pytest.approx(3.0, rel=1e-9)
    assert est.lambda_min == pytest.approx(1.0, rel=1e-9)


@pytest.mark.parametrize("seed", range(50, 56))
def test_kappa_at_least_one(dyg, seed):
    g = dyg.make_random_connected(30, 45, seed)
    h = dyg.build_initial_sparsifier(g, 0.05, seed)
    assert dyg.condition_number(g, h).kappa >= 1.0 - 1e-9


def test_disconnected_sparsifier_is_a_data_error(dyg):
    h = dyg.DynamicGraph(3)
    h.insert_edge(0, 1, 1.0)
    with pytest.raises(dyg.Error) as e:
        dyg.condition_number(triangle(dyg), h)
    assert e.value.kind == dyg.ErrorKind.Data


def test_dense_and_iterative_pencils_agree(dyg):
    compared = 0
    for seed in range(1, 26):
        n = 40 + 6 * seed
        g = dyg.make_random_connected(n, n, seed, 0.2, 5.0)
        h = dyg.build_initial_sparsifier(g, 0.04, seed)
        a = dyg.condition_number(g, h, dyg.ConditionOptions(method=dyg.ConditionMethod.Dense))
        b = dyg.condition_number(g, h, dyg.ConditionOptions(
            method=dyg.ConditionMethod.Iterative, tolerance=1e-9, max_iterations=2 * n))
        assert abs(a.kappa - b.kappa) <= 1e-4 * a.kappa, (seed, a, b)
        assert abs(a.lambda_max - b.lambda_max) <= 1e-4 * a.lambda_max, (seed, a, b)
        assert abs(a.lambda_min - b.lambda_min) <= 1e-4 * abs(a.lambda_min), (seed, a, b)
        compared += 1
    assert compared == 25


@pytest.mark.parametrize("seed", range(60, 70))
def test_pencil_bound_chain_on_pendant_graphs(dyg, seed):
    g = dyg.make_random_connected(24, 30, seed, 0.1, 10.0, True)
    h = dyg.build_initial_sparsifier(g, 0.05, seed)
    est = dyg.condition_number(g, h)
    assert est.lambda_min == pytest.approx(1.0, rel=1e-6)
    rg, rh = resistances(dyg, g), resistances(dyg, h)
    iu = np.triu_indices(24, 1)
    assert (rh[iu] / rg[iu]).max() <= est.lambda_max * (1.0 + 1e-6)


def test_calibrate_budget_default_rho_is_the_reference_default(dyg):
    """calibrate_budget's rho defaults to 0.1 (sparsifier.hpp:118-120)."""
    g = dyg.make_random_connected(200, 260, 5)
    h = dyg.build_initial_sparsifier(g, 0.05, 5)
    assert dyg.calibrate_budget(g, h, 0.05) == dyg.calibrate_budget(g, h, 0.05, 0.1, 0)
