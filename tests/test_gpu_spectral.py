"""GPU: condition number, calibrate_budget and PCG of csrc/spectral.cu
against the restatement (oracle/spectral_ref.py) and dense ground truth.
Floating-point tolerances (the device sums in a different order and solves
L_H with the same exact grounded factorisation but its own sparse Cholesky):
  kappa (dense path)            rel 1e-9
  kappa (iterative, converged)  rel 1e-6 of the dense truth
  calibrate_budget (coarse)     rel 1e-2 of the restatement
  PCG solution                  1e-6 of the exact grounded solve (max-norm)."""
import numpy as np
import pytest

import paper_2505_02741_b200 as D
from oracle import spectral_ref as S

pytestmark = pytest.mark.gpu


def rows(g):
    rp, ids, w = g.rows()
    return np.asarray(rp), np.asarray(ids), np.asarray(w)


@pytest.fixture(scope="module")
def mesh():
    g = D.make_mesh(24, 20, 1)
    h = D.build_initial_sparsifier(g, 0.10, 1)
    return g, h


def test_condition_dense(mesh):
    g, h = mesh
    e = D.condition_number(g, h)  # Auto: n = 480 <= dense_cap
    d = S.condition_dense(S.laplacian(*rows(g)), S.laplacian(*rows(h)))
    assert e.method == "Dense" and e.converged
    assert e.kappa == pytest.approx(d["kappa"], rel=1e-9)
    assert e.lambda_min == pytest.approx(d["lambda_min"], rel=1e-9)


def test_condition_iterative(mesh):
    g, h = mesh
    o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-9)
    e = D.condition_number(g, h, o)
    d = S.condition_dense(S.laplacian(*rows(g)), S.laplacian(*rows(h)))
    it = S.condition_iterative(S.laplacian(*rows(g)), S.laplacian(*rows(h)), 1e-9, 400)
    assert e.method == "Iterative" and e.converged
    assert e.kappa == pytest.approx(d["kappa"], rel=1e-6)
    assert e.lambda_max == pytest.approx(it["lambda_max"], rel=1e-6)
    assert abs(e.iterations_used - it["iterations"]) <= 3


def test_condition_iterative_larger():
    g = D.make_mesh(64, 64, 1)
    h = D.build_initial_sparsifier(g, 0.10, 1)
    o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-8)
    e = D.condition_number(g, h, o)
    ref = S.condition_iterative(S.laplacian(*rows(g)), S.laplacian(*rows(h)), 1e-8, 400)
    assert e.converged
    assert e.kappa == pytest.approx(ref["kappa"], rel=1e-5)


def test_calibrate_budget(mesh):
    g, h = mesh
    k = D.calibrate_budget(g, h, 0.05, 2.0, 11)
    ref = S.calibrate_budget(rows(g), rows(h), 0.05, 2.0, 11)
    assert k == pytest.approx(ref, rel=1e-9)  # dense path at this size
    g2 = D.make_mesh(90, 80, 1)  # n = 7200 > dense_cap: the coarse Lanczos
    h2 = D.build_initial_sparsifier(g2, 0.10, 1)
    k2 = D.calibrate_budget(g2, h2, 0.01, 1.0, 5)
    ref2 = S.calibrate_budget(rows(g2), rows(h2), 0.01, 1.0, 5)
    assert k2 == pytest.approx(ref2, rel=1e-2)


def test_session_calibrate_budget(mesh):
    g, h = mesh
    st = D.SparsifierState(g, h, D.SparsifierOptions(D.WalkConfig(10.0, 100, 16, 42), True, False))
    assert D.calibrate_budget(st, probe_fraction=0.05, rho=1.5) == pytest.approx(
        D.calibrate_budget(g, h, 0.05, 1.5, 42), rel=1e-12)
    assert D.condition_number(st).kappa == pytest.approx(D.condition_number(g, h).kappa, rel=1e-12)


@pytest.mark.parametrize("precond", ["identity", "H", "H-innercg"])
def test_pcg(mesh, precond):
    g, h = mesh
    n = g.vertex_count()
    b = D.random_rhs(n, 3)
    lg = S.laplacian(*rows(g))
    x_true = S.GroundedSolver(lg).solve(b)
    m = None if precond == "identity" else h
    cap = 1 if precond == "H-innercg" else 2_000_000
    r = D.pcg_solve(g, b, m, tolerance=1e-10, factor_cap=cap, energy_trace=True)
    assert r.converged and r.relative_residual <= 1e-10
    assert np.abs(r.solution - x_true).max() <= 1e-6 * np.abs(x_true).max()
    pm = S.Preconditioner(None, n) if m is None else S.Preconditioner(S.laplacian(*rows(h)),
                                                                      factor_cap=cap)
    _, it, _, _, energy = S.pcg_solve(lg, b, pm, 1e-10)
    assert abs(r.iterations - it) <= max(3, it // 20)  # inexact L_H solves
    e = r.energy_trace
    assert len(e) == r.iterations
    assert np.all(e[1:] <= e[:-1] + 1e-10 * np.abs(e[:-1]))
    if precond != "identity":
        assert r.iterations < S.pcg_solve(lg, b, S.Preconditioner(None, n), 1e-10)[1]


def test_errors(mesh):
    g, h = mesh
    with pytest.raises(D.Error) as ei:
        D.condition_number(g, D.make_mesh(3, 3, 1))
    assert ei.value.kind == D.ErrorKind.Usage
    disc = D.DynamicGraph(g.vertex_count())
    disc.insert_edge(0, 1, 1.0)
    with pytest.raises(D.Error) as ei:
        D.condition_number(g, disc)
    assert ei.value.kind == D.ErrorKind.Data
    with pytest.raises(D.Error) as ei:
        D.condition_number(g, h, D.ConditionOptions(method=D.ConditionMethod.Dense, dense_cap=10))
    assert ei.value.kind == D.ErrorKind.Usage
    with pytest.raises(D.Error) as ei:
        D.calibrate_budget(g, h, 0.0, 1.0, 1)
    assert ei.value.kind == D.ErrorKind.Usage
    with pytest.raises(D.Error) as ei:
        D.pcg_solve(g, np.ones(g.vertex_count()), disc)
    assert ei.value.kind == D.ErrorKind.Data
    r = D.pcg_solve(g, np.ones(g.vertex_count()))  # zero after centring
    assert r.converged and r.iterations == 0 and not r.solution.any()


def test_session_spectral_after_updates(mesh):
    """The session overloads read the CURRENT graph and sparsifier (after a
    replay), not the ones the session was created with."""
    g, h = mesh
    st = D.SparsifierState(g, h, D.SparsifierOptions(D.WalkConfig(10.0, 100, 16, 42), True, False))
    s = D.generate_update_stream(g, D.StreamGenOptions(0.2, 0.05, 2, 9, 0))
    st.replay(s)
    g2, h2 = st.graph(), st.sparsifier()
    e_state = D.condition_number(st)
    e_rows = D.condition_number(g2, h2)
    assert e_state.kappa == pytest.approx(e_rows.kappa, rel=1e-12)
    d = S.condition_dense(S.laplacian(*rows(g2)), S.laplacian(*rows(h2)))
    assert e_state.kappa == pytest.approx(d["kappa"], rel=1e-9)
    assert D.calibrate_budget(st, probe_fraction=0.05, rho=1.0) == pytest.approx(
        min(max(d["kappa"], 1.0), 1e6), rel=1e-9)


def test_ordering_reused_for_same_and_nearby_patterns():
    """kappa twice on one H reuses the ordering (exact pattern); after a
    small edit of H (one added edge) the cached ordering is reused as a near
    pattern; the results match fresh-ordering results to solver precision."""
    from paper_2505_02741_b200.spectral import ordering_cache_stats

    g = D.make_mesh(48, 40, 3)
    h = D.build_initial_sparsifier(g, 0.10, 3)
    o = D.ConditionOptions(method=D.ConditionMethod.Iterative, tolerance=1e-9)
    s0 = ordering_cache_stats()
    e1 = D.condition_number(g, h, o)
    s1 = ordering_cache_stats()
    assert s1["misses"] == s0["misses"] + 1
    e2 = D.condition_number(g, h, o)
    s2 = ordering_cache_stats()
    assert s2["hits"] == s1["hits"] + 1 and s2["misses"] == s1["misses"]
    assert e2.kappa == e1.kappa  # the same ordering: the same factorisation
    # One more edge of G in H: a near pattern.
    rp, ids, w = (np.asarray(x) for x in h.rows())
    grp, gids, gw = (np.asarray(x) for x in g.rows())
    have = {(u, int(v)) for u in range(len(rp) - 1) for v in ids[rp[u]:rp[u + 1]]}
    # (both ends != 0: the grounded pattern drops vertex 0's row and column)
    u = next(u for u in range(1, len(grp) - 1)
             if any((u, int(v)) not in have and v != 0 for v in gids[grp[u]:grp[u + 1]]))
    k = next(i for i in range(grp[u], grp[u + 1]) if (u, int(gids[i])) not in have and gids[i] != 0)
    h.insert_edge(u, int(gids[k]), float(gw[k]))
    e3 = D.condition_number(g, h, o)
    s3 = ordering_cache_stats()
    assert s3["near_hits"] == s2["near_hits"] + 1 and s3["misses"] == s2["misses"]
    ref = S.condition_iterative(S.laplacian(*rows(g)), S.laplacian(*rows(h)), 1e-9, 400)
    assert e3.kappa == pytest.approx(ref["kappa"], rel=1e-6)
