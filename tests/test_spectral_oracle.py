"""CPU: the spectral restatement (oracle/spectral_ref.py) against ground
truth -- dense generalized eigenvalues and exact grounded solves -- and the
host random_rhs of libdyg (no GPU needed). The reference's own spectral code
needs Eigen, which is absent, so this is how the checker is pinned."""
import numpy as np
import pytest
import scipy.linalg as sla

import paper_2505_02741_b200 as D
from oracle import spectral_ref as S


def rows(g):
    rp, ids, w = g.rows()
    return np.asarray(rp), np.asarray(ids), np.asarray(w)


@pytest.fixture(scope="module")
def mesh():
    g = D.make_mesh(12, 11, 1)
    h = D.build_initial_sparsifier(g, 0.10, 1)
    return rows(g), rows(h)


def test_dense_matches_grounded_pencil(mesh):
    g, h = mesh
    lg, lh = S.laplacian(*g), S.laplacian(*h)
    d = S.condition_dense(lg, lh)
    # the grounded pencil has the same generalized eigenvalues (the Rayleigh
    # quotient is invariant under adding constants)
    ev = sla.eigh(lg.toarray()[1:, 1:], lh.toarray()[1:, 1:], eigvals_only=True)
    assert d["lambda_min"] == pytest.approx(ev[0], rel=1e-10)
    assert d["lambda_max"] == pytest.approx(ev[-1], rel=1e-10)
    assert d["lambda_min"] >= 1.0 - 1e-9  # H is a subgraph of G: L_G >= L_H


def test_lanczos_converges_to_dense(mesh):
    g, h = mesh
    lg, lh = S.laplacian(*g), S.laplacian(*h)
    d = S.condition_dense(lg, lh)
    it = S.condition_iterative(lg, lh, tolerance=1e-10, max_iterations=400)
    assert it["kappa"] == pytest.approx(d["kappa"], rel=1e-6)


def test_pcg_solves_the_grounded_system(mesh):
    g, h = mesh
    lg, lh = S.laplacian(*g), S.laplacian(*h)
    n = lg.shape[0]
    b = S.random_rhs(n, 3)
    x_true = S.GroundedSolver(lg).solve(b)
    for m in (S.Preconditioner(None, n), S.Preconditioner(lh), S.Preconditioner(lh, factor_cap=0)):
        x, it, rel, ok, energy = S.pcg_solve(lg, b, m, 1e-10)
        assert ok and rel <= 1e-10
        assert np.allclose(x, x_true, rtol=0, atol=1e-7 * np.abs(x_true).max())
        assert all(e2 <= e1 + 1e-10 * abs(e1) for e1, e2 in zip(energy, energy[1:]))


def test_random_rhs_host_abi_matches_restatement():
    for n, seed in ((1, 0), (7, 3), (1000, 0xB0C4)):
        a = D.random_rhs(n, seed)
        b = S.random_rhs(n, seed)
        # same SplitMix64 stream and libm; only the centring sum order differs
        assert np.allclose(a, b, rtol=0, atol=1e-14)
        assert abs(a.sum()) < 1e-10


def test_calibrate_budget_restatement_bounds(mesh):
    g, h = mesh
    k = S.calibrate_budget(g, h, 0.05, 1.0, 7)
    d = S.condition_dense(S.laplacian(*g), S.laplacian(*h))
    assert k == pytest.approx(d["kappa"], rel=1e-9)  # n <= dense_cap: the dense path
    assert S.calibrate_budget(g, h, 0.05, 1e-12, 7) == 1.0  # clamp(., 1, 1e6)
