"""TEST INFRASTRUCTURE ONLY -- numpy/scipy restatement of the reference's
spectral evaluation, the checker for
paper_2505_02741_b200.spectral. Only tests/ may import it.

Follows, line by line where the arithmetic matters:
  laplacian, grounded_laplacian, GroundedLaplacianSolver  laplacian.cpp:7-85
  condition_number_dense                                 spectral.cpp:105-130
  tridiagonal_extremes                                   spectral.cpp:132-145
  condition_number_iterative                             spectral.cpp:147-276
  condition_number                                       spectral.cpp:278-303
  Preconditioner (Factorized / InnerCg / Identity)      solver.cpp:10-69
  pcg_solve                                              solver.cpp:71-144
  random_rhs                                             solver.cpp:146-159
  calibrate_budget                                       sparsifier.cpp:561-577

PARITY UNPINNED against the reference's own build: these files need Eigen,
which is absent, so the C++ reference cannot run here. The
restatement is pinned instead by ground truth -- dense generalized
eigenvalues (scipy.linalg.eigh) and exact grounded solves (scipy splu) --
in tests/test_spectral_oracle.py.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def hash_mix(x: int) -> int:  # rng.hpp:37-43 (SplitMix64 finaliser)
    x = (x + 0) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


class SplitMix64:  # rng.hpp:7-24
    def __init__(self, seed: int):
        self.state = seed & MASK

    def next_double(self) -> float:
        self.state = (self.state + GAMMA) & MASK
        return (hash_mix(self.state) >> 11) * 2.0 ** -53


def laplacian(rp, ids, w) -> sp.csr_matrix:  # laplacian.cpp:7-26
    n = len(rp) - 1
    rows = np.repeat(np.arange(n), np.diff(rp).astype(np.int64))
    deg = np.zeros(n)
    np.add.at(deg, rows, w)
    r = np.concatenate([rows, np.arange(n)])
    c = np.concatenate([ids.astype(np.int64), np.arange(n)])
    v = np.concatenate([-w, deg])
    return sp.csr_matrix((v, (r, c)), shape=(n, n))


def is_connected(rp, ids) -> bool:
    n = len(rp) - 1
    a = sp.csr_matrix((np.ones(len(ids)), ids.astype(np.int64), rp.astype(np.int64)), shape=(n, n))
    return sp.csgraph.connected_components(a, directed=False)[0] == 1


class GroundedSolver:  # laplacian.cpp:57-85: ground vertex 0, exact factorisation
    def __init__(self, lap: sp.csr_matrix):
        self.n = lap.shape[0]
        self.lu = spla.splu(sp.csc_matrix(lap[1:, 1:]))

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        b = rhs - rhs.mean()
        full = np.zeros(self.n)
        full[1:] = self.lu.solve(b[1:])
        return full - full.mean()


def condition_dense(lg, lh) -> dict:  # spectral.cpp:105-130
    n = lg.shape[0]
    q, _ = np.linalg.qr(np.ones((n, 1)), mode="complete")
    basis = q[:, 1:]
    a = basis.T @ lg.toarray() @ basis
    b = basis.T @ lh.toarray() @ basis
    a = 0.5 * (a + a.T)
    b = 0.5 * (b + b.T)
    ev = sla.eigh(a, b, eigvals_only=True)
    return dict(kappa=ev.max() / ev.min(), lambda_min=ev.min(), lambda_max=ev.max(),
                method="Dense", iterations=0, converged=True)


def tridiagonal_extremes(alphas, betas):  # spectral.cpp:132-145
    ev = sla.eigvalsh_tridiagonal(np.array(alphas), np.array(betas[: len(alphas) - 1]))
    return ev[0], ev[-1]


def condition_iterative(lg, lh, tolerance=1e-6, max_iterations=400, seed=0x5EED) -> dict:
    n = lg.shape[0]
    hsolver = GroundedSolver(lh)
    rng = SplitMix64(hash_mix(seed))
    q = np.array([rng.next_double() - 0.5 for _ in range(n)])
    q -= q.mean()
    bq = lh @ q
    norm0 = math.sqrt(q @ bq)
    if not norm0 > 0.0:
        raise ArithmeticError("degenerate Lanczos start vector")
    basis, basis_b = [q / norm0], [bq / norm0]
    alphas, betas = [], []
    est = dict(method="Iterative", converged=False)
    limit = min(max_iterations, n - 1)
    prev_min = prev_max = 0.0
    stable = 0
    for j in range(limit):
        aq = lg @ basis[j]
        wv = hsolver.solve(aq)
        alpha = basis[j] @ aq
        alphas.append(alpha)
        wv = wv - alpha * basis[j]
        if j > 0:
            wv = wv - betas[j - 1] * basis[j - 1]
        for _ in range(2):
            for i in range(len(basis)):
                wv = wv - (basis_b[i] @ wv) * basis[i]
        wv = wv - wv.mean()
        bw = lh @ wv
        beta = math.sqrt(max(wv @ bw, 0.0))
        tmin, tmax = tridiagonal_extremes(alphas, betas)
        est.update(lambda_min=tmin, lambda_max=tmax, iterations=j + 1)
        if beta < 1e-13 * max(1.0, abs(alpha)):
            est["converged"] = True
            break
        if j > 2:
            cmin = abs(tmin - prev_min) / max(abs(tmin), 1e-300)
            cmax = abs(tmax - prev_max) / max(abs(tmax), 1e-300)
            if cmin < tolerance and cmax < tolerance:
                stable += 1
                if stable >= 3:
                    est["converged"] = True
                    break
            else:
                stable = 0
        prev_min, prev_max = tmin, tmax
        betas.append(beta)
        basis.append(wv / beta)
        basis_b.append(bw / beta)
    est["kappa"] = est["lambda_max"] / est["lambda_min"]
    return est


def condition_number(g_rows, h_rows, method="Auto", tolerance=1e-6, max_iterations=400,
                     dense_cap=5000, seed=0x5EED) -> dict:  # spectral.cpp:278-303
    lg, lh = laplacian(*g_rows), laplacian(*h_rows)
    n = lg.shape[0]
    if method == "Auto":
        method = "Dense" if n <= dense_cap else "Iterative"
    if method == "Dense":
        return condition_dense(lg, lh)
    return condition_iterative(lg, lh, tolerance, max_iterations, seed)


def calibrate_budget(g_rows, h_rows, probe_fraction, rho, seed) -> float:
    n = len(g_rows[0]) - 1
    iters = int(min(max(math.ceil(probe_fraction * n), 30.0), 2000.0))
    est = condition_number(g_rows, h_rows, "Auto", 1e-3, iters, 5000, seed)
    return min(max(rho * est["kappa"], 1.0), 1e6)


class Preconditioner:  # solver.cpp:10-69
    def __init__(self, lh=None, n=None, factor_cap=2_000_000):
        self.lh = lh
        self.n = lh.shape[0] if lh is not None else n
        self.exact = GroundedSolver(lh) if lh is not None and self.n <= factor_cap else None

    def apply(self, b):
        rhs = b - b.mean()
        if self.lh is None:
            return rhs
        if self.exact is not None:
            return self.exact.solve(rhs)
        x = np.zeros(self.n)
        r = rhs.copy()
        p = r.copy()
        rho = r @ r
        target = 1e-20 * (rhs @ rhs)
        k = 0
        while k < 20 * self.n and rho > target:
            q = self.lh @ p
            alpha = rho / (p @ q)
            x += alpha * p
            r -= alpha * q
            rho_next = r @ r
            p = r + (rho_next / rho) * p
            rho = rho_next
            k += 1
        return x - x.mean()


def pcg_solve(lg, rhs, m: Preconditioner, tolerance=1e-8, max_iterations=0):
    n = lg.shape[0]  # solver.cpp:71-144
    if max_iterations == 0:
        max_iterations = 10 * n + 100
    b = rhs - rhs.mean()
    b_norm = np.linalg.norm(b)
    if b_norm == 0.0:
        return np.zeros(n), 0, 0.0, True, []
    x = np.zeros(n)
    r = b.copy()
    z = m.apply(r)
    p = z.copy()
    rho = r @ z
    energy = []
    it = 0
    for k in range(1, max_iterations + 1):
        q = lg @ p
        pq = p @ q
        if not pq > 0.0:
            raise ArithmeticError("PCG breakdown: search direction lost positivity")
        alpha = rho / pq
        x += alpha * p
        x -= x.mean()
        r -= alpha * q
        it = k
        energy.append(0.5 * (x @ (lg @ x)) - b @ x)
        if np.linalg.norm(r) <= tolerance * b_norm:
            true_r = b - lg @ x
            if np.linalg.norm(true_r) <= tolerance * b_norm:
                break
            r = true_r
            z = m.apply(r)
            p = z.copy()
            rho = r @ z
            continue
        z = m.apply(r)
        rho_next = r @ z
        p = z + (rho_next / rho) * p
        rho = rho_next
    rel = np.linalg.norm(b - lg @ x) / b_norm
    return x, it, rel, rel <= tolerance, energy


def random_rhs(n: int, seed: int) -> np.ndarray:  # solver.cpp:146-159
    rng = SplitMix64(hash_mix(seed + 0xB0C4))
    b = np.zeros(n)
    for i in range(0, n, 2):
        u1 = max(rng.next_double(), 1e-300)
        u2 = rng.next_double()
        radius = math.sqrt(-2.0 * math.log(u1))
        b[i] = radius * math.cos(2.0 * math.pi * u2)
        if i + 1 < n:
            b[i + 1] = radius * math.sin(2.0 * math.pi * u2)
    return b - b.mean()
