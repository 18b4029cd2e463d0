"""Spectral evaluation on the device.

Mirrors the reference's spectral.hpp / solver.hpp / calibrate_budget:

* ``condition_number(G, H, options)`` -- spectral.cpp:278-303: the extreme
  generalized eigenvalues of the pencil (L_G, L_H) on the complement of the
  constant vector. Dense (n <= dense_cap): cuSOLVER's generalized symmetric
  eigensolver on the grounded pencil. Iterative: Lanczos in the L_H inner
  product with full reorthogonalisation (spectral.cpp:151-276); the L_H solves
  are a sparse Cholesky of the grounded Laplacian, as in the reference.
* ``calibrate_budget(G, H, probe_fraction, rho, seed)`` --
  sparsifier.cpp:561-583.
* ``pcg_solve(G, rhs, H, ...)`` -- solver.cpp:71-144 with
  ``Preconditioner::from_graph(H)`` (H = None: identity).
* ``random_rhs(n, seed)`` -- solver.cpp:146-159.

All of it runs in libdyg.so (csrc/spectral.cu); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ptr
from .api import DynamicGraph, SparsifierState, _check


class ConditionMethod(enum.IntEnum):  # ConditionOptions::Method (spectral.hpp:79)
    Auto = 0
    Dense = 1
    Iterative = 2


@dataclass
class ConditionOptions:  # spectral.hpp:78-85
    method: ConditionMethod = ConditionMethod.Auto
    tolerance: float = 1e-6
    max_iterations: int = 400
    dense_cap: int = 5000
    seed: int = 0x5EED

    def _struct(self) -> _lib.CondOpts:
        return _lib.CondOpts(int(self.method), int(self.max_iterations), float(self.tolerance),
                             int(self.dense_cap), 0, int(self.seed))


@dataclass
class ConditionEstimate:  # spectral.hpp:69-76
    kappa: float
    lambda_max: float
    lambda_min: float
    method: str  # "Dense" | "Iterative"
    iterations_used: int
    converged: bool
    inner_iterations: int = 0

    @classmethod
    def _from(cls, e: _lib.CondEst) -> "ConditionEstimate":
        return cls(e.kappa, e.lambda_max, e.lambda_min, "Dense" if e.method == 0 else "Iterative",
                   int(e.iterations_used), bool(e.converged), int(e.inner_iterations))


@dataclass
class PcgResult:  # solver.hpp:44-49
    solution: np.ndarray
    iterations: int
    relative_residual: float
    converged: bool
    inner_iterations: int = 0
    energy_trace: np.ndarray | None = None


def condition_number(g: DynamicGraph | SparsifierState, h: DynamicGraph | None = None,
                     options: ConditionOptions | None = None, device: int = 0
                     ) -> ConditionEstimate:
    """condition_number(G, H, options) (spectral.cpp:278-303). Pass a
    SparsifierState alone to use its current graph and sparsifier."""
    o = (options or ConditionOptions())._struct()
    out = _lib.CondEst()
    if isinstance(g, SparsifierState):
        _check(_lib.lib().dyg_session_condition_number(g._s, C.byref(o), C.byref(out)))
    else:
        cg, ch = g.csr(), h.csr()
        _check(_lib.lib().dyg_condition_number(C.byref(cg), C.byref(ch), C.byref(o),
                                               int(device), C.byref(out)))
    return ConditionEstimate._from(out)


def calibrate_budget(g: DynamicGraph | SparsifierState, h: DynamicGraph | None = None,
                     probe_fraction: float = 0.05, rho: float = 0.1, seed: int = 0,
                     device: int = 0) -> float:
    """calibrate_budget (sparsifier.cpp:561-583): clamp(rho * kappa, 1, 1e6)
    from a coarse Lanczos estimate. With a SparsifierState the seed is its
    walk.global_seed (the reference's overload)."""
    out = C.c_double(0.0)
    if isinstance(g, SparsifierState):
        _check(_lib.lib().dyg_session_calibrate_budget(g._s, float(probe_fraction), float(rho),
                                                       C.byref(out)))
    else:
        cg, ch = g.csr(), h.csr()
        _check(_lib.lib().dyg_calibrate_budget(C.byref(cg), C.byref(ch), float(probe_fraction),
                                               float(rho), int(seed), int(device), C.byref(out)))
    return float(out.value)


def pcg_solve(g: DynamicGraph, rhs: np.ndarray, preconditioner: DynamicGraph | None = None,
              tolerance: float = 1e-8, max_iterations: int = 0, factor_cap: int = 2_000_000,
              energy_trace: bool = False, device: int = 0) -> PcgResult:
    """pcg_solve(laplacian(G), rhs, Preconditioner::from_graph(H) or identity)
    (solver.cpp:71-144)."""
    n = g.vertex_count()
    b = np.ascontiguousarray(rhs, np.float64)
    if b.shape != (n,):
        raise ValueError("rhs must have one entry per vertex")
    x = np.zeros(n, np.float64)
    res = _lib.PcgRes()
    cap = (max_iterations or 10 * n + 100) if energy_trace else 0
    trace = np.zeros(max(cap, 1), np.float64)
    cg = g.csr()
    chp = None
    if preconditioner is not None:
        ch = preconditioner.csr()
        chp = C.byref(ch)
    _check(_lib.lib().dyg_pcg_solve(C.byref(cg), chp, int(factor_cap), ptr(b), float(tolerance),
                                    int(max_iterations), int(device), ptr(x), C.byref(res),
                                    ptr(trace) if energy_trace else None, cap))
    return PcgResult(x, int(res.iterations), float(res.relative_residual), bool(res.converged),
                     int(res.inner_iterations),
                     trace[: res.energy_count].copy() if energy_trace else None)


def random_rhs(n: int, seed: int) -> np.ndarray:
    """random_rhs(n, seed) (solver.cpp:146-159): seeded standard normals,
    Box-Muller on the SplitMix64 stream, projected to zero mean."""
    out = np.zeros(max(int(n), 1), np.float64)
    _check(_lib.lib().dyg_random_rhs(int(n), int(seed), ptr(out)))
    return out[: int(n)]


def ordering_cache_stats() -> dict:
    """Fill-reducing orderings reused by the exact Laplacian solves in this
    process: exact-pattern hits, near-pattern hits (<= 5 % of nonzeros
    differ) and fresh orderings (dyg_spectral_ordering_stats)."""
    v = [C.c_uint64() for _ in range(3)]
    _check(_lib.lib().dyg_spectral_ordering_stats(*[C.byref(x) for x in v]))
    return {"hits": v[0].value, "near_hits": v[1].value, "misses": v[2].value}
