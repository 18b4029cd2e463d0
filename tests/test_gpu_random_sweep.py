"""Randomised parity sweep: random connected graphs (with pendant vertices)
and meshes, random initial-sparsifier densities, adversarial streams
(coalescing, re-insertions, deletions of just-inserted edges, mixed or
separate batches), random walk configurations (K including 0 and +large, T
from 1, s up to 33 -- more walkers than a warp) in batched and immediate
mode -- every batch's report and every G / H row against the reference."""
import numpy as np
import pytest

from tests.parity import compare_replay
from tests.test_gpu_replay import adversarial_stream

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", list(range(101, 161)))
def test_random_configuration(oracle, dyg, seed):
    rng = np.random.default_rng(seed)
    if rng.random() < 0.5:
        n = int(rng.integers(30, 400))
        g = oracle.make_random_connected(n, int(rng.integers(n // 2, 3 * n)), seed,
                                         with_pendant=bool(rng.random() < 0.7))
    else:
        g = oracle.make_mesh(int(rng.integers(5, 20)), int(rng.integers(5, 20)), seed)
    h = oracle.build_initial_sparsifier(g, float(rng.choice([0.0, 0.05, 0.1, 0.3])), seed)
    ev, nb = adversarial_stream(oracle, g, seed, batches=int(rng.integers(2, 7)),
                                per_batch=int(rng.integers(10, 80)),
                                p_del=float(rng.uniform(0.1, 0.6)), mixed=bool(rng.random() < 0.6))
    K = float(rng.choice([0.0, 1.0, 10.0, 100.0, 1e18]))
    T = int(rng.choice([1, 5, 30, 100]))
    s = int(rng.choice([1, 4, 16, 33]))
    batched = bool(rng.random() < 0.8)
    compare_replay(dyg, oracle, g, h, ev, nb, K=K, T=T, s=s, seed=int(seed), batched=batched)
