"""Every engine alternative of the device path must give the reference's
results bit for bit: the single-pass prepare vs the multi-kernel chain, the
per-row walk shadow vs its dependency rounds, the insertion fast path vs the
round engine, the dataflow deletion commit vs the rounds (and its own
overflow fallback), and CUDA-graph replay vs eager launches. The knobs are
read when a session is created."""
import pytest

from oracle import oracle as O
from tests.parity import compare_replay

pytestmark = pytest.mark.gpu

KNOBS = [
    {},
    {"DYG_SINGLE_PASS": "0"},
    {"DYG_SHADOW_ROUNDS": "1"},
    {"DYG_COMMIT_ROUNDS": "1"},
    {"DYG_NO_FASTPATH": "1"},
    {"DYG_GRAPHS": "0"},
    {"DYG_FLOW_CAP": "64"},  # record buffer overflow -> rounds inside k_del_flow
    {"DYG_REACH_SPLIT": "0"},
    {"DYG_KEEP_SHADOW": "0"},
    {"DYG_FLOW_BALANCE": "0"},
    {"DYG_SINGLE_PASS": "0", "DYG_SHADOW_ROUNDS": "1", "DYG_COMMIT_ROUNDS": "1",
     "DYG_GRAPHS": "0"},
]


@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items())
                         or "default")
def test_engines_match_reference_c2(oracle, dyg, monkeypatch, knobs):
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    c = O.CONFIGS["C2"]
    g, h, s = O.build_config(oracle, c)
    compare_replay(dyg, oracle, g, h, s.events(), s.batch_count, K=c.K, T=c.T, s=c.s,
                   seed=c.walk_seed)


@pytest.mark.parametrize("knobs", KNOBS[:4], ids=["default", "chain", "shadow-rounds",
                                                  "commit-rounds"])
def test_engines_match_reference_mixed(oracle, dyg, monkeypatch, knobs):
    # Mixed insertion + deletion batches with repeats and coalescing.
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    g = oracle.make_mesh(24, 24, 11)
    h = oracle.build_initial_sparsifier(g, 0.1, 11)
    st = oracle.generate_stream(g, 0.2, 0.05, 4, 13, 2)
    ev = st.events().copy()
    # Interleave: move every deletion into the insertion batch before it.
    ev["batch_index"] = ev["batch_index"] % 2
    ev = ev[ev["batch_index"].argsort(kind="stable")]
    compare_replay(dyg, oracle, g, h, ev, 2, K=50.0, T=60, s=8, seed=5)
