#!/usr/bin/env python
"""Benchmark: dyGRASS batched incremental + decremental update on B200.

Workload (BASELINE.json metric, configs[4]): the
delaunay_n22-shaped mesh make_mesh(2048, 2048, seed 1) -- 4.19M vertices,
12.57M edges -- with the initial sparsifier at 10% off-tree density and the
generated 10 insertion + 10 deletion batch stream (1,048,576 insertions,
125,747 deletions; K=100, T=100, s=16, walk seed 42). Synthetic data from the
reference's own deterministic generators (no network datasets).

A step = restore (G0, H0, counter 0) from the device snapshot + replay of all
20 batches through the reference-shaped API. value = edge updates per second
over the timed steps (device timeline, CUDA events on the session stream);
e2e = the same through the C-ABI with host event buffers (H2D of every
batch's events and D2H of every batch report inside the timed region).

--impl reference times the reference CPU implementation (oracle/_ref: the
unmodified /root/reference sources) on the host's cores, one batch per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (rows, cols, generator, insert_fraction, delete_fraction, locality)
    "C1": (100, 100, "mesh", 0.25, 0.0, 3),
    "C2": (100, 110, "mesh", 0.25, 0.01, 3),
    "C3": (512, 512, "mesh", 0.25, 0.01, 3),
    "C4": (1225, 1225, "grid4", 0.25, 0.0, 0),
    "C5": (2048, 2048, "mesh", 0.25, 0.01, 0),
}
WORKLOAD_NAMES = {
    "C1": "grid 100x100", "C2": "fe_4elt-shaped mesh 100x110",
    "C3": "delaunay_n18-shaped mesh 512x512", "C4": "G3_circuit-shaped grid 1225x1225",
    "C5": "delaunay_n22-shaped mesh 2048x2048",
}
K_BUDGET, T_CAP, WALKERS, WALK_SEED = 100.0, 100, 16, 42


def workload_name(cfg, scale=1):
    if scale == 1:
        return WORKLOAD_NAMES[cfg]
    rows, cols = config_shape(cfg, scale)[:2]
    return f"{WORKLOAD_NAMES[cfg]} widened x{scale} for weak scaling ({rows}x{cols})"
METRIC = "edge updates/sec (T_update per batch) at 1/2/4/8 B200 vs CPU ref"
UNIT = "edge_updates/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config_shape(cfg, scale=1):
    """(rows, cols, generator, insert fraction, delete fraction, locality);
    weak scaling widens the mesh by the GPU count (n, m and the events per
    batch all grow by exactly `scale`)."""
    rows, cols, kind, ins, dele, loc = CONFIGS[cfg]
    return rows, cols * scale, kind, ins, dele, loc


def make_inputs_product(cfg, scale=1):
    import paper_2505_02741_b200 as D
    rows, cols, kind, ins, dele, loc = config_shape(cfg, scale)
    gen = D.make_mesh if kind == "mesh" else D.make_grid4
    g = gen(rows, cols, 1)
    # The device builder, bit-identical to the host one.
    h = D.build_initial_sparsifier_gpu(g, 0.10, 1)
    # The stream: insertion sampling on the device for locality 0 (C4 / C5;
    # bit-identical, checked against the reference arm's inputs below).
    o = D.StreamGenOptions(ins, dele, 10, 7, loc)
    s = D.generate_update_stream_gpu(g, o) if loc == 0 else D.generate_update_stream(g, o)
    return g, h, s


def make_inputs_oracle(orc, cfg, scale=1):
    rows, cols, kind, ins, dele, loc = config_shape(cfg, scale)
    g = orc.make_mesh(rows, cols, 1) if kind == "mesh" else orc.make_grid4(rows, cols, 1)
    h = orc.build_initial_sparsifier(g, 0.10, 1)
    s = orc.generate_stream(g, ins, dele, 10, 7, loc)
    return g, h, s


def digest(*arrays) -> str:
    """blake2b over the raw bytes of row exports / event arrays: the two arms'
    inputs and the replicas' states are compared through these."""
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).data)
    return h.hexdigest()


def inputs_digest(g_rows, h_rows, events) -> dict:
    return {"G": digest(*g_rows), "H0": digest(*h_rows), "stream": digest(events)}


REPORT_KEYS = ("insertions_seen", "insertions_kept", "insertions_pruned", "deletions_seen",
               "deletions_in_sparsifier", "paths_recovered", "edges_recovered",
               "fallback_activations", "walker_steps", "max_event_steps")


def report_tuple(reps) -> tuple:
    return tuple(tuple(int(getattr(r, k)) for k in REPORT_KEYS) for r in reps)


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 5 ms from a thread (the timed region is tens of ms), else
    nvidia-smi at its 100 ms minimum."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.stop = index, [], None, threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = self.reasons_fn(self.h)
                self.rows.append((float(mhz), float(self.max_mhz), int(rs)))
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, _, bits in self.rows for n, b in self.REASONS.items()
                          if bits & b})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# Random-gather ceiling measured on this pool (tools/gather_peak.cu ->
# profiles/gather_peak_r1.txt): best rows/s for (row bytes, table MB).
GATHER_CEILING = {(64, 281): 69.6e9, (64, 563): 50.9e9, (128, 281): 43.6e9, (128, 563): 40.2e9}


def gather_ceiling(row_bytes: int, table_mb: float) -> float:
    """Rows/s ceiling, log-linear in table size between the measured points."""
    import math
    lo, hi = GATHER_CEILING[(row_bytes, 281)], GATHER_CEILING[(row_bytes, 563)]
    t = min(max((math.log(table_mb) - math.log(281)) / (math.log(563) - math.log(281)), 0.0), 1.0)
    return lo + t * (hi - lo)


def load_peak():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(kernel: str):
    """dram bytes per launch from the committed ncu --set full capture."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def _spin(n: int) -> int:
    x = 0
    for i in range(n):
        x ^= i * 2654435761 & 0xFFFF
    return x


def effective_parallelism(workers: int, n: int = 3_000_000) -> float:
    """how many of the host's threads really run in parallel
    (vCPUs can be oversubscribed): the same busy loop on 1 and on `workers`
    processes, t1 * workers / t_workers."""
    from concurrent.futures import ProcessPoolExecutor
    with ProcessPoolExecutor(max_workers=workers) as ex:
        list(ex.map(_spin, [1000] * workers))  # start the workers
        t = time.perf_counter()
        list(ex.map(_spin, [n]))
        t1 = time.perf_counter() - t
        t = time.perf_counter()
        list(ex.map(_spin, [n] * workers))
        tw = time.perf_counter() - t
    return t1 * workers / tw


def cpu_baseline(cfg: str, product_inputs: dict | None = None, scale: int = 1):
    """The reference CPU implementation on this host: the WHOLE stream of the
    config replayed (deferred mode, SparsifierState::replay_batch per batch)
    from the initial state on all host threads, timed per batch kind. Its
    inputs come from the reference's own generators; their digests must equal
    the product arm's."""
    from oracle import oracle as O
    kind = "reference" if O.available("reference") else "port"
    orc = O.load("reference" if kind == "reference" else "restate")
    cores = os.cpu_count() or 1
    os.environ["DYSPARSE_THREADS"] = str(cores)
    t0 = time.perf_counter()
    g, h, s = make_inputs_oracle(orc, cfg, scale)
    setup = time.perf_counter() - t0
    ev = s.events()
    ref_inputs = inputs_digest(g.export(), h.export(), ev)
    if product_inputs is not None and ref_inputs != product_inputs:
        raise RuntimeError(f"inputs differ: product {product_inputs} reference {ref_inputs}")
    # the reference's walk-only run_batch time on batch 0's
    # reach queries (built as replay_batch_deferred does, sparsifier.cpp:
    # 433-445: w_pq = G.w(u, v) + w -- the generator's insertions are
    # non-edges -- and a query only when both endpoints have H edges).
    walk_only = None
    try:
        from oracle import oracle as _O
        hrp = np.asarray(h.export()[0]).astype(np.int64)
        hdeg = np.diff(hrp)
        b0 = ev[(ev["batch_index"] == 0) & (ev["kind"] == 0)]
        keep = (hdeg[b0["u"].astype(np.int64)] > 0) & (hdeg[b0["v"].astype(np.int64)] > 0)
        q = np.zeros(int(keep.sum()), _O.QUERY_DTYPE)
        q["kind"], q["p"], q["q"] = 0, b0["u"][keep], b0["v"][keep]
        q["w_pq"], q["update_id"] = b0["weight"][keep], np.nonzero(keep)[0]
        t = time.perf_counter()
        orc.run_batch(h, q, K_BUDGET, T_CAP, WALKERS, WALK_SEED, workers=cores)
        dt = time.perf_counter() - t
        walk_only = {"batch": 0, "queries": len(q), "s": round(dt, 3),
                     "queries_per_s": len(q) / dt}
    except Exception as e:  # noqa: BLE001 -- a diagnostic only
        walk_only = {"unavailable": str(e)[:120]}
    st = orc.state(g, h, K=K_BUDGET, T=T_CAP, s=WALKERS, seed=WALK_SEED)
    split = {"insertion": [0, 0.0, 0], "deletion": [0, 0.0, 0]}
    for b in range(s.batch_count):
        t = time.perf_counter()
        r = st.replay_batch(s, b)
        dt = time.perf_counter() - t
        k = "deletion" if r["deletions_seen"] else "insertion"
        split[k][0] += int(r["insertions_seen"] + r["deletions_seen"])
        split[k][1] += dt
        split[k][2] += 1
    events = sum(v[0] for v in split.values())
    wall = sum(v[1] for v in split.values())
    cpu_model = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")),
                             "")
    except OSError:
        pass
    return {"value": events / wall, "unit": UNIT,
            "cores": cores if kind == "reference" else 1, "kind": kind,
            "per_batch_kind": {k: {"batches": v[2], "events": v[0], "s": round(v[1], 3),
                                   "t_update_ms_per_batch": 1e3 * v[1] / v[2],
                                   "edge_updates_per_s": v[0] / v[1]}
                               for k, v in split.items() if v[2]},
            "cpu_model": cpu_model, "nproc": os.cpu_count(),
            "effective_parallelism": round(effective_parallelism(cores), 2),
            "walk_only_run_batch": walk_only,
            "inputs": ref_inputs, "inputs_match_product": product_inputs is not None,
            "sample": (f"{cfg}: all {s.batch_count} batches ({events} events) replayed from the "
                       f"initial state in {wall:.2f} s (setup {setup:.1f} s excluded), "
                       "SparsifierState::replay_batch batched mode")}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    kind = "reference" if O.available("reference") else "port"
    orc = O.load("reference" if kind == "reference" else "restate")
    cores = os.cpu_count() or 1
    os.environ["DYSPARSE_THREADS"] = str(cores)
    scale = world if args.scaling == "weak" else 1
    g, h, s = make_inputs_oracle(orc, args.config, scale)
    nb = s.batch_count
    ref_inputs = inputs_digest(g.export(), h.export(), s.events())
    st = orc.state(g, h, K=K_BUDGET, T=T_CAP, s=WALKERS, seed=WALK_SEED)
    b = 0

    def step():
        """One batch, in stream order; only replay_batch is timed (the
        state is rebuilt from (G0, H0) outside the clock after the last)."""
        nonlocal st, b
        if b == nb:
            st, b = orc.state(g, h, K=K_BUDGET, T=T_CAP, s=WALKERS, seed=WALK_SEED), 0
        t = time.perf_counter()
        r = st.replay_batch(s, b)
        dt = time.perf_counter() - t
        b += 1
        return int(r["insertions_seen"] + r["deletions_seen"]), dt

    for _ in range(args.warmup):
        step()
    events, el = 0, 0.0
    for _ in range(args.steps):
        e, dt = step()
        events += e
        el += dt
    v = events / el
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators)",
        "config": {"workload": workload_name(args.config, scale), "config": args.config,
                   "step": "one deferred batch of the stream, in order",
                   "K": K_BUDGET, "T": T_CAP, "s": WALKERS, "inputs": ref_inputs},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores if kind == "reference" else 1,
                         "kind": kind,
                         "sample": f"{args.steps} consecutive batches of {args.config}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def gather_block(stats, n):
    """K1 / K2 step rates against the measured random-gather ceiling (the DRAM
    side is access-bound: ~40 G rows/s at any row size once the table is far
    beyond L2, so the copy peak above is not reachable by a gather)."""
    out = {}
    for key, ms, steps, row, table in (
            ("k_reach", stats["reach_ms"], stats["reach_steps"], 64, 96 * n / 2**20),
            ("k_minpath", stats["minpath_walk_ms"], stats["minpath_steps"], 128,
             128 * n / 2**20)):
        if ms <= 0:
            continue
        rate = steps / (ms * 1e-3)
        ceil = gather_ceiling(row, table)
        out[key] = {"steps_per_s": rate, "row_bytes": row, "table_mb": round(table, 1),
                    "ceiling_rows_per_s": ceil, "frac": rate / ceil}
    out["source"] = "profiles/gather_peak_r1.txt (tools/gather_peak.cu, measured on this pool)"
    out["durations"] = ("device stamps per launch: K1 first warp start to last warp exit; "
                        "K2 likewise (the winner kernel K3 excluded)")
    return out


def walk_phase_fracs(stats, walk_key, wms, wbytes, peak):
    """The dominant walk kernel split at the moment its work queue drains:
    the bulk (the GPU full of walkers, access-rate bound) and the tail (the
    last walkers' dependent row fetches, latency bound). Bytes are the
    kernel's own per-step counts, times its device stamps."""
    k = "reach" if walk_key.startswith("k_reach") else "minpath"
    t_ms, t_bytes = stats[f"{k}_tail_ms"], stats[f"{k}_tail_row_bytes"]
    b_ms, b_bytes = wms - t_ms, wbytes - t_bytes
    if not peak or b_ms <= 0 or t_ms <= 0:
        return {}
    return {"frac_bulk": b_bytes / (b_ms * 1e-3) / 1e9 / peak,
            "frac_tail": t_bytes / (t_ms * 1e-3) / 1e9 / peak,
            "tail_share_of_time": t_ms / wms, "tail_share_of_bytes": t_bytes / wbytes}


def run_ours(args):
    import torch

    import paper_2505_02741_b200 as D
    from paper_2505_02741_b200.parallel import ShardedReplay

    rank, world, local = dist_env()
    force_shard = world == 1 and args.force_shard
    if world > 1 or force_shard:
        import torch.distributed as dist
        # rank 0 prints exactly one JSON line on stdout: everything the
        # collectives' libraries print (NCCL's version banner) goes to stderr
        # until then.
        sys.stdout.flush()
        real_stdout = os.dup(1)
        os.dup2(2, 1)
        # DYG_BENCH_SHARED_GPU=1 (a test switch): every rank on cuda:0 over gloo
        # -- the N > 1 script path on a one-GPU box (the ranks' contexts
        # time-slice the GPU, so its numbers are not scaling numbers).
        shared = os.environ.get("DYG_BENCH_SHARED_GPU") == "1"
        if shared:
            local = 0
        torch.cuda.set_device(local)
        if shared:
            dist.init_process_group("gloo")
        elif force_shard:  # the N > 1 code path on one GPU (a world of one rank)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            dist.init_process_group("nccl", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    t0 = time.perf_counter()
    scale = world if args.scaling == "weak" else 1
    g, h, stream = make_inputs_product(args.config, scale)
    prod_inputs = inputs_digest(g.rows(), h.rows(), stream.events)
    log(f"[rank {rank}] inputs {time.perf_counter() - t0:.1f}s")
    opts = D.SparsifierOptions(D.WalkConfig(K_BUDGET, T_CAP, WALKERS, WALK_SEED), True, False)
    st = D.SparsifierState(g, h, opts, device=dev)
    # A dedicated (capturable) stream: the session enqueues each replay as a
    # CUDA graph; the legacy default stream cannot be captured.
    torch_stream = torch.cuda.Stream()
    torch.cuda.set_stream(torch_stream)
    st.set_stream(torch_stream.cuda_stream)
    st.snapshot()
    nb = stream.batch_count
    batches = [stream.batch(b) for b in range(nb)]
    n_events = int(sum(len(e) for e, _ in batches))
    sharded = (ShardedReplay(st, rank, world, transport=args.transport)
               if (world > 1 or force_shard) else None)
    # device-resident events for the device-timed step
    if sharded is None:
        st.upload_stream(stream)
    else:
        sharded.upload(stream)

    def step_device():
        st.restore()
        if sharded is None:
            return st.replay_uploaded_range(0, nb)  # device-resident replay(stream)
        return sharded.replay_uploaded_range(0, nb)

    def step_e2e():
        # The reference-facing replay(stream) from the host stream (page-locked
        # UpdateStream): every batch's events cross PCIe inside the step, the
        # reports come back; the library pipelines the uploads with the work.
        st.restore()
        if sharded is None:
            return st.replay(stream).batches
        return sharded.replay_stream(stream)

    def state_digest():
        return digest(*st.rows(0)), digest(*st.rows(1))

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        dev_t = "cuda" if torch.distributed.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev_t)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    log(f"[rank {rank}] session ready; warm-up")
    # The first replay runs the instrumented walk kernels (per-step steps and
    # algorithmic bytes, ~6 % slower); the timed replays run the default
    # ones. The walks are identical (same stream, same snapshot, same seeds:
    # every timed replay's reports and final G/H digests must equal this
    # one's), so its counts are the timed replays' counts.
    st.set_walk_counters(True)
    st.reset_stats()
    first_reports = report_tuple(step_device())
    torch.cuda.synchronize()
    count_stats = st.stats()
    st.set_walk_counters(False)
    first_state = state_digest()
    for _ in range(args.warmup - 1):
        step_device()
    torch.cuda.synchronize()
    log(f"[rank {rank}] timed steps")
    st.reset_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        barrier()
        torch.cuda.synchronize()
        timed_reports = []
        ev0.record(torch_stream)
        for _ in range(args.steps):
            timed_reports.append(step_device())
        ev1.record(torch_stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    stats = st.stats()
    for f in ("reach_steps", "minpath_steps", "reach_row_bytes", "minpath_row_bytes",
              "reach_tail_row_bytes", "minpath_tail_row_bytes"):
        stats[f] = count_stats[f] * args.steps  # per-step counts of the instrumented replay
    timed_state = state_digest()  # before the restore diagnostic below
    log(f"[rank {rank}] device {ms:.3f} ms/step; end-to-end")
    # Diagnostic: the snapshot restore each step begins with (not update work).
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(torch_stream)
    for _ in range(3):
        st.restore()
    r1.record(torch_stream)
    torch.cuda.synchronize()
    restore_ms = r0.elapsed_time(r1) / 3
    # Self-check: every timed step reported what the first replay reported,
    # and the last one left the first replay's G and H (row digests).
    for reps in timed_reports:
        if report_tuple(reps) != first_reports:
            raise RuntimeError("a timed device replay reported differently from the first")
    if timed_state != first_state:
        raise RuntimeError("the timed device replays ended in a different G/H state")
    kinds = {"insertion": [0, 0.0, 0], "deletion": [0, 0.0, 0]}
    for reps in timed_reports:
        for r in reps:
            k = kinds["deletion" if r.deletions_seen else "insertion"]
            k[0] += int(r.insertions_seen + r.deletions_seen)
            k[1] += r.wall_ms
            k[2] += 1
    t_update = {k: {"batches_per_step": v[2] // args.steps,
                    "t_update_ms_per_batch": v[1] / v[2],
                    "edge_updates_per_s": v[0] / (v[1] * 1e-3)}
                for k, v in kinds.items() if v[2]}
    rep_events = n_events

    # End-to-end through the C-ABI with host buffers.
    st.reset_stats()
    for _ in range(min(args.warmup, 1)):
        step_e2e()
    torch.cuda.synchronize()
    st.reset_stats()
    barrier()
    t = time.perf_counter()
    e2e_reports = []
    for _ in range(args.steps):
        e2e_reports.append(step_e2e())
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(1e3 * (time.perf_counter() - t) / args.steps)
    if any(report_tuple(r) != first_reports for r in e2e_reports) or \
            state_digest() != first_state:
        raise RuntimeError("an end-to-end replay differs from the first device replay")
    estats = st.stats()
    log(f"[rank {rank}] e2e {e2e_ms:.3f} ms/step")

    if rank != 0:
        return
    peak, peak_src = load_peak()
    kern = {
        "k_reach (K1, reach walks on H)": (stats["reach_ms"], stats["reach_row_bytes"]),
        "k_minpath+finish (K2+K3, recovery walks on shadow G)":
            (stats["minpath_ms"], stats["minpath_row_bytes"]),
        "k_rounds<CommitOp> (K6-K8 commit)": (stats["commit_ms"], None),
    }
    dom = max(kern, key=lambda k: kern[k][0])
    walk_key = max(list(kern)[:2], key=lambda k: kern[k][0])
    wms, wbytes = kern[walk_key]
    achieved = wbytes / (wms * 1e-3) / 1e9 if wms > 0 else 0.0
    launches = stats["batches"]  # one reach or min-path launch per batch phase
    out = {
        "metric": METRIC,
        "value": rep_events / (ms * 1e-3),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference generators: make_mesh, build_initial_sparsifier, "
                "generate_update_stream; bit-identical inputs)",
        "config": {
            "workload": workload_name(args.config, scale), "config": args.config,
            "vertices": g.vertex_count(), "edges": g.edge_count(),
            "sparsifier_edges": h.edge_count(), "batches": nb, "events_per_step": rep_events,
            "step": (f"restore(G0,H0) + replay of all batches ({kinds['insertion'][2] // args.steps}"
                     f" incremental + {kinds['deletion'][2] // args.steps} decremental)"),
            "K": K_BUDGET, "T": T_CAP, "s": WALKERS, "walk_seed": WALK_SEED,
            "parallelism": (f"replicated G/H, walks sharded x{world}, {sharded.transport} exchange"
                            if (world > 1 or force_shard)
                            else "1 GPU"),
            "l2": (f"inputs larger than L2 (G slabs {g.vertex_count() * 128 / 1e6:.0f} MB + "
                   f"H slabs {g.vertex_count() * 96 / 1e6:.0f} MB > 126 MB)"),
            "inputs": prod_inputs,
        },
        "self_check": ("every timed step's reports equal the first replay's, and the final "
                       "G/H row digests equal the first replay's (device and e2e)"),
        "t_update_per_batch_kind": t_update,
        "e2e": {
            "value": rep_events / (e2e_ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": int(estats["h2d_bytes"] // args.steps),
            "d2h_bytes_per_step": int(estats["d2h_bytes"] // args.steps),
        },
        "gpu_launches": int(stats["kernel_launches"]),
        "graph_launches": int(stats["graph_launches"]),
        "roofline": {
            "kernel": walk_key, "bound": "hbm", "achieved": achieved, "peak": peak,
            "peak_source": peak_src, "unit": "GB/s",
            "frac": achieved / peak if peak else None,
            **walk_phase_fracs(stats, walk_key, wms, wbytes, peak),
            "traffic": load_traffic(walk_key.split(" ")[0]),
            "algorithmic_bytes_per_launch": wbytes / max(1, stats["batches"] // 2),
            "avg_launch_ms": wms / max(1, stats["batches"] // 2),
            "duration_source": "kernel-written %globaltimer stamps (first warp start to last "
                               "warp exit), summed over the timed steps; the step itself is "
                               "CUDA-event timed",
            "bytes_source": "the kernel's own per-step count of B_step, from the first "
                            "(instrumented) replay of the same stream -- identical walks: "
                            "every timed replay's reports and final G/H digests equal it; "
                            "the bulk / tail byte split is that replay's",
            "dominant_phase": dom,
        },
        "gather_roofline": gather_block(stats, g.vertex_count()),
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in kern.items()},
        "device_ms_per_step": stats["total_ms"] / args.steps,
        "restore_ms_per_step": restore_ms,
        "walker_steps_per_step": (stats["reach_steps"] + stats["minpath_steps"]) / args.steps,
        "commit_rounds_per_step": stats["commit_rounds"] / args.steps,
        "commit_ms_per_step_deletion_batches": stats["commit_ms_deletion"] / args.steps,
        "commit_rounds_per_step_deletion_batches": stats["commit_rounds_deletion"] / args.steps,
        "flow_commit_phase_ms_per_step": {
            k: stats[f"flow_ms_{k}"] / args.steps
            for k in ("promote", "emit", "rank", "apply", "reset")},
        "walk_tail_ms_per_step": {"reach": stats["reach_tail_ms"] / args.steps,
                                  "minpath": stats["minpath_tail_ms"] / args.steps},
        "gaps_ms_per_step": {"prep": stats["prep_ms"] / args.steps,
                             "walk_to_commit": stats["walk_commit_gap_ms"] / args.steps,
                             "between_batches": stats["batch_gap_ms"] / args.steps},
        "clocks": clocks.summary(),
    }
    del launches
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(args.config, prod_inputs, scale)
        except Exception as exc:  # reported, never silently replaced
            out["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if world > 1 or force_shard:
        sys.stdout.flush()
        os.dup2(real_stdout, 1)
    print(json.dumps(out), flush=True)
    st.close()
    if world > 1 or force_shard:
        torch.distributed.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS), default="C5")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                   help="weak: the mesh is widened by the GPU count (cols x N), so the "
                        "events and queries per batch grow with N")
    p.add_argument("--force-shard", action="store_true",
                   help="one GPU through the multi-GPU (sharded) code path")
    p.add_argument("--transport", choices=["peer", "collective"], default="peer",
                   help="multi-GPU record exchange: device peer memory (CUDA IPC over NVLink, "
                        "one graph per range) or a torch.distributed all-gather per batch")
    args = p.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
