#!/usr/bin/env python
"""Benchmark of the batched heuristic evaluator (the hot path of Batch IDA* /
CB-DFS, arXiv 2507.11916) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step = one evaluation pass over one batch of B synthetic packed states per
GPU (random-walk scrambles, inputs resident in HBM for `value`; pinned-host ->
device -> host through the C-ABI for `e2e`).  Multi-GPU: one process per GPU
(torchrun), each GPU evaluates its own batches (no data-path collective,
weak scaling); timing is the max over ranks.

`--impl reference` times the reference's own CPU evaluator
(bida::LinearModelBackend<D>::evaluate compiled unchanged into
oracle/_ref/libbida_ref.so; for the BMLP1 workloads, which the reference does
not have, the oracle's C restatement) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (domain, model kind, params)
    "rc-linear-e1-c21": dict(domain="rc", kind="linear", E=1, C=21, q=0.5, batch=1 << 22),
    "rc-linear-e4-c21": dict(domain="rc", kind="linear", E=4, C=21, q=0.5, batch=1 << 22),
    "stp4-linear-c72": dict(domain="stp4", kind="linear", E=1, C=72, q=0.5, batch=1 << 22),
    # BMLP1 int8 MLPs; widths bracket the paper's 0.2 / 2.3 / 13.6 MB fp32 model-size
    # anchors (H ~ 85 / 547 / 1610 at two hidden layers)
    "rc-mlp-h128": dict(domain="rc", kind="mlp", H=[128, 128], E=1, C=21, q=0.5, batch=1 << 22),
    "rc-mlp-h256": dict(domain="rc", kind="mlp", H=[256, 256], E=1, C=21, q=0.5, batch=1 << 22),
    "rc-mlp-h512": dict(domain="rc", kind="mlp", H=[512, 512], E=1, C=21, q=0.5, batch=1 << 22),
    "rc-mlp-h1610": dict(domain="rc", kind="mlp", H=[1610, 1610], E=1, C=21, q=0.5, batch=1 << 21),
}
DEFAULT_WORKLOAD = "rc-mlp-h128"
LINEAR_WORKLOAD = "rc-linear-e1-c21"
WIDE_WORKLOAD = "rc-mlp-h1610"

PACKED = {"rc": 16, "stp4": 8, "stp3": 8, "stp2": 8}
NNZ = {"rc": 20, "stp4": 16, "stp3": 9, "stp2": 4}
FEAT = {"rc": 480, "stp4": 256, "stp3": 81, "stp2": 16}
L2_BYTES = 126 * 1024 * 1024

THROTTLE_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


def weights_for(wl, seed=2507):
    rng = np.random.default_rng(seed)
    return rng.uniform(-0.1, 0.1, (wl["E"], wl["C"], FEAT[wl["domain"]])).astype(np.float32)


def algorithmic(wl):
    """(bytes, flops) per state of the fused evaluator."""
    pb = PACKED[wl["domain"]]
    by = pb + 4
    if wl["kind"] == "linear":
        fl = 2 * FEAT[wl["domain"]] * wl["C"] * wl["E"]
    else:
        dims = [FEAT[wl["domain"]], *wl["H"], wl["C"]]
        fl = 2 * wl["E"] * sum(a * b for a, b in zip(dims[:-1], dims[1:]))
    return by, fl


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons through NVML every
    `period` seconds while the timed region runs (the recipe's clocks line)."""

    def __init__(self, device: int, period: float = 0.005):
        self.device, self.period = device, period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                try:
                    bits = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    bits = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((sm, bits))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join(1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        reasons = set()
        for _, bits in self.samples:
            for b, name in THROTTLE_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "source": "NVML, 5 ms period, device-timed + e2e regions"}


# ---------------------------------------------------------- dist helpers
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BIDA_BENCH_SINGLE_DEVICE") == "1":
        local = 0  # plumbing test: every rank on cuda:0 (use BIDA_BENCH_BACKEND=gloo)
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if os.environ.get("BIDA_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def whole_job_rate(states_per_rank_step: int, steps: int, world: int, max_ms: float) -> float:
    """Whole-job throughput: all ranks' states over the slowest rank's time."""
    return states_per_rank_step * steps * world / (max_ms / 1000.0)


def reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------ our arm
def make_backend(wl, device):
    import paper_2507_11916_b200 as bida

    if wl["kind"] == "linear":
        return bida.LinearModelBackend(wl["domain"], weights_for(wl), wl["C"], wl["q"], device=device)
    from paper_2507_11916_b200.models import make_bmlp1

    blob = make_bmlp1(wl["domain"], hidden=wl["H"], classes=wl["C"], ensemble=wl["E"], seed=2507)
    return bida.MlpModelBackend(wl["domain"], blob, wl["q"], device=device)


def run_ours(args, wl, rank, world, local, e2e=True):
    import torch

    import paper_2507_11916_b200 as bida

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B = args.batch or wl["batch"]
    pb = PACKED[wl["domain"]]
    # rotate input buffers whose total exceeds L2 so every step streams from HBM
    nbuf = max(2, int(np.ceil(2 * L2_BYTES / (B * pb))))
    # synthetic scrambles generated on the GPU (bida_gpu_random_walks), copied to the host
    host = [bida.random_walks_fast(wl["domain"], B, 0, 30, seed=1000 * rank + i, device=local)
            for i in range(min(nbuf, 2))]
    d_in = [torch.from_numpy(host[i % len(host)].view(np.uint8).copy()).to(dev) for i in range(nbuf)]
    d_h = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(nbuf)]
    be = make_backend(wl, local)
    stream = torch.cuda.current_stream()

    # ---- device-resident timing (value) ---------------------------------
    for i in range(args.warmup):
        be.evaluate_device(d_in[i % nbuf], d_h[i % nbuf])
    torch.cuda.synchronize()
    be.status()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = be.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local).__enter__()
    t_start.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        be.evaluate_device(d_in[i % nbuf], d_h[i % nbuf])
        ev[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    be.status()
    launches = be.launch_count() - launches0
    barrier(world)
    total_ms = t_start.elapsed_time(t_end)
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms_max = reduce_max(total_ms, world)
    kern_avg_ms = float(np.mean(kern_ms))

    if not e2e:
        clk.__exit__(None, None, None)
        be.close()
        return dict(B=B, nbuf=nbuf, total_ms=total_ms_max, kern_avg_ms=kern_avg_ms, launches=launches,
                    clocks=clk.summary(), host0=host[0])

    # ---- end-to-end through the C-ABI with host buffers (e2e) ------------
    try:
        hostbufs = [torch.from_numpy(h.view(np.uint8).copy()).pin_memory().numpy().view(h.dtype) for h in host]
    except RuntimeError:
        hostbufs = host
    try:
        out = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
    except RuntimeError:
        out = np.empty(B, np.int32)
    for i in range(max(1, args.warmup)):
        be.evaluate(hostbufs[i % len(hostbufs)], out=out)
    barrier(world)
    t0 = time.perf_counter()
    for i in range(args.steps):
        be.evaluate(hostbufs[i % len(hostbufs)], out=out)
    e2e_s = time.perf_counter() - t0
    barrier(world)
    clk.__exit__(None, None, None)
    e2e_s_max = reduce_max(e2e_s, world)
    clocks = clk.summary()
    be.close()
    return dict(B=B, nbuf=nbuf, total_ms=total_ms_max, kern_avg_ms=kern_avg_ms, launches=launches,
                e2e_s=e2e_s_max, clocks=clocks, host0=host[0])


# --------------------------------------------------------- CPU baselines
def cpu_eval_fn(wl, packed, threads):
    """Returns a zero-arg callable evaluating `packed` on `threads` host
    threads with the reference's own CPU evaluator (oracle/_ref), or the
    oracle's C restatement for BMLP1 (no reference MLP exists)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    from oracle_lib import DOMAINS, Oracle, RefLib

    d = DOMAINS[wl["domain"]]
    h = np.empty(len(packed), np.int32)
    if wl["kind"] == "linear":
        ref = RefLib()
        W = np.ascontiguousarray(weights_for(wl))
        E, Cc, _ = W.shape
        prep = ref.L.ref_linear_prepare(d, W.ctypes.data_as(C.c_void_p), E, Cc, wl["q"],
                                        packed.ctypes.data_as(C.c_void_p), len(packed))
        if not prep:
            raise RuntimeError(ref.L.ref_last_error().decode())

        def run():
            rc = ref.L.ref_linear_run(C.c_void_p(prep), h.ctypes.data_as(C.c_void_p), threads)
            if rc:
                raise RuntimeError(ref.L.ref_last_error().decode())
            return h

        return run, "reference"
    from paper_2507_11916_b200.models import make_bmlp1

    blob = make_bmlp1(wl["domain"], hidden=wl["H"], classes=wl["C"], ensemble=wl["E"], seed=2507)
    orc = Oracle()

    def run():
        return orc.mlp_evaluate(blob, d, wl["q"], packed, threads=threads)

    return run, "port"


def cpu_rate(wl, seconds_target, threads, seed=7, source=None):
    """Returns (run, kind, states, sample): run() evaluates `sample` (reps
    times) on the CPU.  `source`: draw the sample from these packed states
    (the timed batch) instead of fresh random walks."""
    import paper_2507_11916_b200 as bida

    # calibrate on a small sample, then size the sample to ~seconds_target
    probe_n = 16384 if wl["kind"] == "linear" else 65536
    packed = bida.random_walks(wl["domain"], probe_n, 0, 30, seed=seed)
    run, kind = cpu_eval_fn(wl, packed, threads)
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    per = dt / probe_n
    want = seconds_target / max(per, 1e-9)
    # the reference materialises a float feature vector per state (1.9 KB for
    # RC), so the sample is capped at 2^19 states and repeated to fill the time
    n = int(max(probe_n, min(1 << 19, want)))
    reps = int(max(1, round(want / n)))
    if source is not None:
        n = min(n, len(source))
        packed = np.ascontiguousarray(source[:n])
    else:
        packed = bida.random_walks(wl["domain"], n, 0, 30, seed=seed + 1)
    run1, kind = cpu_eval_fn(wl, packed, threads)

    def run():
        for _ in range(reps):
            out = run1()
        return out

    return run, kind, n * reps, packed


# Config-2 search instance (BASELINE configs[1]: Rubik's random walks of 14-16
# moves): solved in Table-1 mode with the 8-corner PDB (tests/search_screen.py,
# profiles/r2_search_screen.jsonl), so the leg reports time-to-solve as well
SEARCH_WALK = (14, 2508)   # (length, seed) for random_walk_instance (instance.hpp:36-57): cost 13, ~0.7 G nodes
SEARCH_CORNERS = 8


def search_command(impl, model, q, seconds, threads, gpus, evaluators, batch, timeout_us, walk, work_num=128):
    """argv of one Batch IDA* run (see search_leg).  GPU legs spread
    `evaluators` GpuBackends over `gpus` devices (evaluator e on device
    e % gpus, tools/bida_search.cpp) and route searcher thread tid to
    evaluator tid % E (batch_eval.hpp:398-400)."""
    L, seed = walk
    exe = {"fast": "tools/bin/bida_search_fast", "ring": "tools/bin/bida_search_ring",
           "reference": "tools/bin/bida_search", "cpu": "tests/cpp/bin/search_parity",
           "cpu_pdb": "tools/bin/bida_search"}[impl]
    if impl in ("fast", "ring", "reference"):
        extra = ["--mode", "gpu", "--gpu-pdb", "--gpus", str(gpus), "--evaluators", str(evaluators),
                 "--work-num", str(work_num), "--batch", str(batch), "--timeout-us", str(timeout_us)]
    elif impl == "cpu":
        extra = ["--mode", "cpu", "--immediate", "--work-num", "1"]
    else:
        extra = ["--mode", "pdb", "--immediate", "--work-num", "1"]
    return [os.path.join(ROOT, exe), "--domain", "rc", "--walks", f"1:{L}:{L}:{seed}", "--model", "mlp:" + model,
            "--q", str(q), "--table1-pdb", str(SEARCH_CORNERS), "--pdb-build", "gpu", "--threads", str(threads),
            "--time-limit", str(seconds), *extra]


def search_plan(rank, world):
    """The search legs of a bench run: rank 0 alone drives all `world` GPUs
    from one host process (one evaluator per GPU); other ranks run none."""
    if rank != 0:
        return None
    return {"impl": "fast", "gpus": world, "evaluators": world}


def search_leg(wl, seconds, threads, impl="fast", gpus=1, evaluators=1, agents=4, shards=16, batch=16384,
               timeout_us=None, walk=None, work_num=None):
    """Batch IDA* nodes/s (BASELINE metric, second half): the reference's own
    batch_idastar (search.hpp:101-237, unchanged) on one config-2 Rubik's
    scramble, the workload's BMLP1 network evaluated for every generated node,
    search guided by the reference's 8-corner PDB (PAPER.md:407 Table-1 mode;
    on the GPU the PDB lookup is fused into the device readout; the table is
    built by bida_gpu_pdb_build, byte-identical to PdbTable::build).
      impl="fast"      tools/bin/bida_search_fast: ring evaluator (SURVEY 8(f)
                       row 1) + CB-DFS searcher overlay (row 2); GpuBackend on
                       `gpus` devices, evaluator e on device e % gpus
      impl="ring"      tools/bin/bida_search_ring: ring evaluator, reference cb_dfs
      impl="reference" tools/bin/bida_search: reference Evaluator and cb_dfs
      impl="cpu"       tests/cpp/bin/search_parity: the oracle's CPU network on
                       every searcher thread (AIDA*, immediate evaluators)
      impl="cpu_pdb"   tools/bin/bida_search --mode pdb --immediate: CPU AIDA* with
                       the PDB only, no network (the paper's AIDA* row)"""
    from paper_2507_11916_b200.models import make_bmlp1

    if wl["domain"] != "rc" or wl["kind"] != "mlp":
        return None
    L, seed = walk or SEARCH_WALK
    model = f"/tmp/bida_bench_{os.getpid()}.bmlp"
    with open(model, "wb") as f:
        f.write(make_bmlp1("rc", hidden=wl["H"], classes=wl["C"], ensemble=wl["E"], seed=2507))
    # subtrees per searcher thread and flush timeout: 256 open subtrees helps
    # every GPU leg (profiles/r2_search_knobs.jsonl, r2_ring_knobs.jsonl); the
    # fast path's best flush timeout is 15 us, the others keep 25 us
    if work_num is None:
        work_num = 256
    if timeout_us is None:
        timeout_us = 15 if impl == "fast" else 25
    cmd = search_command(impl, model, wl["q"], seconds, threads, gpus, evaluators, batch, timeout_us, (L, seed),
                         work_num=work_num)
    if not os.path.exists(cmd[0]):
        return {"unavailable": f"{cmd[0]} not built"}
    env = {**os.environ, "BIDA_EVAL_AGENTS": str(agents), "BIDA_EVAL_SHARDS": str(shards)}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=seconds * 3 + 300, env=env)
    os.unlink(model)
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode or not rows:
        return {"unavailable": (out.stderr or "no output").strip().splitlines()[-1][:200]}
    r = rows[0]
    leg = {"value": r["nodes_per_s"], "unit": "nodes/s", "evals_per_s": r["evals_per_s"],
           "generated": r["generated"], "wall_s": r["wall_s"], "status": r["status"], "cost": r["cost"],
           "time_to_solve_s": r["wall_s"] if r["status"] == "solved" else None, "thresholds": r["thresholds"],
           "mean_batch": r["mean_batch"], "threads": threads, "gpus": gpus if impl in ("fast", "ring", "reference") else 0,
           "evaluators": r["evaluators"], "work_num": r["work_num"], "timeout_us": r["timeout_us"],
           "batch": r["batch"], "evaluator_impl": r.get("evaluator_impl"), "search_impl": r.get("search_impl"),
           "instance": f"random_walk_instance(solved, {L}, seed {seed})", "pdb_corners": SEARCH_CORNERS}
    if r.get("evaluator_impl") == "ring":
        leg.update(agents=agents, shards=shards)
    return leg


KORF_LEG = (4, 56, 14)  # korf10 index (#5), optimal cost, d_init (profiles/r2_korf_dinit.jsonl)


def config1_leg(seconds, threads):
    """BASELINE configs[0]: Korf's 4x4 #5 (tests/golden/instances.npz, from
    proj/data/korf10.txt) with the linear-Manhattan model (C = 72) -- the
    reference's own LinearModelBackend on the GPU (ring evaluator + CB-DFS
    overlay) and on the CPU (reference AIDA*, one subtree per thread), the same
    work-generation depth on both sides so the trees are identical."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_2507_11916_b200 as bida

    idx, cost, d_init = KORF_LEG
    g = np.load(os.path.join(ROOT, "tests", "golden", "instances.npz"))
    inst, w = f"/tmp/bida_bench_korf_{os.getpid()}.txt", f"/tmp/bida_bench_man4_{os.getpid()}.blin"
    with open(inst, "w") as f:
        f.write("".join("stp 4 " + " ".join(str((int(v) >> (4 * c)) & 15) for c in range(16)) + "\n"
                        for v in g["korf10"]))
    K, alpha, C = 16, 4.0, 72  # linear-Manhattan weights
    W = np.zeros((1, C, K * K), np.float32)
    for c in range(C):
        for cell in range(K):
            for t in range(K):
                md = 0 if t == 0 else abs(cell // 4 - t // 4) + abs(cell % 4 - t % 4)
                W[0, c, cell * K + t] = alpha * c * md - alpha * c * c / (2 * K)
    with open(w, "wb") as f:
        f.write(bida.blin1_bytes("stp4", W, C))
    common = ["--domain", "stp4", "--instances", inst, "--model", "linear:" + w, "--q", "0.5", "--first", str(idx),
              "--count", "1", "--threads", str(threads), "--d-init", str(d_init), "--time-limit", str(seconds)]
    out = {}
    for side, exe, extra, env in (
            # GPU sides: 2 agents + cores - 2 searcher threads, 10 us flush timeout
            # (tests/korf_tune.sh, profiles/r2_korf_tune_final.jsonl)
            ("gpu", "tools/bin/bida_search_fast", ["--mode", "gpu", "--work-num", "256", "--batch", "8192",
                                                   "--timeout-us", "10", "--threads", str(max(1, threads - 2))],
             {"BIDA_EVAL_AGENTS": "2", "BIDA_EVAL_SHARDS": "16"}),
            ("cpu_aidastar", "tools/bin/bida_search", ["--mode", "cpu", "--immediate", "--work-num", "1"], {}),
            # the GPU at its own best work-generation depth (18: more, shorter subtrees for the
            # latency-bound final iteration; the CPU is slowest there: profiles/r2_korf_dinit18.jsonl)
            ("gpu_d_init_18", "tools/bin/bida_search_fast", ["--mode", "gpu", "--work-num", "256", "--batch", "8192",
                                                             "--timeout-us", "10", "--threads", str(max(1, threads - 2)),
                                                             "--d-init", "18"],
             {"BIDA_EVAL_AGENTS": "2", "BIDA_EVAL_SHARDS": "16"})):
        base = list(common)
        for flag in ("--d-init", "--threads"):  # this leg's own setting replaces the shared one
            if flag in extra:
                i = base.index(flag)
                del base[i:i + 2]
        r = subprocess.run([os.path.join(ROOT, exe), *base, *extra], capture_output=True, text=True,
                           timeout=seconds * 3 + 120, env={**os.environ, **env})
        rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
        if r.returncode or not rows:
            out[side] = {"unavailable": (r.stderr or "no output").strip()[-200:]}
            continue
        x = rows[0]
        out[side] = {"value": x["nodes_per_s"], "unit": "nodes/s", "status": x["status"], "cost": x["cost"],
                     "time_to_solve_s": x["wall_s"] if x["status"] == "solved" else None,
                     "generated": x["generated"], "thresholds": x["thresholds"], "mean_batch": x["mean_batch"]}
    os.unlink(inst)
    os.unlink(w)
    g_, c_ = out.get("gpu", {}), out.get("cpu_aidastar", {})
    same = g_.get("thresholds") is not None and g_.get("thresholds") == c_.get("thresholds")
    return {"metric": "batch_idastar_nodes_per_s", "instance": f"korf10 #{idx + 1} (optimal cost {cost})",
            "model": "linear-Manhattan BLIN1, C=72 (LinearModelBackend)", "d_init": d_init, "threads": threads,
            **out, "same_thresholds": same,
            "cpu_baseline": {"value": c_.get("value"), "unit": "nodes/s", "cores": threads, "kind": "reference",
                             "sample": "the same search, reference AIDA* (immediate LinearModelBackend)"}}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, wl, rank, world):
    if rank != 0:
        return None
    threads = host_cores()
    run, kind, n, _ = cpu_rate(wl, args.ref_step_seconds, threads)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n * args.steps / total
    _, fl = algorithmic(wl)
    sample = f"{n} packed {wl['domain']} random-walk states per step (lengths 0-30), {wl['kind']} E={wl['E']} C={wl['C']}"
    return {
        "metric": "heuristic_evals_per_s", "value": value, "unit": "evals/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "batch_per_step": n, "domain": wl["domain"]},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline_and_parity(args, wl, timed_batch, local):
    """cpu_baseline leg: the reference's CPU evaluator (oracle/_ref) or the
    oracle port on all host threads over the first states of the timed batch;
    the same states through the GPU C-ABI give the parity check (flips = h
    differences, exact_replays = readouts that took the float64 replay)."""
    threads = host_cores()
    run, kind, n, sample = cpu_rate(wl, args.cpu_seconds, threads, source=timed_batch)
    t0 = time.perf_counter()
    want = run()
    dt = time.perf_counter() - t0
    cpu = {"value": n / dt, "unit": "evals/s", "cores": threads, "kind": kind,
           "sample": f"first {len(sample)} states of the timed batch (packed {wl['domain']} random walks, lengths "
                     f"0-30) x {n // len(sample)} repetition(s), {dt:.1f} s"}
    be = make_backend(wl, local)
    h = be.evaluate(sample)
    replays = be.exact_replays()
    be.close()
    flips = int((np.asarray(h) != np.asarray(want)).sum())
    parity = {"sample": len(sample), "flips": flips, "exact_replays": replays,
              "checker": "oracle/_ref LinearModelBackend<D>::evaluate (reference, unchanged)" if kind == "reference"
              else "oracle/bida_oracle.c BMLP1 port, pinned to torch-float64 + reference-readout goldens",
              "path": "bida_gpu_evaluate (C-ABI), same states as the cpu_baseline sample"}
    return cpu, parity


def pcie_h2d_gbs(local, nbytes=1 << 28, reps=5):
    """Measured host->device copy bandwidth from page-locked memory (the link
    the end-to-end path streams packed states over), best of `reps`."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", local))
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def batch_sweep(wl, local, sizes=None):
    """BASELINE configs[2]: evals/s vs batch size 2^10..2^20 on one GPU, device-
    resident (CUDA events over R back-to-back launches on the launching
    stream; small batches are L2-resident by construction -- the latency
    regime) and end to end through bida_gpu_evaluate from page-locked host
    buffers (wall clock per synchronous call, what a search agent waits on)."""
    import torch

    import paper_2507_11916_b200 as bida

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sizes = sizes or [1 << k for k in range(10, 21)]
    peak = roofline_for(DEFAULT_WORKLOAD, wl, 1, 1.0).get("peak") if wl["kind"] == "mlp" else None
    be = make_backend(wl, local)
    _, fl = algorithmic(wl)
    stream = torch.cuda.current_stream()
    out = []
    for B in sizes:
        host = bida.random_walks_fast(wl["domain"], B, 0, 30, seed=B, device=local)
        d_in = torch.from_numpy(host.view(np.uint8).copy()).to(dev)
        d_h = torch.empty(B, dtype=torch.int32, device=dev)
        R = int(min(2000, max(20, (1 << 23) // B)))
        for _ in range(3):
            be.evaluate_device(d_in, d_h)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(R):
            be.evaluate_device(d_in, d_h)
        b.record(stream)
        torch.cuda.synchronize()
        be.status()
        dev_us = a.elapsed_time(b) * 1000.0 / R
        hp = torch.from_numpy(host.view(np.uint8).copy()).pin_memory().numpy().view(host.dtype)
        ho = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
        Re = int(min(1000, max(10, (1 << 22) // B)))
        for _ in range(3):
            be.evaluate(hp, out=ho)
        t0 = time.perf_counter()
        for _ in range(Re):
            be.evaluate(hp, out=ho)
        e2e_us = (time.perf_counter() - t0) * 1e6 / Re
        tops = fl * B / dev_us / 1e6 if wl["kind"] == "mlp" else None
        out.append({"batch": B, "device_us_per_call": dev_us, "device_evals_per_s": B / dev_us * 1e6,
                    "e2e_us_per_call": e2e_us, "e2e_evals_per_s": B / e2e_us * 1e6,
                    "device_tops": tops, "tensor_frac": tops / peak if tops and peak else None})
    be.close()
    return out


def roofline_for(name, wl, B, kern_avg_ms):
    """Roofline of the dominant (only) kernel: algorithmic bytes or flops per
    launch / its CUDA-event time; peaks from MEASURED_PEAKS.json; traffic from
    the committed ncu capture of this workload (profiles/traffic.json)."""
    by, fl = algorithmic(wl)
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    kern_s = kern_avg_ms / 1000.0
    traffic, traffic_src = None, None
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tj):
        t = json.load(open(tj)).get(name)
        if t:
            traffic = t["bytes_per_launch"] * B / t["states_per_launch"]
            traffic_src = t["source"]
    if wl["kind"] == "linear":
        achieved = by * B / kern_s / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                "algorithmic_bytes_per_state": by}
    achieved = fl * B / kern_s / 1e12
    # dense int8 peak MEASURED on this pool's B200s (profiles/r2_int8_peak.json,
    # tests/int8_peak.py): back-to-back M128 N256 K32 tcgen05.mma kind::i8 on all
    # 148 SMs for ~1 s (sustained clocks); cuBLAS int8 GEMM given beside it
    pk, src, lib = None, None, None
    ip = os.path.join(ROOT, "profiles", "r2_int8_peak.json")
    if os.path.exists(ip):
        j = json.load(open(ip))
        pk, lib = j.get("int8_tcgen05_sustained_tops"), j.get("cublas_int8_tops")
        src = "measured: tcgen05 kind::i8 sustained on 148 SMs (profiles/r2_int8_peak.json)"
    if not pk:
        pk = 4500.0
        src = "fallback: B200_PROFILING.md dense 8-bit 4.5 POPS"
    return {"bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
            "frac": achieved / pk, "traffic": traffic, "traffic_source": traffic_src, "flops_per_state": fl,
            "peak_source": src, "cublas_int8_tops": lib,
            "frac_of_cublas_int8": achieved / lib if lib else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="states per GPU per step (default: workload's)")
    ap.add_argument("--cpu-seconds", type=float, default=6.0, help="CPU baseline sample size (seconds of work)")
    ap.add_argument("--ref-step-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-wide-leg", dest="wide_leg", action="store_false",
                    help="skip the config-4 (H=1610) device-resident leg of an N=1 run")
    ap.add_argument("--no-linear-leg", dest="linear_leg", action="store_false",
                    help="skip the reference-model (rc-linear-e1-c21) leg of an N=1 run")
    ap.add_argument("--no-sweep", dest="sweep", action="store_false",
                    help="skip the batch-size sweep (BASELINE configs[2]) of an N=1 run")
    ap.add_argument("--search-seconds", type=float, default=60.0,
                    help="time limit of each Batch IDA* leg (RC MLP workloads); 0 disables")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    rank, world, local = dist_init()

    if args.impl == "reference":
        line = run_reference_arm(args, wl, rank, world)
        if rank == 0:
            print(json.dumps(line), flush=True)
        return

    T0 = time.perf_counter()
    timings = {}

    def mark(name):
        timings[name] = round(time.perf_counter() - T0, 1)
        print(f"[bench] {name} done at {timings[name]} s", file=sys.stderr, flush=True)

    r = run_ours(args, wl, rank, world, local)
    mark("headline")
    if rank != 0:
        return
    B = r["B"]
    total_states = B * args.steps * world
    value = whole_job_rate(B, args.steps, world, r["total_ms"])
    roof = roofline_for(args.workload, wl, B, r["kern_avg_ms"])
    line = {
        "metric": "heuristic_evals_per_s",
        "value": value,
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["total_ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64" if wl["kind"] == "linear" else "i8",
        "data": "synthetic",
        "config": {
            "workload": args.workload,
            "domain": wl["domain"],
            "model": {k: v for k, v in wl.items() if k in ("kind", "E", "C", "q", "H")},
            "batch_per_gpu": B,
            "parallelism": f"replicas x{world} (independent batches, no collective)",
            "l2": f"{r['nbuf']} rotating input buffers, {r['nbuf'] * B * PACKED[wl['domain']] >> 20} MB total > 126 MB L2",
        },
        "roofline": roof,
        "e2e": {"value": total_states / r["e2e_s"], "unit": "evals/s",
                "h2d_bytes_per_step": B * PACKED[wl["domain"]] * world, "d2h_bytes_per_step": B * 4 * world,
                "path": "bida_gpu_evaluate (C-ABI) from/to page-locked host buffers, mapped into the device address space: one launch reads the packed states over PCIe and writes h back (direct path)"},
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
        "kernel_ms_avg": r["kern_avg_ms"],
    }
    if world == 1:
        # the end-to-end path's own roofline: packed states over PCIe, host -> device
        h2d = pcie_h2d_gbs(local)
        got = line["e2e"]["value"] * PACKED[wl["domain"]] / 1e9
        line["e2e"]["pcie"] = {"h2d_gbs_measured": h2d, "h2d_gbs_achieved": got, "frac": got / h2d,
                               "how": "pinned 256 MB torch copy_, best of 5, CUDA events"}
    if world == 1 and args.wide_leg and args.workload != WIDE_WORKLOAD:
        # config 4 (the paper's 13.6 MB model): the tensor-bound case
        # the north star's tensor-utilisation target refers to; device-resident only
        ww = WORKLOADS[WIDE_WORKLOAD]
        rw = run_ours(args, ww, rank, world, local, e2e=False)
        mark("wide_model_run")
        line["wide_model"] = {
            "workload": WIDE_WORKLOAD, "model": {k: v for k, v in ww.items() if k in ("kind", "E", "C", "q", "H")},
            "value": whole_job_rate(rw["B"], args.steps, world, rw["total_ms"]), "unit": "evals/s",
            "batch_per_gpu": rw["B"], "kernel_ms_avg": rw["kern_avg_ms"], "gpu_launches": int(rw["launches"]),
            "roofline": roofline_for(WIDE_WORKLOAD, ww, rw["B"], rw["kern_avg_ms"]), "clocks": rw["clocks"]}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = cpu_baseline_and_parity(args, wl, r["host0"], local)
        mark("cpu_baseline")
    if world == 1 and args.linear_leg and wl["kind"] != "linear":
        # the reference's own model (LinearModelBackend, BLIN1): device value, e2e,
        # roofline and its reference CPU baseline on the same timed batch
        lw = WORKLOADS[LINEAR_WORKLOAD]
        rl = run_ours(args, lw, rank, world, local)
        leg = {"workload": LINEAR_WORKLOAD, "model": {k: v for k, v in lw.items() if k in ("kind", "E", "C", "q")},
               "value": whole_job_rate(rl["B"], args.steps, world, rl["total_ms"]), "unit": "evals/s",
               "batch_per_gpu": rl["B"], "kernel_ms_avg": rl["kern_avg_ms"], "gpu_launches": int(rl["launches"]),
               "e2e": {"value": rl["B"] * args.steps / rl["e2e_s"], "unit": "evals/s",
                       "h2d_bytes_per_step": rl["B"] * PACKED[lw["domain"]], "d2h_bytes_per_step": rl["B"] * 4},
               "roofline": roofline_for(LINEAR_WORKLOAD, lw, rl["B"], rl["kern_avg_ms"]), "clocks": rl["clocks"]}
        if not args.no_cpu_baseline:
            leg["cpu_baseline"], leg["parity"] = cpu_baseline_and_parity(args, lw, rl["host0"], local)
        line["linear_model"] = leg
        mark("linear_model")
    if world == 1 and args.sweep:
        line["batch_sweep"] = {"workload": args.workload, "config": "BASELINE configs[2]: batch 2^10..2^20",
                               "points": batch_sweep(wl, local)}
        mark("batch_sweep")
    if args.search_seconds > 0 and wl["kind"] == "mlp" and wl["domain"] == "rc":
        # Batch IDA* nodes/s on all `world` GPUs from one host process (rank 0; one
        # evaluator per GPU, tid % E routing, batch_eval.hpp:398-400)
        threads = host_cores()
        # host-core budget: up to 3 agent threads per GPU evaluator within half the
        # cores, searcher threads on the rest (13 + 3 on 16 cores is the best split
        # once the submitters pre-pack: profiles/r2_search_balance_256.jsonl)
        agents = max(1, min(3, (threads // 2) // world))
        gpu_threads = max(threads // 2, threads - agents * world)
        plan = search_plan(rank, world)
        sr = search_leg(wl, args.search_seconds, gpu_threads, agents=agents, **plan)
        mark("search_" + plan["impl"])
        if sr is not None:
            sr = {"metric": "batch_idastar_nodes_per_s", **sr,
                  "config": {"domain": "rc", "heuristic": "BMLP1 evaluated per node + 8-corner PDB guidance "
                             "(PAPER.md:407 Table-1 mode)", "search": "reference batch_idastar (search.hpp:101-237)",
                             "host": f"{gpu_threads} searcher threads + {agents} agent threads per GPU on {threads} host cores"}}
            if world == 1:
                legs = {}
                for impl, kw in (("ring", {"agents": agents}), ("reference", {"evaluators": 8, "agents": 1})):
                    r2 = search_leg(wl, args.search_seconds, gpu_threads, impl=impl, **kw)
                    if r2 is not None:
                        legs[impl] = r2
                    mark("search_" + impl)
                sr["variants"] = legs
                if not args.no_cpu_baseline:
                    cb = search_leg(wl, min(args.search_seconds, 10.0), threads, impl="cpu")
                    mark("search_cpu")
                    if cb and "value" in cb:
                        sr["cpu_baseline"] = {"value": cb["value"], "unit": "nodes/s", "cores": threads, "kind": "port",
                                              "sample": f"{cb['wall_s']:.0f} s of the same search (AIDA*, immediate "
                                                        f"evaluators), oracle BMLP1 on {threads} searcher threads"}
                    cp = search_leg(wl, min(args.search_seconds, 30.0), threads, impl="cpu_pdb")
                    mark("search_cpu_pdb")
                    if cp and "value" in cp:
                        sr["cpu_pdb_only"] = cp
            line["search"] = sr
            if world == 1:
                line["search_config1"] = config1_leg(min(args.search_seconds, 60.0), threads)
                mark("search_config1")
    line["bench_seconds"] = timings
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
