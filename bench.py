#!/usr/bin/env python
"""bench.py -- BLR prefill forward on B200: tokens/s, speedup vs cuBLAS dense bf16, roofline.

Default workload = BASELINE.json configs[1] (C2): the GPT2-S MLP (c_fc 768->3072, then
c_proj 3072->768) over batch 8 x seq 1024 = 8192 tokens, run in each BLR format of PAPER.md
Table 3 (low-rank r=192; Monarch r=192 b=4; BLAST r=192 b=6).  One *step* = one pass of the
whole hot path over the batch: the three MLPs back to back (6 BLR layer calls, 12 kernels).
value = tokens/s counting one token through one BLR MLP as one token (3 * 8192 per step).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2|C1|C3|C4|C4M]

Multi-GPU (torchrun, one process per GPU): every rank runs the full batch on its own GPU
(token-sharded weak scaling, factors replicated, no collective on the data path); the step
time is the max over ranks; value = tokens of all ranks / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_20861_b200 import configs, roofline, synth  # noqa: E402

METRIC = "BLR layer tokens/s & speedup vs cuBLAS dense bf16; % of B200 HBM/TC roofline"


# ------------------------------------------------------------------------------- helpers -------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def factors_for(L, layer_id, device):
    if L.method == "lowrank":
        return synth.lowrank_factors(L.i, L.o, L.r, 0, layer_id, device)
    if L.method == "monarch":
        return synth.monarch_factors(L.i, L.o, L.b1, L.b2, L.r_blk, 0, layer_id, device)
    return synth.blast_factors(L.i, L.o, L.b1, L.b2, L.r, 0, layer_id, device)


def build_chains(w):
    """Group the workload's layers into chains (one per method): c_fc -> c_proj style MLPs when
    consecutive layers connect (o == next i), else single layers."""
    by_method = {}
    for j, L in enumerate(w.layers):
        by_method.setdefault(L.method, []).append((j, L))
    chains = []
    for m, items in by_method.items():
        cur = []
        for j, L in items:
            if cur and cur[-1][1].o != L.i:
                chains.append(cur)
                cur = []
            cur.append((j, L))
        chains.append(cur)
    return chains


class Sampler:
    """nvml clock / throttle-reason sampler running during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.ok = False
        self.samples = []
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        mhz = [s[0] for s in self.samples]
        mask = 0
        for _, rs in self.samples:
            mask |= rs
        reasons = [v for k, v in self.REASONS.items() if mask & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(mhz)}


# ------------------------------------------------------------------------------- reference ----
def run_reference(args, w):
    """--impl reference: the fp64 oracle as it stands, on this host's cores, on a bounded sample
    of the same workload (each step = `rows` token rows through every layer of the workload)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    from oracle import oracle as orc
    rows = args.ref_rows
    chains = build_chains(w)
    facs = {j: [t.float().numpy().astype(np.float64) for t in factors_for(L, j, "cpu")] for j, L in enumerate(w.layers)}
    X = synth.make_x(rows, w.layers[0].i, seed=0).float().numpy().astype(np.float64)

    def step():
        for chain in chains:
            h = X if chain[0][1].i == X.shape[1] else synth.make_x(rows, chain[0][1].i, seed=1).double().numpy()
            for j, L in chain:
                f = facs[j]
                if L.method == "lowrank":
                    h = orc.lowrank_forward(h, *f)
                elif L.method == "monarch":
                    h = orc.monarch_forward(h, *f, L.b1, L.b2)
                else:
                    h = orc.blast_forward(h, *f)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = rows * len(chains) / dt
    cores = orc.num_threads()
    sample = f"{rows} token rows of {w.key} through all {len(w.layers)} layers per step (fp64 oracle)"
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.key}: {w.desc}", "rows_per_step": rows},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(w, target_s=10.0):
    """Time the oracle (as it stands) on a bounded token sample of the same workload."""
    import numpy as np

    from oracle import oracle as orc
    chains = build_chains(w)
    facs = {j: [t.float().numpy().astype(np.float64) for t in factors_for(L, j, "cpu")] for j, L in enumerate(w.layers)}

    def run(rows):
        t0 = time.perf_counter()
        for chain in chains:
            h = synth.make_x(rows, chain[0][1].i, seed=0).double().numpy()
            for j, L in chain:
                f = facs[j]
                if L.method == "lowrank":
                    h = orc.lowrank_forward(h, *f)
                elif L.method == "monarch":
                    h = orc.monarch_forward(h, *f, L.b1, L.b2)
                else:
                    h = orc.blast_forward(h, *f)
        return time.perf_counter() - t0

    rows = 16
    dt = run(rows)
    rows = int(max(16, min(w.n, rows * target_s / max(dt, 1e-3))))
    dt = run(rows)
    # single-thread figure on a smaller sample (report the 1-thread run too)
    cores = orc.num_threads()
    orc.set_num_threads(1)
    rows1 = max(4, rows // max(1, cores) // 4)
    dt1 = run(rows1)
    orc.set_num_threads(0)
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": rows * len(chains) / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} token rows of {w.key} through every layer ({dt:.1f} s fp64 on host)",
            "single_thread_value": rows1 * len(chains) / dt1, "cpu_model": model}


# ------------------------------------------------------------------------------- main bench ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch every step from the host (no CUDA graph)")
    ap.add_argument("--flush", default="write+read", choices=["write+read", "write"],
                    help="L2 flush between timed steps (see L2Flush)")
    args = ap.parse_args()
    w = configs.WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)

    import paper_2512_20861_b200 as blr

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    lib = blr.load()
    stream = torch.cuda.current_stream(dev)

    # ---- inputs (seeded, synthetic; rank offset in the seed so shards differ)
    chains = build_chains(w)
    n = w.n
    facs = {j: [t.to(dev) for t in factors_for(L, j, "cpu")] for j, L in enumerate(w.layers)}
    xs = {}
    for ci, chain in enumerate(chains):
        xs[ci] = synth.make_x(n, chain[0][1].i, seed=rank, layer_id=ci, device=dev)

    def call(L, j, h):
        f = facs[j]
        if L.method == "lowrank":
            return blr.lowrank_matmul(h, *f, out=outs[j], workspace=wss[j])
        if L.method == "monarch":
            return blr.monarch_matmul(h, *f, L.b1, L.b2, out=outs[j], workspace=wss[j])
        return blr.blast_matmul(h, *f, out=outs[j], workspace=wss[j])

    outs, wss = {}, {}
    for j, L in enumerate(w.layers):
        outs[j] = torch.empty((n, L.o), dtype=torch.bfloat16, device=dev)
        if L.method == "lowrank":
            nb = lib.blr_lowrank_workspace_size(n, L.i, L.o, L.r)
        elif L.method == "monarch":
            nb = lib.blr_monarch_workspace_size(n, L.i, L.o, L.b1, L.b2, L.r_blk)
        else:
            nb = lib.blr_blast_workspace_size(n, L.i, L.o, L.b1, L.b2, L.r)
        wss[j] = torch.empty(nb, dtype=torch.uint8, device=dev)

    def step(x_by_chain):
        for ci, chain in enumerate(chains):
            h = x_by_chain[ci]
            for j, L in chain:
                h = call(L, j, h)
        return h

    # ---- launch map: which layer / phase each kernel launch of a step belongs to
    phases = []  # (layer index, phase name) per launch, in launch order
    for ci, chain in enumerate(chains):
        h = xs[ci]
        for j, L in chain:
            h = call(L, j, h)
            nl = lib.blr_last_launch_count()
            names = (["layer"] if nl == 1 else ["proj", "expand"] if nl == 2 else ["s1", "s2", "expand"] if nl == 3
                     else [f"k{i}" for i in range(nl)])
            phases += [(j, nm) for nm in names]
    torch.cuda.synchronize()
    n_launch = len(phases)
    if os.environ.get("BLR_DUMP_PHASES"):
        json.dump([f"{w.layers[j].model}.{w.layers[j].name}.{w.layers[j].method}.{nm}" for j, nm in phases],
                  open(os.environ["BLR_DUMP_PHASES"], "w"))

    # ---- per-launch events (C-ABI profiling hook) and L2 flush buffer
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = L2Flush(max(2 * l2, 256 << 20), dev, args.flush)
    K, W = args.steps, args.warmup
    gev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n_launch)]
    for e in gev:
        e.record(stream)  # forces creation of the underlying cudaEvent_t
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]

    import ctypes
    # ---- the step as a CUDA graph (host launch overhead removed, as under the paper's
    #      torch.compile + CUDA-graph protocol); the per-launch events of the
    #      C-ABI profiling hook are captured as event-record nodes inside the graph.
    # Two graphs of the same step: `graph` (timed; nothing but the kernels, so programmatic
    # dependent launch overlaps each kernel's prologue with its predecessor) and `graph_prof`
    # (per-launch event-record nodes between the kernels, replayed separately after the timed
    # region for the per-phase breakdown -- the events serialise the launches, so its per-launch
    # sum is an upper bound of the step).
    graph = graph_prof = None
    if not args.eager:
        for _ in range(2):
            step(xs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(xs)
        graph_prof = torch.cuda.CUDAGraph()
        arr = (ctypes.c_void_p * (2 * n_launch))(*[e.cuda_event for e in gev])
        with torch.cuda.graph(graph_prof):
            lib.blr_profile_begin(arr, 2 * n_launch)
            step(xs)
            per_replay_prof = lib.blr_profile_end()
        assert per_replay_prof == n_launch
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
            return n_launch
        step(xs)
        return n_launch

    def run_step_profiled():
        if graph_prof is not None:
            graph_prof.replay()
            return
        arr = (ctypes.c_void_p * (2 * n_launch))(*[e.cuda_event for e in gev])
        lib.blr_profile_begin(arr, 2 * n_launch)
        step(xs)
        lib.blr_profile_end()

    for _ in range(W):
        flush()
        run_step()
    torch.cuda.synchronize()

    def timed_region():
        nl = 0
        smp = Sampler(dev.index)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with smp:
            for s in range(K):
                flush()  # L2 flush between timed steps (outside the step events)
                step_ev[s][0].record(stream)
                nl += run_step()
                step_ev[s][1].record(stream)
            torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        return nl, smp

    launches, sampler = timed_region()
    # a run that saw hardware / thermal slowdown is re-measured once (all ranks decide together)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    slow = torch.tensor([1.0 if bad & set(sampler.summary().get("reasons", [])) else 0.0], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(slow, op=torch.distributed.ReduceOp.MAX)
    remeasured = bool(slow.item() > 0)
    if remeasured:
        launches, sampler = timed_region()

    # per-launch breakdown (profiled graph, outside the timed region)
    launch_tot = [0.0] * n_launch
    kp = max(3, min(K, 20))
    prof_step_ms = 0.0
    pe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for s in range(kp):
        flush()
        pe[0].record(stream)
        run_step_profiled()
        pe[1].record(stream)
        torch.cuda.synchronize()
        prof_step_ms += pe[0].elapsed_time(pe[1]) / kp
        for j in range(n_launch):
            launch_tot[j] += gev[2 * j].elapsed_time(gev[2 * j + 1])
    launch_tot = [v * K / kp for v in launch_tot]

    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    t_ms = sum(step_ms) / K
    srt = sorted(step_ms)
    step_stats = {"mean": t_ms, "median": srt[len(srt) // 2], "min": srt[0],
                  "p90": srt[min(len(srt) - 1, int(0.9 * len(srt)))]}
    # warm-L2 figure (no flush between steps), reported separately
    wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(min(K, 10))]
    for a, b in wev:
        a.record(stream)
        run_step()
        b.record(stream)
    torch.cuda.synchronize()
    step_stats["warm_l2_mean"] = sum(a.elapsed_time(b) for a, b in wev) / len(wev)
    launch_ms = [v / K for v in launch_tot]
    if ws > 1:
        from paper_2512_20861_b200 import dist as bdist
        t_ms = bdist.max_over_ranks(t_ms, device=dev)

    tokens_per_step = n * len(chains)
    value = ws * tokens_per_step / (t_ms * 1e-3)

    # ---- per-layer accounting (sum of that layer's launches; phases named per launch)
    peaks = roofline.load_peaks(ROOT)
    per_layer = []
    for j, L in enumerate(w.layers):
        c = roofline.layer_counts(L, n)
        mine = [(nm, launch_ms[x]) for x, (jj, nm) in enumerate(phases) if jj == j]
        ms = sum(v for _, v in mine)
        t_roof = roofline.roofline_time_s(c["flops"], c["bytes"], peaks) * 1e3
        per_layer.append({"layer": f"{L.model}.{L.name}.{L.method}", "ms": ms,
                          "launch_ms": {nm: v for nm, v in mine}, "tflops": c["flops"] / ms * 1e-9,
                          "gbs_alg": c["bytes"] / ms * 1e-6, "roofline_frac": t_roof / ms})

    # ---- dominant kernel roofline (algorithmic bytes/flops per launch)
    jmax = max(range(n_launch), key=lambda x: launch_ms[x])
    Ld = w.layers[phases[jmax][0]]
    phase = phases[jmax][1]
    alg = phase_counts(Ld, n, phase)
    dt_s = launch_ms[jmax] * 1e-3
    bw_t = alg["bytes"] / peaks["hbm_gbs"] / 1e9
    tc_t = alg["flops"] / (peaks["bf16_tflops"] * 1e12)
    bound = "hbm" if bw_t >= tc_t else "tensor"
    if bound == "hbm":
        achieved, peak, unit = alg["bytes"] / dt_s / 1e9, peaks["hbm_gbs"], "GB/s"
    else:
        achieved, peak, unit = alg["flops"] / dt_s / 1e12, peaks["bf16_tflops"], "TFLOP/s"
    traffic = profiled_traffic(Ld, phase, w.key)
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "kernel": f"{phase_kind(Ld, phase)} ({Ld.model}.{Ld.name}.{Ld.method} {phase})",
            "algorithmic_bytes": alg["bytes"], "algorithmic_flops": alg["flops"], "launch_ms": launch_ms[jmax],
            "share_of_step": launch_ms[jmax] / t_ms, "peak_source": peaks.get("source", "measured")}
    io = phase_io_bytes(Ld, n, phase)
    roof["kernel_io_bytes"] = io  # incl. the intermediate this design moves
    roof["kernel_io_gbs"] = io / dt_s / 1e9

    # ---- cuBLAS dense bf16 comparator on the same shapes (X @ W, W reconstructed once)
    dense = None
    if not args.no_dense:
        dense = dense_comparator(w, chains, facs, xs, flush, stream, K, W, dev, not args.eager)

    # ---- end to end through the public API with host buffers (H2D X, D2H Y inside the region)
    e2e = e2e_run(w, chains, facs, xs, flush, stream, min(K, 20), dev)

    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": t_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{w.key}: {w.desc}", "n_tokens_per_gpu": n,
                       "value_def": f"tokens/s; one step = {len(chains)} BLR MLPs/layer chains x {n} tokens",
                       "layers": [f"{L.model}.{L.name}.{L.method}(r={L.r},b={L.b})" for L in w.layers],
                       "l2": flush.describe(),
                       "launch": "eager" if args.eager else "CUDA graph replay of the step (both arms)",
                       "parallelism": f"token-sharded dp{ws}, no data-path collective"},
            "roofline": roof, "per_layer": per_layer, "ms_per_step_stats": step_stats,
            "ms_per_step_with_launch_events": prof_step_ms, "gpu_launches": launches,
            "clocks": dict(sampler.summary(), remeasured=remeasured), "e2e": e2e}
    if dense is not None:
        line["cublas_dense_bf16"] = dense
        line["speedup_vs_cublas"] = dense["ms_per_step"] / t_ms
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def phase_kind(L, phase):
    if phase == "layer":   # one-launch low-rank / Monarch layer (csrc/blr_fused.cuh)
        return "blr_fused_kernel"
    if phase in ("expand", "s1"):
        return "blr_gemm_kernel<KIND_GEMM>"
    if phase == "s2":      # tensor-core S2 unless the intermediate is compensated (r < 128)
        return "blast_s2_mma_kernel" if L.r >= 128 else "blast_s2_kernel"
    return "blr_gemm_kernel<%s>" % {"lowrank": "KIND_GEMM", "monarch": "KIND_MONARCH_PROJ",
                                    "blast": "KIND_BLAST_PROJ"}[L.method]


def phase_counts(L, n, phase):
    """Algorithmic bytes / FLOPs of one phase: proj reads X and the first-stage
    factors (V, and S for BLAST); expand reads U and writes Y.  The intermediate is excluded."""
    B = roofline.BF16
    if phase == "layer":  # fused layer: X, every factor, Y
        p1 = phase_counts(L, n, "proj")
        p3 = phase_counts(L, n, "expand")
        return {"bytes": p1["bytes"] + p3["bytes"], "flops": p1["flops"] + p3["flops"]}
    if phase == "s1":   # BLAST split path: Z_l = X_l V_l
        return {"bytes": B * (n * L.i + L.i * L.r), "flops": 2 * n * L.i * L.r}
    if phase == "s2":   # BLAST split path: S-weighted block sum (reads S only, algorithmically)
        return {"bytes": B * L.b1 * L.b2 * L.r, "flops": 2 * n * L.r * L.b1 * L.b2}
    if phase == "proj":
        if L.method == "lowrank":
            fl, pb = 2 * n * L.i * L.r, L.i * L.r
        elif L.method == "monarch":
            fl, pb = 2 * n * L.i * L.r, L.i * L.r
        else:
            fl, pb = 2 * n * L.i * L.r + 2 * n * L.r * L.b1 * L.b2, L.i * L.r + L.b1 * L.b2 * L.r
        return {"bytes": B * (n * L.i + pb), "flops": fl}
    fl = 2 * n * L.r * L.o
    return {"bytes": B * (L.r * L.o + n * L.o), "flops": fl}


def phase_io_bytes(L, n, phase):
    """Bytes the phase's kernel must move in this implementation: its inputs and outputs
    including the intermediate it reads or writes (the compensated hi|lo intermediate counts
    twice; the BLAST split path's S1 output is fp16).  Context for the fused-roofline figure."""
    B = roofline.BF16
    k3 = L.r if L.method != "monarch" else L.b1 * L.r_blk      # S3 contraction length
    comp = 2 if k3 < 128 else 1
    inter = n * L.r * comp if L.method == "lowrank" else (n * L.b * L.r * comp if L.method == "monarch"
                                                          else n * L.b2 * L.r * comp)
    x_v = n * L.i + L.i * L.r
    if phase == "layer":  # the intermediate stays on chip
        return B * (x_v + L.r * L.o + n * L.o)
    if phase == "s1":     # fp16 Z_l (R13)
        return B * x_v + 2 * n * L.b1 * L.r
    if phase == "s2":
        return 2 * n * L.b1 * L.r + B * (L.b1 * L.b2 * L.r + inter)
    if phase == "proj":
        return B * (x_v + inter + (L.b1 * L.b2 * L.r if L.method == "blast" else 0))
    return B * (inter + L.r * L.o + n * L.o)


def profiled_traffic(L, phase, cfg_key):
    """dram__bytes_read.sum + dram__bytes_write.sum of that launch from the committed
    `ncu --set full` capture (profiles/ncu_traffic_<config>.json, scripts/profile_round.sh)."""
    path = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg_key}.json")
    try:
        d = json.load(open(path))
        return d.get(f"{L.model}.{L.name}.{L.method}.{phase}")
    except (OSError, ValueError):
        return None


def dense_weight(L, f):
    """Dense W (i x o, bf16) for the cuBLAS comparator, reconstructed once in fp32 with torch."""
    if L.method == "lowrank":
        V, U = f
        return (V.float() @ U.float()).to(torch.bfloat16)
    if L.method == "monarch":
        V, U = f
        b1, b2, rp = L.b1, L.b2, L.r_blk
        p, q = L.p, L.q
        Vb = V.float().reshape(b1, rp, b2, p)           # m = rho*b2 + k
        Ub = U.float().reshape(b2, q, b1, rp)           # U[k, c, l*r' + rho]
        W = torch.einsum("lrka,kclr->lakc", Vb, Ub)     # (b1, p, b2, q)
        return W.reshape(b1 * p, b2 * q).to(torch.bfloat16)
    V, S, U = f
    W = torch.einsum("lar,lkr,krc->lakc", V.float(), S.float(), U.float())
    return W.reshape(L.i, L.o).to(torch.bfloat16)


class L2Flush:
    """L2 flush between timed steps, outside the step events.  "write": write a buffer of 2x L2.
    "write+read" (default): the same write, then a read of a second 2x-L2 buffer, so the flush's
    own dirty lines are written back during the flush instead of being evicted -- at HBM write
    cost -- by the first writes of the timed step."""

    def __init__(self, nbytes, dev, mode):
        self.mode = mode
        self.wbuf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.rbuf = torch.ones(nbytes // 4, dtype=torch.float32, device=dev) if mode == "write+read" else None

    def __call__(self):
        self.wbuf.zero_()
        if self.rbuf is not None:
            self.rbuf.sum()

    def describe(self):
        if self.mode == "write+read":
            return "flushed between timed steps (write of 2x L2, then read of another 2x L2), outside the step events"
        return "flushed between timed steps (write of 2x L2), outside the step events"


def dense_comparator(w, chains, facs, xs, flush, stream, K, W, dev, use_graph=True):
    Ws = {j: dense_weight(L, facs[j]) for j, L in enumerate(w.layers)}
    outs = {j: torch.empty((w.n, L.o), dtype=torch.bfloat16, device=dev) for j, L in enumerate(w.layers)}

    def step():
        for ci, chain in enumerate(chains):
            h = xs[ci]
            for j, L in chain:
                h = torch.matmul(h, Ws[j], out=outs[j])

    for _ in range(max(W, 2)):
        flush()
        step()
    torch.cuda.synchronize()
    run = step
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        run = g.replay
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for s in range(K):
        flush()
        evs[s][0].record(stream)
        run()
        evs[s][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / K
    return {"ms_per_step": ms, "tokens_per_s": w.n * len(chains) / (ms * 1e-3),
            "impl": "torch.matmul (cuBLAS/cuBLASLt) bf16" + (", CUDA graph" if use_graph else ", eager")}


def e2e_run(w, chains, facs, xs, flush, stream, K, dev):
    """Same step through the public API with pinned HOST buffers: H2D of each chain's X and
    D2H of each chain's final Y are inside the timed region every step (copy streams overlap
    them with the kernels of the other chains)."""
    xh = {ci: xs[ci].cpu().pin_memory() for ci in xs}
    last = {ci: chain[-1][1] for ci, chain in enumerate(chains)}
    yh = {ci: torch.empty((w.n, last[ci].o), dtype=torch.bfloat16).pin_memory() for ci in xs}
    xd = {ci: torch.empty_like(xs[ci]) for ci in xs}
    h2d = sum(t.numel() * 2 for t in xh.values())
    d2h = sum(t.numel() * 2 for t in yh.values())

    # copies on their own streams so PCIe traffic overlaps the kernels (full duplex): chain c's X
    # lands while chain c-1 computes, chain c's Y drains while chain c+1 computes; the step's end
    # event waits for the last D2H, so every step still carries all of its own copies
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_start = torch.cuda.Event()
    ev_in = {ci: torch.cuda.Event() for ci in xs}
    ev_done = {ci: torch.cuda.Event() for ci in xs}
    ev_out = torch.cuda.Event()

    def one():
        ev_start.record(stream)
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_start)
            for ci in xd:
                xd[ci].copy_(xh[ci], non_blocking=True)
                ev_in[ci].record(s_in)
        for ci, chain in enumerate(chains):
            stream.wait_event(ev_in[ci])
            h = xd[ci]
            for j, L in chain:
                h = step_call(L, j, h)
            ev_done[ci].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[ci])
                h.record_stream(s_out)  # the allocator must not recycle h before the D2H read it
                yh[ci].copy_(h, non_blocking=True)
        ev_out.record(s_out)
        stream.wait_event(ev_out)

    import paper_2512_20861_b200 as blr

    def step_call(L, j, h):
        f = facs[j]
        if L.method == "lowrank":
            return blr.lowrank_matmul(h, *f)
        if L.method == "monarch":
            return blr.monarch_matmul(h, *f, L.b1, L.b2)
        return blr.blast_matmul(h, *f)

    one()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for s in range(K):
        flush()
        evs[s][0].record(stream)
        one()
        evs[s][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / K
    return {"value": w.n * len(chains) / (ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms}



if __name__ == "__main__":
    sys.exit(main())
