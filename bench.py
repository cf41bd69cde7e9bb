#!/usr/bin/env python
"""bench.py -- BLR prefill forward on B200: tokens/s, speedup vs cuBLAS dense bf16, roofline.

Default workload = BASELINE.json configs[3] (C4), the Llama-7B MLP that north_star's target
names: gate/up 4096 -> 11008 then down 11008 -> 4096, BLAST (r = 1488, b = 16, Table 3
L335-342), over batch 8 x seq 8192 = 65,536 tokens.  One *step* = one pass of the whole hot path
(S1, S2, S3 of both layers) over the batch; value = tokens/s through the BLR MLP.  The same line
carries `variants`: the Monarch MLP of Table 3 (C4M, r' = 96) and the >= 2x-compression ranks
(C4X: BLAST r = 1456, Monarch r' = 88), each timed the same way next to cuBLAS.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C4|C4M|C4X|C2|...]

Multi-GPU (one process per GPU; `--gpus N` re-launches itself through torch.distributed.run
when it is not already under torchrun): the workload's tokens are sharded contiguously across
the ranks (strong scaling: 65,536 tokens in total, 8,192 per GPU at N = 8), factors replicated,
no collective on the data path; the step time is the max over ranks and
value = all tokens / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(nproc: int) -> int:
    """`--gpus N` outside torchrun: start N ranks of this script (one per GPU) and exit with
    their status.  Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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
    """nvml clock / throttle-reason sampler running during a timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}

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

    def bad(self):
        return bool(self.BAD & set(self.summary().get("reasons", [])))


def _any_rank(flag: bool, ws: int, dev) -> bool:
    t = torch.tensor([1.0 if flag else 0.0], device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return bool(t.item() > 0)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------- reference ----
def oracle_step_fn(w, rows, seed=0):
    """One step of the workload through the fp64 oracle on `rows` token rows."""
    import numpy as np

    from oracle import oracle as orc
    chains = build_chains(w)
    facs = {j: [t.float().numpy().astype(np.float64) for t in factors_for(L, j, "cpu")] for j, L in enumerate(w.layers)}
    xs = {ci: synth.make_x(rows, chain[0][1].i, seed=seed, layer_id=ci).double().numpy()
          for ci, chain in enumerate(chains)}

    def step():
        for ci, chain in enumerate(chains):
            h = xs[ci]
            for j, L in chain:
                f = facs[j]
                if L.method == "lowrank":
                    h = orc.lowrank_forward(h, *f)
                elif L.method == "monarch":
                    h = orc.monarch_forward(h, *f, L.b1, L.b2)
                else:
                    h = orc.blast_forward(h, *f)
        return h

    return step, len(chains)


def run_reference(args, w):
    """--impl reference: the fp64 oracle as it stands, on this host's cores, on a bounded sample
    of the same workload (each step = `rows` token rows through every layer of the workload).
    Under torchrun only rank 0 runs; the other ranks exit without work."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    orc.set_num_threads(host_cores())  # torchrun sets OMP_NUM_THREADS=1 for every rank
    rows = args.ref_rows
    step, nchains = oracle_step_fn(w, rows)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = rows * nchains / dt
    cores = orc.num_threads()
    sample = f"{rows} token rows of {w.key} through all {len(w.layers)} layers per step (fp64 oracle)"
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{w.key}: {w.desc}", "rows_per_step": rows},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(w, target_s=10.0):
    """Time the oracle (as it stands) on a bounded token sample of the same workload."""
    from oracle import oracle as orc
    orc.set_num_threads(host_cores())

    def run(rows):
        step, nch = oracle_step_fn(w, rows)
        t0 = time.perf_counter()
        step()
        return time.perf_counter() - t0, nch

    rows = 16
    dt, nch = run(rows)
    rows = int(max(16, min(w.n, rows * target_s / max(dt, 1e-3))))
    dt, nch = run(rows)
    # single-thread figure on a smaller sample (report the 1-thread run too)
    cores = orc.num_threads()
    orc.set_num_threads(1)
    rows1 = max(4, rows // max(1, cores) // 4)
    dt1, _ = run(rows1)
    orc.set_num_threads(host_cores())
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": rows * nch / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} token rows of {w.key} through every layer ({dt:.1f} s fp64 on host)",
            "single_thread_value": rows1 * nch / dt1, "cpu_model": model}


# ------------------------------------------------------------------------------- the arm ------
class Arm:
    """One workload on this rank's token shard: inputs, outputs, workspaces and the step."""

    def __init__(self, w, n, dev, seed):
        import paper_2512_20861_b200 as blr
        self.blr = blr
        self.lib = blr.load()
        self.w, self.n, self.dev = w, n, dev
        self.chains = build_chains(w)
        self.facs = {j: [t.to(dev) for t in factors_for(L, j, "cpu")] for j, L in enumerate(w.layers)}
        # K-major BLAST storage (workload C4K): re-laid-out once here, outside every timed region
        self.kfacs = {}
        if getattr(w, "kmajor", False):
            for j, L in enumerate(w.layers):
                if L.method == "blast":
                    V, S, U = self.facs[j]
                    Vt, Ut = blr.blast_kmajor_factors(V, U)
                    self.kfacs[j] = [Vt, S, Ut]
        self.xs = {ci: synth.make_x(n, chain[0][1].i, seed=seed, layer_id=ci, device=dev)
                   for ci, chain in enumerate(self.chains)}
        self.outs, self.wss = {}, {}
        for j, L in enumerate(w.layers):
            self.outs[j] = torch.empty((n, L.o), dtype=torch.bfloat16, device=dev)
            if L.method == "lowrank":
                nb = self.lib.blr_lowrank_workspace_size(n, L.i, L.o, L.r)
            elif L.method == "monarch":
                nb = self.lib.blr_monarch_workspace_size(n, L.i, L.o, L.b1, L.b2, L.r_blk)
            else:
                nb = self.lib.blr_blast_workspace_size(n, L.i, L.o, L.b1, L.b2, L.r)
            self.wss[j] = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)

    def call(self, L, j, h, out=None, ws=None):
        f = self.facs[j]
        blr = self.blr
        if L.method == "lowrank":
            return blr.lowrank_matmul(h, *f, out=out, workspace=ws)
        if L.method == "monarch":
            return blr.monarch_matmul(h, *f, L.b1, L.b2, out=out, workspace=ws)
        if j in self.kfacs:
            return blr.blast_matmul(h, *self.kfacs[j], out=out, workspace=ws, kmajor=True)
        return blr.blast_matmul(h, *f, out=out, workspace=ws, fp8_intermediate=self.w.fp8z)

    def step(self):
        for ci, chain in enumerate(self.chains):
            h = self.xs[ci]
            for j, L in chain:
                h = self.call(L, j, h, self.outs[j], self.wss[j])
        return h

    def phases(self):
        """(layer index, phase name) of every kernel launch of one step, in launch order."""
        ph = []
        for ci, chain in enumerate(self.chains):
            h = self.xs[ci]
            for j, L in chain:
                h = self.call(L, j, h, self.outs[j], self.wss[j])
                nl = self.lib.blr_last_launch_count()
                names = (["layer"] if nl == 1 else ["proj", "expand"] if nl == 2 else ["s1", "s2", "expand"]
                         if nl == 3 else [f"k{i}" for i in range(nl)])
                ph += [(j, nm) for nm in names]
        torch.cuda.synchronize()
        return ph


def graph_of(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g


def timed(run, flush, stream, K, dev, ws):
    """K steps, L2 flushed between them (outside the events), bracketed by barrier + sync;
    clocks sampled during the region; re-measured once if any rank saw hw/thermal slowdown."""
    def region():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        smp = Sampler(dev.index)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with smp:
            for s in range(K):
                flush()
                evs[s][0].record(stream)
                run()
                evs[s][1].record(stream)
            torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        return [a.elapsed_time(b) for a, b in evs], smp

    ms, smp = region()
    remeasured = _any_rank(smp.bad(), ws, dev)
    if remeasured:
        ms, smp = region()
    return ms, dict(smp.summary(), remeasured=remeasured)


def stats(ms):
    srt = sorted(ms)
    return {"mean": sum(ms) / len(ms), "median": srt[len(srt) // 2], "min": srt[0],
            "p90": srt[min(len(srt) - 1, int(0.9 * len(srt)))]}


def dense_comparator(arm, flush, stream, K, W, dev, ws, use_graph=True):
    """cuBLAS dense bf16 on the same shapes: X @ W with W reconstructed once (torch.matmul)."""
    w = arm.w
    Ws = {j: dense_weight(L, arm.facs[j]) for j, L in enumerate(w.layers)}
    outs = {j: torch.empty((arm.n, L.o), dtype=torch.bfloat16, device=dev) for j, L in enumerate(w.layers)}

    def step():
        for ci, chain in enumerate(arm.chains):
            h = arm.xs[ci]
            for j, L in chain:
                h = torch.matmul(h, Ws[j], out=outs[j])

    for _ in range(max(W, 2)):
        flush()
        step()
    torch.cuda.synchronize()
    run = graph_of(step).replay if use_graph else step
    ms, clocks = timed(run, flush, stream, K, dev, ws)
    t = sum(ms) / K
    if ws > 1:
        from paper_2512_20861_b200 import dist as bdist
        t = bdist.max_over_ranks(t, device=dev)
    del Ws, outs
    return {"ms_per_step": t, "tokens_per_s": ws * arm.n * len(arm.chains) / (t * 1e-3),
            "impl": "torch.matmul (cuBLAS/cuBLASLt) bf16" + (", CUDA graph" if use_graph else ", eager"),
            "clocks": clocks}


def e2e_run(arm, flush, stream, K, dev, ws):
    """The step end to end through the public API with pinned HOST buffers: H2D of the step's X
    and D2H of its Y are inside the timed region every step.  The tokens are processed in chunks
    so PCIe (full duplex) overlaps the kernels: chunk c's X lands while chunk c-1 computes and
    chunk c's Y drains while chunk c+1 computes; the step's end event waits for the last D2H."""
    blr = arm.blr
    # 16 chunks of >= 2048 tokens (C4 e2e 12.95 -> 12.45 ms against 8 chunks; 32: 12.68 ms)
    nch = 16 if arm.n >= 16 * 2048 else 8 if arm.n >= 8 * 2048 else 1
    if os.environ.get("BLR_E2E_CHUNKS"):  # A/B of the pipeline depth
        nch = max(1, min(int(os.environ["BLR_E2E_CHUNKS"]), arm.n // 256))
    bounds = [(c * arm.n // nch, (c + 1) * arm.n // nch) for c in range(nch)]
    xh = {ci: arm.xs[ci].cpu().pin_memory() for ci in arm.xs}
    last = {ci: chain[-1][1] for ci, chain in enumerate(arm.chains)}
    yh = {ci: torch.empty((arm.n, last[ci].o), dtype=torch.bfloat16).pin_memory() for ci in arm.xs}
    xd = {ci: torch.empty_like(arm.xs[ci]) for ci in arm.xs}
    yd = {ci: torch.empty((arm.n, last[ci].o), dtype=torch.bfloat16, device=dev) for ci in arm.xs}
    h2d = sum(t.numel() * 2 for t in xh.values())
    d2h = sum(t.numel() * 2 for t in yh.values())
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_start, ev_out = torch.cuda.Event(), torch.cuda.Event()
    ev_in = {(ci, c): torch.cuda.Event() for ci in arm.xs for c in range(nch)}
    ev_done = {(ci, c): torch.cuda.Event() for ci in arm.xs for c in range(nch)}

    def fwd(L, j, h, out=None):
        f = arm.facs[j]
        if L.method == "lowrank":
            return blr.lowrank_matmul(h, *f, out=out)
        if L.method == "monarch":
            return blr.monarch_matmul(h, *f, L.b1, L.b2, out=out)
        if j in arm.kfacs:
            return blr.blast_matmul(h, *arm.kfacs[j], out=out, kmajor=True)
        return blr.blast_matmul(h, *f, out=out, fp8_intermediate=arm.w.fp8z)

    def one():
        ev_start.record(stream)
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_start)
            for ci in xd:
                for c, (lo, hi) in enumerate(bounds):
                    xd[ci][lo:hi].copy_(xh[ci][lo:hi], non_blocking=True)
                    ev_in[(ci, c)].record(s_in)
        for ci, chain in enumerate(arm.chains):
            for c, (lo, hi) in enumerate(bounds):
                stream.wait_event(ev_in[(ci, c)])
                h = xd[ci][lo:hi]
                for jj, (j, L) in enumerate(chain):
                    h = fwd(L, j, h, out=yd[ci][lo:hi] if jj == len(chain) - 1 else None)
                ev_done[(ci, c)].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_done[(ci, c)])
                    yh[ci][lo:hi].copy_(yd[ci][lo:hi], non_blocking=True)
        ev_out.record(s_out)
        stream.wait_event(ev_out)

    one()
    torch.cuda.synchronize()
    ms, _ = timed(one, flush, stream, K, dev, ws)
    t = sum(ms) / K
    if ws > 1:
        from paper_2512_20861_b200 import dist as bdist
        t = bdist.max_over_ranks(t, device=dev)
    return {"value": ws * arm.n * len(arm.chains) / (t * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": t, "chunks": nch,
            "how": "public API (blr.*_matmul) on pinned host X/Y, H2D + kernels + D2H per step, "
                   f"{nch} token chunks pipelined over copy streams"}


def measure(w, n, dev, stream, args, ws, rank, flush, full=True):
    """Time workload `w` on this rank's n tokens: graph-replayed step (the headline), per-launch
    breakdown, dominant-kernel roofline, cuBLAS comparator and (full) the e2e run."""
    arm = Arm(w, n, dev, seed=rank)
    lib = arm.lib
    ph = arm.phases()
    n_launch = len(ph)
    if os.environ.get("BLR_DUMP_PHASES"):  # launch labels for the ncu summaries (scripts/profile_summary.py)
        json.dump([f"{w.layers[j].model}.{w.layers[j].name}.{w.layers[j].method}.{nm}" for j, nm in ph],
                  open(os.environ["BLR_DUMP_PHASES"], "w"))
    K, W = args.steps, args.warmup
    graph = None if args.eager else graph_of(arm.step)
    run = graph.replay if graph is not None else arm.step
    for _ in range(W):
        flush()
        run()
    torch.cuda.synchronize()
    step_ms, clocks = timed(run, flush, stream, K, dev, ws)
    t_ms = sum(step_ms) / K
    st = stats(step_ms)
    # warm-L2 figure (no flush between steps), reported separately
    wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(min(K, 10))]
    for a, b in wev:
        a.record(stream)
        run()
        b.record(stream)
    torch.cuda.synchronize()
    st["warm_l2_mean"] = sum(a.elapsed_time(b) for a, b in wev) / len(wev)

    # per-launch breakdown: a second graph of the step with the C-ABI hook's event-record nodes
    # (the events serialise the launches: upper bounds), replayed after the timed region
    import ctypes
    gev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n_launch)]
    for e in gev:
        e.record(stream)
    arr = (ctypes.c_void_p * (2 * n_launch))(*[e.cuda_event for e in gev])

    def prof_step():
        lib.blr_profile_begin(arr, 2 * n_launch)
        arm.step()
        got = lib.blr_profile_end()
        assert got == n_launch, (got, n_launch)

    prun = graph_of(prof_step).replay if not args.eager else prof_step
    kp = max(3, min(K, 10))
    launch_ms = [0.0] * n_launch
    prof_step_ms = 0.0
    pe = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for _ in range(kp):
        flush()
        pe[0].record(stream)
        prun()
        pe[1].record(stream)
        torch.cuda.synchronize()
        prof_step_ms += pe[0].elapsed_time(pe[1]) / kp
        for j in range(n_launch):
            launch_ms[j] += gev[2 * j].elapsed_time(gev[2 * j + 1]) / kp
    if ws > 1:
        from paper_2512_20861_b200 import dist as bdist
        t_ms = bdist.max_over_ranks(t_ms, device=dev)

    peaks = roofline.load_peaks(ROOT)
    per_layer = []
    for j, L in enumerate(w.layers):
        c = roofline.layer_counts(L, n)
        mine = [(nm, launch_ms[x]) for x, (jj, nm) in enumerate(ph) if jj == j]
        ms = sum(v for _, v in mine)
        t_roof = roofline.roofline_time_s(c["flops"], c["bytes"], peaks) * 1e3
        per_layer.append({"layer": f"{L.model}.{L.name}.{L.method}(r={L.r},b={L.b})", "ms": ms,
                          "launch_ms": {nm: v for nm, v in mine}, "tflops": c["flops"] / ms * 1e-9,
                          "gbs_alg": c["bytes"] / ms * 1e-6, "roofline_frac": t_roof / ms,
                          "roofline_ms": t_roof})
    # step roofline: all layers' FLOPs / bytes against the peaks
    fl = sum(roofline.layer_counts(L, n)["flops"] for L in w.layers)
    by = sum(roofline.layer_counts(L, n)["bytes"] for L in w.layers)
    step_roof_ms = roofline.roofline_time_s(fl, by, peaks) * 1e3

    # dominant kernel (algorithmic bytes / FLOPs per launch)
    jmax = max(range(n_launch), key=lambda x: launch_ms[x])
    Ld = w.layers[ph[jmax][0]]
    phase = ph[jmax][1]
    alg = phase_counts(Ld, n, phase)
    dt_s = launch_ms[jmax] * 1e-3
    bw_t = alg["bytes"] / peaks["hbm_gbs"] / 1e9
    tc_t = alg["flops"] / (peaks["bf16_tflops"] * 1e12)
    bound = "hbm" if bw_t >= tc_t else "tensor"
    # the contract's denominator: the burst figure for a kernel timed alone, the sustained one for
    # a kernel timed inside a long step (the dominant launch is timed inside the graph of the whole
    # step, which runs for milliseconds at the power-capped steady-state clock)
    long_step = t_ms >= 1.0 and bool(peaks.get("bf16_tflops_sustained"))
    if bound == "hbm":
        achieved, peak, unit = alg["bytes"] / dt_s / 1e9, peaks["hbm_gbs"], "GB/s"
        note = "copy HBM GB/s from MEASURED_PEAKS.json"
    else:
        achieved, unit = alg["flops"] / dt_s / 1e12, "TFLOP/s"
        peak = peaks["bf16_tflops_sustained"] if long_step else peaks["bf16_tflops"]
        note = (f"sustained bf16 TF/s from MEASURED_PEAKS.json (kernel timed inside a {t_ms:.1f}-ms step)"
                if long_step else "burst bf16 TF/s from MEASURED_PEAKS.json (short step)")
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": profiled_traffic(Ld, phase, w.key),
            "kernel": f"{phase_kind(Ld, phase)} ({Ld.model}.{Ld.name}.{Ld.method} {phase})",
            "algorithmic_bytes": alg["bytes"], "algorithmic_flops": alg["flops"], "launch_ms": launch_ms[jmax],
            "share_of_step": launch_ms[jmax] / t_ms, "peak_source": peaks.get("source", "measured"),
            "peak_note": note,
            "kernel_io_bytes": phase_io_bytes(Ld, n, phase)}
    roof["kernel_io_gbs"] = roof["kernel_io_bytes"] / dt_s / 1e9
    if bound == "tensor":
        roof["frac_of_burst"] = achieved / peaks["bf16_tflops"]

    dense = None if args.no_dense else dense_comparator(arm, flush, stream, K, W, dev, ws, not args.eager)
    e2e = e2e_run(arm, flush, stream, min(K, 10), dev, ws) if full else None
    tokens = ws * n * len(arm.chains)
    res = {"t_ms": t_ms, "value": tokens / (t_ms * 1e-3), "stats": st, "clocks": clocks, "per_layer": per_layer,
           "roofline": roof, "dense": dense, "e2e": e2e, "launches_per_step": n_launch,
           "prof_step_ms": prof_step_ms, "step_roofline_ms": step_roof_ms, "n_chains": len(arm.chains)}
    del arm, graph
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------------------- main bench ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--ref-rows", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--variants", default="C2,C4M,C4X,C4F8,C4K", help="comma-separated extra workloads (N = 1 only)")
    ap.add_argument("--eager", action="store_true", help="launch every step from the host (no CUDA graph)")
    ap.add_argument("--flush", default="write+read", choices=["write+read", "write"],
                    help="L2 flush between timed steps (see L2Flush)")
    ap.add_argument("--dry-run", action="store_true",
                    help="rank/shard plumbing only (gloo, no GPU work): prints n_gpus and the shards")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    w = configs.WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)

    from paper_2512_20861_b200 import dist as bdist
    lo, hi = bdist.shard_rows(w.n, rank, ws)
    if args.dry_run:
        if ws > 1:
            torch.distributed.init_process_group("gloo")
        shards = [bdist.shard_rows(w.n, r, ws) for r in range(ws)]
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": ws, "dry_run": True,
                              "scaling": "strong",
                              "config": {"workload": f"{w.key}: {w.desc}", "n_tokens_total": w.n,
                                         "shards": shards}}), flush=True)
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    if ws > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    n = hi - lo
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = L2Flush(max(2 * l2, 256 << 20), dev, args.flush)

    r = measure(w, n, dev, stream, args, ws, rank, flush, full=True)
    variants = []
    if ws == 1 and not args.no_variants:
        for key in [k for k in args.variants.split(",") if k and k != w.key]:
            wv = configs.WORKLOADS[key]
            v = measure(wv, wv.n, dev, stream, args, ws, rank, flush, full=False)
            ent = {"workload": f"{wv.key}: {wv.desc}", "value": v["value"], "unit": "tokens/s",
                   "ms_per_step": v["t_ms"], "clocks": v["clocks"],
                   "per_layer": [{k2: pl[k2] for k2 in ("layer", "ms", "launch_ms", "tflops", "roofline_frac")}
                                 for pl in v["per_layer"]],
                   "roofline": {k2: v["roofline"][k2] for k2 in ("bound", "achieved", "peak", "unit", "frac", "kernel")},
                   "step_roofline_ms": v["step_roofline_ms"]}
            if v["dense"] is not None:
                ent["cublas_dense_bf16_ms"] = v["dense"]["ms_per_step"]
                ent["speedup_vs_cublas"] = v["dense"]["ms_per_step"] / v["t_ms"]
            variants.append(ent)

    t_ms = r["t_ms"]
    line = {"metric": METRIC, "value": r["value"], "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{w.key}: {w.desc}", "n_tokens_total": w.n, "n_tokens_per_gpu": n,
                       "value_def": f"tokens/s through the BLR MLP; one step = {r['n_chains']} chain(s) x {w.n} tokens"
                                    + (f", token rows sharded contiguously over {ws} GPUs" if ws > 1 else ""),
                       "layers": [f"{L.model}.{L.name}.{L.method}(r={L.r},b={L.b})" for L in w.layers],
                       "l2": flush.describe(),
                       "launch": "eager" if args.eager else "CUDA graph replay of the step (both arms)",
                       "parallelism": f"token-sharded dp{ws}, factors replicated, no data-path collective"},
            "roofline": r["roofline"], "step_roofline_ms": r["step_roofline_ms"],
            "step_roofline_frac": r["step_roofline_ms"] / t_ms,
            "per_layer": r["per_layer"], "ms_per_step_stats": r["stats"],
            "ms_per_step_with_launch_events": r["prof_step_ms"],
            "gpu_launches": r["launches_per_step"] * args.steps, "launches_per_step": r["launches_per_step"],
            "clocks": r["clocks"], "e2e": r["e2e"]}
    if r["dense"] is not None:
        line["cublas_dense_bf16"] = r["dense"]
        line["speedup_vs_cublas"] = r["dense"]["ms_per_step"] / t_ms
    if variants:
        line["variants"] = variants
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
    `ncu --set full` capture of the same build (profiles/ncu_traffic_<config>.json)."""
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


if __name__ == "__main__":
    sys.exit(main())
