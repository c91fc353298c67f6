#!/usr/bin/env python
"""bench.py -- AFN-PCG on B200 (arXiv 2304.05460 hot path), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl afn|reference]

Workload (BASELINE.json configs[1], "C2"): n = 16384 points uniform in a 3-D
cube of edge 10*(16384/1000)^(1/3), Gaussian kernel, l swept over
{0.1, 0.5, 1, 2, 5, 10}, mu = 1e-4, b ~ N(0,1) (seed 0), adaptive k <= 2000
(Algorithm 1), FSAI 100 nnz/row, PCG tol 1e-4.  One *step* = the whole hot
path (all SURVEY.md 8(a) rows: Alg. 1, FPS, permutation, Cholesky, W, kNN,
FSAI, PCG with kernel matvec + AFN apply) for every l of the sweep.

Metric: AFN-PCG seconds per solve (build + PCG, device time from CUDA events,
lower is better) with the kernel-matvec Gpairs/s and the FP64 roofline
fraction of the dominant kernel beside it.  With N GPUs the six sweep problems
are split across ranks (independent problems, no data-path collective); the
job time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AFN-PCG solve sec & kernel-matvec Gpairs/s (fp64) vs FP64 roofline"
# FP64 peak derived from the guide's unit counts:
# 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak()
# kernel matvec: algorithmic flops per pair for d = 3: 3d + 19
KMV_FLOPS_PER_PAIR = lambda d: 3 * d + 19  # noqa: E731


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="afn", choices=["afn", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="sweep", choices=["sweep", "dist"],
                    help="sweep: the C2 l-sweep, problems split over ranks (default); "
                         "dist: every rank solves the same problem row-sharded (SURVEY 8(e))")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def fsai_flops(N2: int, k: int, w: int) -> float:
    """Algorithmic flops of the FSAI row kernel: lower-triangle Gram
    (wp(wp+1)/2 dot products of length k, FMA = 2) + Cholesky wp^3/3 + solve wp^2."""
    tot = 0.0
    for wp in range(1, min(w, N2) + 1):  # rows 0..w-2 have wp = i+1
        cnt = 1 if wp < w else max(0, N2 - (w - 1))
        tot += cnt * (wp * (wp + 1) * k + wp ** 3 / 3.0 + wp * wp)
    return tot


def oracle_solve_estimate(X, b, cfg, l, gpu_iters=None, frac=16, threads=None):
    """Oracle (CPU) seconds for one AFN-PCG solve of this workload, from a
    bounded sample: Alg. 1, FPS and the landmark block run in full; kNN and
    FSAI on every `frac`-th non-landmark row, the kernel matvec on every
    `frac`-th row (both scaled by frac); the apply in full.  PCG iterations
    from the oracle's own Alg. 1 k and, if given, the GPU's iteration count."""
    import numpy as np
    import scipy.linalg as sla
    import oracle as O
    t = {}
    t0 = time.perf_counter()
    a1 = O.alg1(X, l)
    t["alg1"] = time.perf_counter() - t0
    k = min(cfg.k_cap, max(1, a1["khat"]), len(X))
    t0 = time.perf_counter()
    idx, _ = O.fps(X, k, 0)
    t["fps"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    n = len(X)
    mask = np.ones(n, bool)
    mask[idx] = False
    perm = np.concatenate([idx, np.nonzero(mask)[0]])
    Xp = X[perm]
    X1, X2 = Xp[:k], Xp[k:]
    L = np.linalg.cholesky(O.kernel_block(X1, X1, l) + cfg.mu * np.eye(k))
    K12 = O.kernel_block(X1, X2, l)
    V = sla.solve_triangular(L, K12, lower=True)
    t["chol_V"] = time.perf_counter() - t0
    N2 = n - k
    rows = np.arange(0, N2, frac)
    t0 = time.perf_counter()
    pat = [O.knn_row(X2, int(i), cfg.w) for i in rows]
    t["knn"] = (time.perf_counter() - t0) * frac
    rp = np.zeros(len(rows) + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(p) for p in pat])
    col = np.concatenate(pat)
    t0 = time.perf_counter()
    O.fsai_rows(lambda J: O.kernel_block(X2[J], X2[J], l) + cfg.mu * np.eye(len(J))
                - V[:, J].T @ V[:, J], rp, col)
    t["fsai"] = (time.perf_counter() - t0) * frac
    v = np.asarray(b, dtype=np.float64)
    t0 = time.perf_counter()
    O.kmv_rows(Xp, l, cfg.mu, v, np.arange(0, n, frac))
    t_kmv = (time.perf_counter() - t0) * frac
    import scipy.sparse as sp
    G = sp.identity(N2, format="csr")
    B = dict(k=k, L=L, K12=K12, G=G)
    t0 = time.perf_counter()
    O.apply_afn(B, v)
    t_apply = time.perf_counter() - t0
    its = gpu_iters if gpu_iters is not None else 10
    t["pcg"] = (its + 1) * t_kmv + (its + 1) * t_apply
    total = sum(t.values())
    return total, t, k


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import CONFIGS, gen_problem
    cfg = CONFIGS[args.config]
    X, b = gen_problem(cfg)
    ls = cfg.ls
    for s in range(args.warmup):
        oracle_solve_estimate(X, b, cfg, ls[s % len(ls)])
    vals = []
    t0 = time.perf_counter()
    for s in range(args.steps):
        v, parts, k = oracle_solve_estimate(X, b, cfg, ls[s % len(ls)])
        vals.append(v)
    wall = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    sample = (f"{args.config}: per step one sweep value of l (cycling {list(ls)}); Alg.1, FPS, "
              f"Cholesky and V=L^-1 K12 in full; kNN, FSAI and kernel-matvec rows 1/16 sampled "
              f"and scaled x16; PCG iterations assumed 10")
    line = {"metric": METRIC, "value": value, "unit": "s/solve", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "n": cfg.n, "d": cfg.d, "ls": list(ls),
                       "mu": cfg.mu, "k_cap": cfg.k_cap, "w": cfg.w, "tol": cfg.tol},
            "cpu_baseline": {"value": value, "unit": "s/solve", "cores": cpu_cores(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "s/solve", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_dist(args):
    """--mode dist: one AFN-PCG problem per step, rows sharded over all ranks
    (one GPU each, NCCL all-gathers; include/afn.h "Multi-GPU").  Strong
    scaling: the total work is fixed as N grows."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import __graft_entry__ as ge
    if local == 0:  # (one builder per node: ranks must not write the same objects)
        ge._build_module().build()
    if dist:
        dist.barrier()
    import paper_2304_05460_b200 as afn
    from synth import CONFIGS, gen_problem
    cfg = CONFIGS[args.config]
    X, b = gen_problem(cfg)
    Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
    comm = afn.Comm.from_process_group(dist) if dist else None
    recs = []

    def step(record=False):
        for l in cfg.ls:
            h = afn.afn_build(Xd, afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True),
                              comm=comm)
            a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
            if record:
                recs.append((l, h.info(), rep))
            h.close()

    for _ in range(max(3, args.warmup)):
        step()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = afn.launch_count()
    with sampler:
        for s in range(args.steps):
            evs[s][0].record(stream)
            step(record=True)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    launches = afn.launch_count() - l0
    if dist:
        dist.barrier()
    t = torch.tensor([sum(a.elapsed_time(c) for a, c in evs)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    job_ms = float(t.item())
    nsolve = args.steps * len(cfg.ls)
    mv_ms = sum(r["matvec_ms"] for _, _, r in recs)
    its = sum(r["iterations"] for _, _, r in recs)
    if rank == 0:
        inf, rep = recs[0][1], recs[0][2]
        line = {"metric": METRIC, "value": job_ms / 1e3 / nsolve, "unit": "s/solve", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": job_ms / args.steps,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, BASELINE configs)",
                "config": {"workload": args.config, "n": cfg.n, "d": cfg.d, "ls": list(cfg.ls),
                           "mu": cfg.mu, "k_cap": cfg.k_cap, "w": cfg.w, "tol": cfg.tol,
                           "parallelism": f"rows sharded over {world} rank(s), points replicated",
                           "l2": "inputs and working set (W) larger than L2"},
                "kmv_gpairs_per_s": float(cfg.n) ** 2 * its / (mv_ms * 1e-3) / 1e9 if mv_ms > 0 else None,
                "per_solve": {"k": inf["k"], "khat": inf["khat"], "iters": rep["iterations"],
                              "setup_ms": inf["ms_total"], "pcg_ms": rep["solve_ms"],
                              "matvec_ms": rep["matvec_ms"], "apply_ms": rep["apply_ms"],
                              "comm_ms": rep["comm_ms"], "relres_true": rep["relres_true"]},
                "gpu_launches": launches, "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "dist":
        if args.config == "C2":
            args.config = "C3"
        return run_dist(args)

    import numpy as np
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    import __graft_entry__ as ge
    if local == 0:  # (one builder per node: ranks must not write the same objects)
        ge._build_module().build()
    if dist:
        dist.barrier()
    import paper_2304_05460_b200 as afn
    from synth import CONFIGS, gen_problem

    cfg = CONFIGS[args.config]
    X, b = gen_problem(cfg)
    Xd = torch.from_numpy(X).to(dev)
    bd = torch.from_numpy(b).to(dev)
    my_ls = list(cfg.ls[rank::world])

    def params(l):
        return afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True)

    records = []

    def step(record=False):
        for l in my_ls:
            h = afn.afn_build(Xd, params(l))
            a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
            if record:
                records.append((l, h.info(), rep))
            h.close()

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = afn.launch_count()
    afn.kernel_timers(reset=True, enable=True)
    with sampler:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the event pair)
            evs[s][0].record(stream)
            step(record=True)
            evs[s][1].record(stream)
        torch.cuda.synchronize()
    launches = afn.launch_count() - l0
    kt = afn.kernel_timers(enable=False)
    if dist:
        dist.barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    job_ms = float(t.item())
    n_solves = len(cfg.ls)
    value_s = job_ms / 1e3 / (args.steps * n_solves)

    # ---- per-kernel accounting (CUDA events inside the library, timed region)
    n = cfg.n
    kmv_ms = sum(r["matvec_ms"] for _, _, r in records)
    kmv_calls = sum(r["iterations"] for _, _, r in records)
    per_l = {}
    for l, inf, rep in records[: len(my_ls)]:
        per_l[str(l)] = {"khat": inf["khat"], "k": inf["k"], "iters": rep["iterations"],
                         "setup_ms": inf["ms_total"], "pcg_ms": rep["solve_ms"],
                         "relres_true": rep["relres_true"]}
    kmv_gpairs = (float(n) * n * kmv_calls) / (kmv_ms * 1e-3) / 1e9 if kmv_ms > 0 else None
    shares = {"fsai_phase": sum(i["ms_fsai_rows"] for _, i, _ in records), "kmv_kernel": kmv_ms,
              "fps": sum(i["ms_fps"] for _, i, _ in records),
              "W": sum(i["ms_trsm"] for _, i, _ in records),
              "chol_Linv": sum(i["ms_chol"] for _, i, _ in records),
              "alg1": sum(i["ms_alg1"] for _, i, _ in records),
              "knn": sum(i["ms_knn"] for _, i, _ in records),
              "apply": sum(r["apply_ms"] for _, _, r in records)}
    single = {k: v for k, v in kt.items() if k not in ("potrf", "alg1") and v["count"] > 0}
    dom = max(single, key=lambda k: single[k]["ms"]) if single else None
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path) and dom:
        try:
            traffic = json.load(open(tr_path)).get(dom)
        except Exception:
            traffic = None

    def roof(name):
        v = kt.get(name)
        if not v or v["count"] <= 0 or v["ms"] <= 0:
            return None
        per_ms = v["ms"] / v["count"]
        out = {"kernel": name, "launches": v["count"], "ms_per_launch": per_ms,
               "share_of_step": v["ms"] / total_ms if total_ms > 0 else None, "traffic": None}
        if name == "apply":
            ach = v["work"] / (v["ms"] * 1e-3) / 1e9
            out.update({"bound": "hbm", "achieved": ach, "peak": HBM_PEAK_GBS, "unit": "GB/s",
                        "frac": ach / HBM_PEAK_GBS, "bytes_per_launch": v["work"] / v["count"],
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"})
        elif v["work"] > 0:
            ach = v["work"] / (v["ms"] * 1e-3) / 1e12
            out.update({"bound": "alu", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": ach / FP64_PEAK_TFLOPS, "flops_per_launch": v["work"] / v["count"],
                        "peak_source": "guide unit counts: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz"})
        else:
            out.update({"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None})
        return out

    roofline = roof(dom) if dom else None
    if roofline is not None:
        roofline["traffic"] = traffic
    r_kmv = roof("kmv_kernel")
    kernel_ms = {k: round(v["ms"], 3) for k, v in kt.items() if v["count"] > 0}

    # ---- e2e: host buffers through the C ABI (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        bh = torch.from_numpy(b).pin_memory()
        E = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
        if my_ls:  # (ranks past the sweep's length have no problem: N > 6 GPUs)
            afn.afn_solve_host(Xh.numpy(), bh.numpy(), params(my_ls[0]), tol=cfg.tol)  # warm
        for s in range(args.steps):
            flush.zero_()
            E[s][0].record(stream)
            for l in my_ls:
                afn.afn_solve_host(Xh.numpy(), bh.numpy(), params(l), tol=cfg.tol, maxit=cfg.maxit)
            E[s][1].record(stream)
        torch.cuda.synchronize()
        e_ms = sum(a.elapsed_time(c) for a, c in E)
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": float(te.item()) / 1e3 / (args.steps * n_solves), "unit": "s/solve",
               "h2d_bytes_per_step": n_solves * (X.nbytes + b.nbytes),
               "d2h_bytes_per_step": n_solves * b.nbytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        its = per_l.get("1.0", {}).get("iters")
        v, parts, k = oracle_solve_estimate(X, b, cfg, 1.0, gpu_iters=its)
        cpu = {"value": v, "unit": "s/solve", "cores": cpu_cores(), "kind": "oracle",
               "sample": (f"{args.config} at l=1 (k={k}): Alg.1, FPS, Cholesky, V in full; kNN, "
                          f"FSAI and kernel-matvec rows 1/16 sampled and scaled x16; "
                          f"{its} PCG iterations (the GPU's count)"),
               "parts_s": parts}

    if rank == 0:
        line = {"metric": METRIC, "value": value_s, "unit": "s/solve", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup),
                "ms_per_step": job_ms / args.steps, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded uniform cube, b~N(0,1))",
                "config": {"workload": args.config, "n": cfg.n, "d": cfg.d, "ls": list(cfg.ls),
                           "mu": cfg.mu, "k_cap": cfg.k_cap, "k_adaptive": True, "w": cfg.w,
                           "tol": cfg.tol, "maxit": cfg.maxit,
                           "l2": "flushed between timed steps (256 MiB write, outside events)",
                           "parallelism": f"sweep split over {world} rank(s)",
                           "per_l": per_l},
                "kmv_gpairs_per_s": kmv_gpairs,
                "gpu_launches": launches,
                "roofline": roofline, "roofline_kmv": r_kmv,
                "time_share_ms": shares, "kernel_ms": kernel_ms,
                "clocks": sampler.summary(),
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
