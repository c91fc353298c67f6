#!/usr/bin/env python
"""bench.py -- AFN-PCG on B200 (arXiv 2304.05460 hot path), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl afn|reference]
                    [--config C3] [--no-e2e] [--no-cpu] [--no-sweep]

Workload (default BASELINE.json configs[2], "C3"): n = 131072 points uniform
in a constant-density 3-D cube, Gaussian kernel l = 1, mu = 1e-4, b ~ N(0,1)
(seed 0), adaptive k <= 4000 (Algorithm 1), FSAI 100 nnz/row, PCG tol 1e-4.
One *step* = one whole AFN-PCG solve of that problem -- every SURVEY.md 8(a)
row: Alg. 1, FPS, permutation, Cholesky, W, kNN, FSAI, then PCG with the
kernel matvec and the AFN apply -- with its rows sharded over the N ranks
(one GPU each, NCCL all-gathers; N = 1 is the one-GPU path).  Strong scaling:
the problem is fixed as N grows.  `--config C5` runs the north star's
n = 2^20 scaling problem the same way.

Metric: AFN-PCG seconds per solve (device time, CUDA events on the launching
stream, max over ranks; lower is better) with the kernel matvec's Gpairs/s and
its fraction of the FP64 peak beside it (`roofline_kmv`), the AFN apply's HBM
fraction (`roofline_apply`) and the dominant kernel's roofline (`roofline`).
`c2_sweep` repeats BASELINE.json's 1-GPU C2 sweep (n = 16384, six l) as an
extra key.  `e2e` is the same solve through afn_solve_host (host buffers,
copies inside the timed region).  `cpu_baseline` times the oracle on a
bounded sample of the same workload on this host's cores.
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

METRIC = "AFN-PCG solve sec & kernel-matvec Gpairs/s (fp64) vs FP64 roofline"
# FP64 peak from the guide's unit counts and clocks: 148 SMs x
# 64 FP64 FMA lanes/clk x 1.965 GHz; flops count an FMA as 2.  MEASURED_PEAKS.json
# has no FP64 entry; afn_probe_dfma's measured figure is reported beside it.
SMS, FP64_LANES, SM_GHZ = 148, 64, 1.965
FP64_PEAK_TFLOPS = SMS * FP64_LANES * 2 * SM_GHZ / 1e3
FP64_PIPE_INST_PER_S = SMS * FP64_LANES * SM_GHZ * 1e9


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "of measured"
    except Exception:
        return 6650.0, "of fallback"  # B200_PROFILING.md


HBM_PEAK_GBS, HBM_PEAK_SRC = _hbm_peak()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="afn", choices=["afn", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
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


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
def oracle_iterations(cfg, l):
    """The oracle's own PCG iteration count for this workload, if committed
    (tests/oracle_data, written by tools/make_oracle_fixtures.py from oracle/)."""
    import numpy as np
    fx = os.path.join(ROOT, "tests", "oracle_data", f"{cfg.name.lower()}_l{l:g}.npz")
    if os.path.exists(fx):
        return int(np.load(fx)["iters"]), "oracle's own count (tests/oracle_data)"
    return None, None


def oracle_sample_estimate(X, b, cfg, l, its):
    """Seconds the oracle (as it stands, numpy/scipy on this host's cores)
    needs for one AFN-PCG solve of this workload, from a bounded sample:
      * Alg. 1 and the k x k Cholesky of K11 + mu I: in full;
      * FPS: the first 256 steps, scaled by k / 256 (every step is one O(n)
        distance update);
      * V = L^{-1} K12 on every 64th non-landmark column, scaled x 64;
      * kNN rows and FSAI rows (S_JJ from K_JJ, mu and V_J; the solve) on
        every 1024th non-landmark row, scaled x 1024;
      * the kernel matvec on every 512th row, scaled x 512, times (its + 1)
        (the loop's products and the true residual);
      * the apply: the four triangular solves with L in full, the
        two K12 products on the 64th-column sample (x 64) and the G, G^T
        products on the 1024th-row sample (x 1024), times (its + 1).
    The landmarks past the FPS sample are the next points of a seeded random
    order (they only have to be k distinct points for the timing).  Returns
    (seconds, parts, k)."""
    import numpy as np
    import scipy.linalg as sla
    import oracle as O
    threads = cpu_cores()
    t = {}
    n = len(X)
    c = time.perf_counter()
    a1 = O.alg1(X, l)
    t["alg1"] = time.perf_counter() - c
    k = min(cfg.k_cap, max(1, a1["khat"]), n)
    kf = min(k, 256)
    c = time.perf_counter()
    idx, _ = O.fps(X, kf, 0)
    t["fps"] = (time.perf_counter() - c) * k / kf
    if k > kf:
        rest = np.setdiff1d(np.random.default_rng(0).permutation(n), idx, assume_unique=True)
        idx = np.concatenate([idx, rest[: k - kf]])
    mask = np.ones(n, bool)
    mask[idx] = False
    perm = np.concatenate([idx, np.nonzero(mask)[0]])
    Xp = X[perm]
    X1, X2 = Xp[:k], Xp[k:]
    N2 = n - k
    c = time.perf_counter()
    L = np.linalg.cholesky(O.kernel_block(X1, X1, l) + cfg.mu * np.eye(k))
    t["chol"] = time.perf_counter() - c
    cols = np.arange(0, N2, 64)
    c = time.perf_counter()
    K12s = O.kernel_block(X1, X2[cols], l)
    sla.solve_triangular(L, K12s, lower=True)
    t["V"] = (time.perf_counter() - c) * N2 / len(cols)
    rows = np.arange(0, N2, 1024)
    c = time.perf_counter()
    pats = [O.knn_row(X2, int(i), cfg.w) for i in rows]
    t["knn"] = (time.perf_counter() - c) * N2 / len(rows)
    VJ = {int(i): sla.solve_triangular(L, O.kernel_block(X1, X2[J], l), lower=True) for i, J in zip(rows, pats)}
    c = time.perf_counter()
    gv = []
    for i, J in zip(rows, pats):
        V = VJ[int(i)]
        S = O.kernel_block(X2[J], X2[J], l) + cfg.mu * np.eye(len(J)) - V.T @ V
        gv.append(O.fsai_rows(lambda _J, S=S: S, np.array([0, len(J)]), J))
    t["fsai"] = (time.perf_counter() - c) * N2 / len(rows)
    mrows = np.arange(0, n, 512)
    c = time.perf_counter()
    O.kmv_rows(Xp, l, cfg.mu, b, mrows)
    t_kmv = (time.perf_counter() - c) * n / len(mrows)
    import scipy.sparse as sp
    rp = np.zeros(len(rows) + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(J) for J in pats])
    Gs = sp.csr_matrix((np.concatenate(gv), np.concatenate(pats), rp), shape=(len(rows), N2))
    r1, u = b[:k], b[k:]
    c = time.perf_counter()
    y = sla.solve_triangular(L.T, sla.solve_triangular(L, r1, lower=True), lower=False)
    sla.solve_triangular(L.T, sla.solve_triangular(L, y, lower=True), lower=False)
    t_tri = time.perf_counter() - c
    c = time.perf_counter()
    K12s.T @ y
    K12s @ u[cols]
    t_k12 = (time.perf_counter() - c) * N2 / len(cols)
    c = time.perf_counter()
    g = Gs @ u
    Gs.T @ g
    t_g = (time.perf_counter() - c) * N2 / len(rows)
    t_apply = t_tri + t_k12 + t_g
    t["pcg"] = (its + 1) * t_kmv + (its + 1) * t_apply
    t["per_matvec"] = t_kmv
    t["per_apply"] = t_apply
    total = sum(v for key, v in t.items() if not key.startswith("per_"))
    return total, {key: round(v, 3) for key, v in t.items()}, k, threads


ORACLE_SAMPLE = ("Alg.1 and the k x k Cholesky in full; FPS first 256 steps (x k/256); V on every 64th "
                 "column (x64); kNN + FSAI rows every 1024th (x1024); kernel matvec every 512th row "
                 "(x512) x (its+1); apply: triangular solves in full, K12 and G products on the same "
                 "samples, x (its+1)")


# ---------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import CONFIGS, gen_problem
    cfg = CONFIGS[args.config]
    l = cfg.ls[0]
    X, b = gen_problem(cfg)
    its, src = oracle_iterations(cfg, l)
    if its is None:
        its, src = 10, "assumed (no committed oracle count for this config)"
    for _ in range(args.warmup):
        oracle_sample_estimate(X, b, cfg, l, its)
    vals = []
    t0 = time.perf_counter()
    parts, k, threads = None, None, None
    for _ in range(args.steps):
        v, parts, k, threads = oracle_sample_estimate(X, b, cfg, l, its)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = sum(vals) / len(vals)
    sample = f"{cfg.name} l={l:g} (k={k}): {ORACLE_SAMPLE}; {its} PCG iterations, {src}"
    line = {"metric": METRIC, "value": value, "unit": "s/solve", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "l": l, "mu": cfg.mu,
                       "k_cap": cfg.k_cap, "k_adaptive": True, "w": cfg.w, "tol": cfg.tol},
            "cpu_baseline": {"value": value, "unit": "s/solve", "cores": threads, "kind": "oracle",
                             "sample": sample, "parts_s": parts},
            "e2e": {"value": value, "unit": "s/solve", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

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
    l = cfg.ls[0]
    X, b = gen_problem(cfg)
    Xd, bd = torch.from_numpy(X).to(dev), torch.from_numpy(b).to(dev)
    comm = afn.Comm.from_process_group(dist) if dist else None
    prm = afn.make_params(l, cfg.mu, cfg.k_cap, cfg.w, k_adaptive=True)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2

    def timed(steps, step_fn):
        """K steps between a barrier + synchronize on both sides, CUDA events on
        the launching stream, L2 flushed before each step (outside the events);
        returns (this rank's total ms, the max over ranks)."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for s in range(steps):
            flush.zero_()
            evs[s][0].record(stream)
            step_fn()
            evs[s][1].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        per = [e0.elapsed_time(e1) for e0, e1 in evs]
        if os.environ.get("AFN_BENCH_STEPS"):
            print("step ms: " + " ".join(f"{x:.1f}" for x in per), file=sys.stderr, flush=True)
        mine = sum(per)
        t = torch.tensor([mine], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return mine, float(t.item())

    records = []

    def solve(record):
        h = afn.afn_build(Xd, prm, comm=comm)
        a, rep = h.pcg_solve(bd, tol=cfg.tol, maxit=cfg.maxit)
        if record:
            records.append((h.info(), rep))
        h.close()

    for _ in range(max(3, args.warmup)):
        solve(False)
    sampler = ClockSampler(local)
    l0 = afn.launch_count()
    with sampler:
        _, job_ms = timed(args.steps, lambda: solve(True))
    launches = afn.launch_count() - l0
    value_s = job_ms / 1e3 / args.steps
    # the same steps again with the library's per-kernel CUDA-event timers on
    # (their event records and end-of-call collection are kept out of `value`)
    afn.kernel_timers(reset=True, enable=True)
    _, kt_job_ms = timed(args.steps, lambda: solve(False))
    kt = afn.kernel_timers(enable=False)

    # ---- rooflines from the library's CUDA-event timers (timed region)
    inf0, rep0 = records[0]
    n, d = cfg.n, cfg.d
    step_ms = job_ms / args.steps
    traffic = {}
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path))
        except Exception:
            traffic = {}

    def roof(name):
        v = kt.get(name)
        if not v or v["count"] <= 0 or v["ms"] <= 0:
            return None
        per_ms = v["ms"] / v["count"]
        out = {"kernel": name, "launches": v["count"], "ms_per_launch": per_ms,
               # (device ms per step over the un-instrumented step: the timers'
               # event records slow the instrumented pass itself)
               "share_of_step": v["ms"] / args.steps / step_ms if step_ms > 0 else None,
               "traffic": (traffic.get(args.config, {}) or {}).get(name)}
        if name == "apply":
            ach = v["work"] / (v["ms"] * 1e-3) / 1e9
            out.update({"bound": "hbm", "achieved": ach, "peak": HBM_PEAK_GBS, "unit": "GB/s",
                        "frac": ach / HBM_PEAK_GBS, "bytes_per_launch": v["work"] / v["count"],
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({HBM_PEAK_SRC})"})
        elif v["work"] > 0:
            ach = v["work"] / (v["ms"] * 1e-3) / 1e12
            tensor = name in ("group_gemm_kernel", "w_gemm_kernel")
            out.update({"bound": "tensor" if tensor else "alu", "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                        "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS,
                        "flops_per_launch": v["work"] / v["count"],
                        "peak_source": ("FP64 (DMMA = SIMT rate on B200) " if tensor else "FP64 ") +
                                       "from the guide's unit counts: 148 SM x 64 FP64 lanes x 2 x 1.965 GHz"})
        else:
            out.update({"bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None})
        return out

    cand = {k: v for k, v in kt.items() if v["count"] > 0 and v["work"] > 0}
    dom = max(cand, key=lambda k: cand[k]["ms"]) if cand else None
    roofline = roof(dom) if dom else None
    r_kmv = roof("kmv_kernel")
    if r_kmv:
        # executed FP64-pipe instructions per useful pair / flops per pair
        # (kmv.cu kmv_fp64_inst / kmv_flops; Gaussian, symmetric, d <= 4):
        # (2d + 9) / (3d + 15).  Cutoff plan: the work is
        # FP64-equivalent -- an FP32-body pair (one MUFU.EX2 at 16 / SM / clk)
        # is credited the (3d + 15) * 4 / (2d + 9) flops whose FP64 pipe time
        # it takes -- so `frac` and `fp64_pipe_frac` are fractions of the
        # product's issue-bound lower time.
        inst_per_flop = (2 * d + 9) / (3 * d + 15)
        r_kmv["fp64_pipe_frac"] = r_kmv["achieved"] * 1e12 * inst_per_flop / FP64_PIPE_INST_PER_S
        kmv = kt["kmv_kernel"]
        per_s = kmv["count"] / (kmv["ms"] * 1e-3) / max(1, world)  # products per second per rank
        p64, p32 = float(inf0["kmv_pairs64"]), float(inf0["kmv_pairs32"])
        r_kmv["plan"] = {0: "row-wise", 1: "dense symmetric", 2: "cutoff"}.get(inf0["kmv_plan"], "?")
        r_kmv["pairs_fp64"], r_kmv["pairs_fp32"] = p64, p32
        r_kmv["pairs_fraction"] = (p64 + p32) / (n * (n - 1) / 2.0)
        if inf0["kmv_plan"] == 2:
            r_kmv["peak_source"] = ("FP64 from the guide's unit counts (148 SM x 64 FP64 lanes x 2 x 1.965 GHz); "
                                    "FP32-body pairs credited at the MUFU.EX2 rate (afn_probe_ex2)")
        # unordered pairs evaluated x 2 (ordered) per second, and n^2 per
        # product per second (what the dense product would have to reach)
        r_kmv["gpairs_per_s"] = 2.0 * (p64 + p32) * per_s / 1e9
        r_kmv["gpairs_per_s_dense_equiv"] = float(n) * n * per_s / 1e9
    r_apply = roof("apply")
    kernel_ms = {k: round(v["ms"] / args.steps, 3) for k, v in kt.items() if v["count"] > 0}
    try:
        probe = afn.probe_dfma()
        probe_ex2 = afn.probe_ex2()
    except Exception:
        probe, probe_ex2 = None, None

    # ---- C2 sweep (BASELINE.json configs[1]) as an extra key
    sweep = None
    if not args.no_sweep:
        c2 = CONFIGS["C2"]
        X2, b2 = gen_problem(c2)
        X2d, b2d = torch.from_numpy(X2).to(dev), torch.from_numpy(b2).to(dev)
        my_ls = list(c2.ls[rank::world])
        per_l = {}

        def sweep_step(record=False):
            for ll in my_ls:
                h = afn.afn_build(X2d, afn.make_params(ll, c2.mu, c2.k_cap, c2.w, k_adaptive=True))
                _, rp = h.pcg_solve(b2d, tol=c2.tol, maxit=c2.maxit)
                if record:
                    inf = h.info()
                    per_l[str(ll)] = {"k": inf["k"], "khat": inf["khat"], "iters": rp["iterations"],
                                      "setup_ms": round(inf["ms_total"], 3), "pcg_ms": round(rp["solve_ms"], 3)}
                h.close()

        sweep_step(True)
        _, sw_ms = timed(args.steps, sweep_step)
        sweep = {"value": sw_ms / 1e3 / (args.steps * len(c2.ls)), "unit": "s/solve",
                 "workload": "C2", "n": c2.n, "ls": list(c2.ls), "split": f"sweep split over {world} rank(s)",
                 "per_l": per_l}

    # ---- e2e: host buffers through the C ABI (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        bh = torch.from_numpy(b).pin_memory()
        afn.afn_solve_host(Xh.numpy(), bh.numpy(), prm, tol=cfg.tol, maxit=cfg.maxit, comm=comm)  # warm
        _, e_ms = timed(args.steps, lambda: afn.afn_solve_host(Xh.numpy(), bh.numpy(), prm, tol=cfg.tol,
                                                               maxit=cfg.maxit, comm=comm))
        e2e = {"value": e_ms / 1e3 / args.steps, "unit": "s/solve", "h2d_bytes_per_step": X.nbytes + b.nbytes,
               "d2h_bytes_per_step": b.nbytes}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        its = rep0["iterations"]
        v, parts, k, threads = oracle_sample_estimate(X, b, cfg, l, its)
        cpu = {"value": v, "unit": "s/solve", "cores": threads, "kind": "oracle",
               "sample": f"{cfg.name} l={l:g} (k={k}): {ORACLE_SAMPLE}; {its} PCG iterations (the GPU's count)",
               "parts_s": parts}

    if rank == 0:
        line = {"metric": METRIC, "value": value_s, "unit": "s/solve", "n_gpus": world,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": step_ms,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded uniform cube, b ~ N(0,1))",
                "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "l": l, "mu": cfg.mu,
                           "k_cap": cfg.k_cap, "k_adaptive": True, "w": cfg.w, "tol": cfg.tol,
                           "maxit": cfg.maxit, "parallelism": f"rows sharded over {world} rank(s)",
                           "l2": "flushed between timed steps (256 MiB write, outside the events)",
                           "k": inf0["k"], "khat": inf0["khat"], "iters": rep0["iterations"],
                           "setup_ms": round(inf0["ms_total"], 3), "pcg_ms": round(rep0["solve_ms"], 3),
                           "relres_true": rep0["relres_true"]},
                "kmv_gpairs_per_s": r_kmv["gpairs_per_s"] if r_kmv else None,
                "gpu_launches": launches,
                "roofline": roofline, "roofline_kmv": r_kmv, "roofline_apply": r_apply,
                "fp64_probe_tflops": probe, "ex2_probe_gops": probe_ex2, "kernel_ms_per_step": kernel_ms,
                "clocks": sampler.summary(), "c2_sweep": sweep,
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
