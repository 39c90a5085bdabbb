#!/usr/bin/env python
"""bench.py -- HODLR factor + logdet + solve throughput on B200 (BASELINE.json config 3).

One "step" is one pass of the whole hot path over the config-3 workload with the inputs resident
in HBM: hodlr_build (sort + tree + ACA, the paper's "Assembly"), hodlr_factor, hodlr_logdet and
hodlr_solve of one right-hand side (PAPER.md:1270-1281 columns Assembly/Factor/Det./Solve).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement).
--impl reference times the CPU oracle (oracle/, plain single-threaded C) on a bounded sample of
the same workload; it is the reference arm of this tier (there is no reference implementation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import threading
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1403_6015_b200 import inputs  # noqa: E402

METRIC = "HODLR factor+logdet+solve seconds and points/s at n=2^20, 1/2/4/8 B200"
UNIT = "points/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="cfg3")
    p.add_argument("--cpu-sample", type=int, default=1 << 19,
                   help="oracle sample size (points): about 10 s of single-thread CPU work at config 3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_desc(cfg):
    kname = {0: "squared-exponential", 1: "Matern-3/2", 2: "Matern-5/2"}[cfg.kernel]
    return (f"{cfg.name}: n={cfg.n} 1-D x~U[{cfg.lo:g},{cfg.hi:g}] sorted (seed {cfg.seed}), {kname} a={cfg.a:g} "
            f"ell={cfg.ell:g} sigma2={cfg.sigma2:g}, y~N(0,1), leaf {cfg.leaf}, eps={cfg.eps:g}, FP64")


# ------------------------------------------------------------------ oracle (CPU) timing
def oracle_sample(cfg, n_sample):
    """Time the oracle as it stands (build + factor + logdet + solve) on the first n_sample points of the
    same density (interval scaled), single-threaded.  Returns (seconds, n_sample)."""
    from oracle import OracleHODLR
    c = inputs.scaled(cfg, n_sample)
    x = inputs.points(c); y = inputs.rhs(c)
    t0 = time.perf_counter()
    h = OracleHODLR(x, c.kernel, c.theta, c.sigma2, c.leaf, c.eps).factor()
    h.logdet()
    h.solve(y)
    return time.perf_counter() - t0, n_sample


def cpu_baseline_obj(cfg, n_sample):
    t, ns = oracle_sample(cfg, n_sample)
    return {"value": ns / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle (oracle/hodlr_oracle.c, gcc -O2, 1 thread) build+factor+logdet+solve on n={ns} "
                      f"points of the {cfg.name} workload (same density: interval scaled to "
                      f"[{cfg.lo:g},{cfg.lo + (cfg.hi - cfg.lo) * ns / cfg.n:g}]), {t:.2f} s"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = inputs.CONFIGS[args.config]
    ns = args.cpu_sample
    for _ in range(args.warmup):
        oracle_sample(cfg, ns)
    ts = [oracle_sample(cfg, ns)[0] for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    value = ns / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "sample_points": ns, "parallelism": "1 CPU thread"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"n={ns} points of {cfg.name} (same density), per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML (nvidia_ml_py) polled every 2 ms from a
    background thread, else `nvidia-smi -lms 100`."""

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.samples = []

    def __enter__(self):
        self.samples, self.lines = [], []
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = self.dev
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.dev])
                except ValueError:
                    pass
            hdl = pynvml.nvmlDeviceGetHandleByIndex(idx)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(hdl, pynvml.NVML_CLOCK_SM)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}

            def run():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(hdl) \
                            if hasattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons") \
                            else pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hdl)
                        self.samples.append((float(sm), float(mx), [k for k, b in bits.items() if rs & b]))
                    except Exception:
                        pass
                    self._stop.wait(0.002)
            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
            while not self.samples and self.th.is_alive():      # first sample before the timed region starts
                time.sleep(0.001)
            self.samples.clear()
            return self
        except Exception:
            self.th = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if getattr(self, "th", None):
            self._stop.set()
            self.th.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill(); out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for s, m, rs in self.samples:
            mx = max(mx, m)
            if s > 0.5 * m:
                sm.append(s)
            reasons.update(rs)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                s = float(f[0]); m = float(f[1])
            except ValueError:
                continue
            mx = max(mx, m)
            if s > 0.5 * m:                      # under load
                sm.append(s)
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(self.samples) + len(self.lines),
                "source": "nvml" if self.samples else "nvidia-smi"}


# ------------------------------------------------------------------ algorithmic counts
def algorithmic(info, n, leaf):
    """Per-launch algorithmic work of each kernel family of the formulation implemented:
    (bound, amount, unit_of_amount, kernel name)."""
    K = info["K"]
    r = info["max_rank_by_depth"]
    p = leaf
    nl = n // p
    kap = info["kappa"]
    Kd = [0]
    for x in r:
        Kd.append(Kd[-1] + x)
    ntile_bytes = (p // 8) * (p // 8 + 1) // 2 * 64 * 8           # X = L^{-1} tiles per leaf
    fam = {}
    # ACA (all levels): every step streams the previous factor columns of its block side once and writes one
    # column: sum_k 8 (k + 1) bytes per element, plus the points -- 8 n K + 4 n sum r_d^2 in total
    fam["aca"] = ("hbm", 8 * n * K + 4 * n * sum(x * x for x in r), "bytes", "k_aca_pass/k_aca_fused")
    # leaf Cholesky + triangular inverse (tensor pipe): p^3/3 + p^3/3 flop per leaf
    fam["leaf_chol"] = ("tensor", nl * (2 * p ** 3 / 3), "flop", "k_leaf_chol")
    # Z = X E (p^2 K) and Pi = Z^T Z (p K^2) per leaf (tensor pipe)
    fam["leaf_factor"] = ("tensor", nl * (p * p * K + p * K * K), "flop", "k_leaf_zsyrk")
    # coupling tree: per node q^3 (S^-1) + 4 q^2 K_d (T, refinement) + q K_d^2 (Schur update of Pi), FP64 ALU
    tree = 0
    for d in range(kap):
        q = 2 * r[d]
        tree += 2 ** d * (q ** 3 + 4 * q * q * Kd[d] + q * Kd[d] ** 2)
    fam["coupling_tree"] = ("alu", 2 * tree, "flop", "k_tree_factor")
    # solve: X tiles and the panel E read twice (up and down), y gathered twice, x written
    fam["solve"] = ("hbm", 2 * (nl * ntile_bytes + 8 * n * K) + 3 * 8 * n, "bytes", "k_solve")
    return fam


def ncu_traffic():
    """DRAM bytes per launch from the newest committed ncu summary (profiles/rNN_ncu_summary.json)."""
    import glob
    fs = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not fs:
        return {}, None
    with open(fs[-1]) as f:
        d = json.load(f)
    return {k: v.get("dram_bytes") for k, v in d.get("kernels", {}).items()}, os.path.basename(fs[-1])


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp64_peak_tflops(peaks, sm_mhz):
    """FP64 tensor (DMMA) peak.  MEASURED_PEAKS.json has no FP64 figure; use the DMMA microbenchmark
    (tools/fp64_peak.cu, profiles/fp64_peak_r01.json: 37.13 TFLOP/s at 1965 MHz = 148 SM x 64 FMA/clk x 2)."""
    if "fp64_tflops" in peaks:
        return peaks["fp64_tflops"], "measured (MEASURED_PEAKS.json fp64_tflops)"
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
            v = json.load(f)["fp64_dmma_m8n8k4_tflops"]
        return v, "measured DMMA peak, tools/fp64_peak.cu (profiles/fp64_peak_r01.json), 1965 MHz"
    except (OSError, KeyError, ValueError):
        f = (sm_mhz or 1965.0) * 1e6
        return 148 * 64 * 2 * f / 1e12, f"derived: 148 SMs x 64 FP64 FMA/clk x 2 x {f / 1e6:.0f} MHz"


def dfma_peak_tflops(sm_mhz):
    """Plain FP64 FMA (DFMA) peak for ALU-bound kernels: the DFMA-only microbenchmark (tools/fp64_peak.cu,
    profiles/fp64_peak_r01.json, 33.37 TFLOP/s at 1965 MHz); else 148 SMs x 64 FP64 lanes x 2 x clock."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
            v = json.load(f)["fp64_dfma_tflops"]
        return v, "measured DFMA peak, tools/fp64_peak.cu (profiles/fp64_peak_r01.json), 1965 MHz"
    except (OSError, KeyError, ValueError):
        f = (sm_mhz or 1965.0) * 1e6
        return 148 * 64 * 2 * f / 1e12, f"derived: 148 SMs x 64 FP64 lanes x 2 x {f / 1e6:.0f} MHz"


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.cuda.current_device()
    from paper_1403_6015_b200 import hodlr as hb
    hb.load()
    dd = None
    if ws > 1:       # subtree sharding (north_star): rank g owns the depth-log2(N) subtree g, NCCL allgathers
        from paper_1403_6015_b200.dist import Dist
        dd = Dist.from_torch()
    cfg = inputs.CONFIGS[args.config]
    n = cfg.n
    x = inputs.points(cfg); y = inputs.rhs(cfg)
    xd = torch.from_numpy(x).to(dev); yd = torch.from_numpy(y).to(dev)
    xh = torch.from_numpy(x).pin_memory(); yh = torch.from_numpy(y).pin_memory()
    sol_h = torch.empty(n, dtype=torch.float64).pin_memory()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)     # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(xin, yin):
        h = hb.HODLR(xin, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps, dist=dd)
        h.factor()
        ld = h.logdet()
        sol = h.solve(yin)
        info = h.info()
        h.close()
        return ld, sol, info

    def barrier():
        if ws > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step(xd, yd)
    torch.cuda.synchronize()
    # ---------------- device-resident timed region
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    fam_ms = {}
    infos = []
    barrier(); torch.cuda.synchronize()
    l0 = hb.hodlr_launch_count()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.zero_()                                    # L2 flush between timed steps (untimed)
            evs[i][0].record(stream)
            ld, sol, info = step(xd, yd)
            evs[i][1].record(stream)
            infos.append(info)
        torch.cuda.synchronize()
    barrier()
    launches = hb.hodlr_launch_count() - l0
    ms = [a.elapsed_time(b) for a, b in evs]
    t_step = sum(ms) / len(ms) / 1e3
    for inf in infos:
        for k, v in inf["kernel_ms"].items():
            fam_ms[k] = fam_ms.get(k, 0.0) + v
    fam_ms = {k: v / len(infos) for k, v in fam_ms.items() if not k.startswith("unused")}
    t_max = t_step
    if ws > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    # ---------------- end-to-end through the C-ABI with host buffers: x copied first (the build needs it), y on a
    # side stream concurrently with the build/factor (only the solve needs it), solution read back; all inside
    # the timed region
    ys = torch.cuda.Stream()
    ev_y = torch.cuda.Event()

    def step_e2e():
        xd.copy_(xh, non_blocking=True)
        ys.wait_stream(stream)
        with torch.cuda.stream(ys):
            yd.copy_(yh, non_blocking=True)
            ev_y.record(ys)
        h = hb.HODLR(xd, cfg.kernel, cfg.theta, cfg.sigma2, cfg.leaf, cfg.eps, dist=dd)
        h.factor()
        ld_ = h.logdet()
        stream.wait_event(ev_y)
        s_ = h.solve(yd)
        sol_h.copy_(s_, non_blocking=True)
        h.close()
        return ld_, s_

    for _ in range(max(1, args.warmup)):
        step_e2e(); torch.cuda.synchronize()
    e2e_ms = []
    barrier(); torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ld_e, s = step_e2e()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    barrier()
    t_e2e = sum(e2e_ms) / len(e2e_ms) / 1e3
    if ws > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    # sanity: solution is finite and the log det is the expected magnitude
    assert math.isfinite(ld) and torch.isfinite(sol).all().item()
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0
    info = infos[-1]
    clocks = clk.summary()
    peaks = load_peaks()
    # ---------------- rooflines: algorithmic work / live event time per kernel family; dominant = longest
    alg = algorithmic(info, n, cfg.leaf)
    fp64_peak, fp64_how = fp64_peak_tflops(peaks, clocks.get("sm_mhz"))
    dfma_peak, dfma_how = dfma_peak_tflops(clocks.get("sm_mhz"))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic, traffic_src = ncu_traffic()
    rows = []
    for fam, (bound, amount, unit, kname) in alg.items():
        ms = fam_ms.get(fam, 0.0)
        calls = info["kernel_calls"].get(fam) or 1
        if ms <= 0.0:
            continue
        t_launch = ms / calls / 1e3
        if bound == "hbm":
            ach, peak, u = amount / t_launch / 1e9, hbm_peak, "GB/s"
        elif bound == "alu":       # plain FP64 FMA pipe (DFMA), not the DMMA tensor path
            ach, peak, u = amount / t_launch / 1e12, dfma_peak, "TFLOP/s"
        else:
            ach, peak, u = amount / t_launch / 1e12, fp64_peak, "TFLOP/s"
        kk = kname.split("/")[0]
        tr = traffic.get(kk)
        if tr is not None and fam == "aca":
            tr = None          # the capture is one pass of one step, not the whole ACA family
        rows.append({"kernel": kname, "family": fam, "bound": bound, "achieved": ach, "peak": peak, "unit": u,
                     "frac": ach / peak, "traffic": tr, "ms": ms / calls,
                     ("algorithmic_bytes_per_launch" if bound == "hbm" else "algorithmic_flops_per_launch"): amount})
    main = [r_ for r_ in rows if r_["family"] != "leaf_chol"]     # leaf_chol runs on a side stream under the ACA
    dom = max(main, key=lambda r_: r_["ms"])
    roof = dict(dom)
    roof["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if dom["bound"] == "hbm"
                           else (dfma_how if dom["bound"] == "alu" else fp64_how))
    roof["traffic_source"] = traffic_src
    roof["all_kernels"] = rows
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = cpu_baseline_obj(cfg, args.cpu_sample)
    value = n / t_max                  # one n-point problem per step, sharded over the ranks (strong scaling)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "n": n,
                       "parallelism": (f"subtree sharding over {ws} GPUs (top log2(N) levels redundant, NCCL "
                                       f"allgather of the depth-log2(N) projections)") if ws > 1 else "1 GPU",
                       "l2": "flushed between timed steps (512 MB device write, untimed)",
                       "kappa": info["kappa"], "K": info["K"], "ranks_by_depth": info["max_rank_by_depth"],
                       "phase_ms": {"assembly(build)": 1e3 * info["t_build"], "factor": 1e3 * info["t_factor"],
                                    "det": 1e3 * info["t_logdet"], "solve": 1e3 * info["t_solve"]},
                       "kernel_family_ms": fam_ms, "seconds_per_step": t_max,
                       "gpu_launches_per_step": launches / args.steps},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": n / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 16 * n,
                    "d2h_bytes_per_step": 8 * n + 8, "ms_per_step": 1e3 * t_e2e},
            "gpu_launches": launches, "clocks": clocks}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
