#!/usr/bin/env python
"""SPARTan PARAFAC2-ALS benchmark (BASELINE.json metric: sec/iter & nnz/s at
1/2/4/8 B200, % of HBM roofline).

A "step" is one full PARAFAC2-ALS outer iteration (Procrustes + MTTKRP modes
1-3 + H/V/W updates + fit, solver.hpp:274-318) over the whole synthetic
workload.  Default workload: BASELINE.json configs[1] ("cfg2": K=1M
subjects, J=5000, R=10, ~63M nnz, fp64), generated on the host (seeded,
SURVEY.md §8d); inputs are far larger than L2 (CSR 1.2 GB + Q 4 GB vs
126 MB), so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl b200|reference]

Under torchrun (N>1) each rank owns the subjects partition_weighted gives it
(weak per-rank share of one fixed workload -> "scaling": "strong").
``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port; the reference itself cannot be compiled here) on
the host cores, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_RANK = {1: 5, 2: 10, 3: 40, 4: 40, 5: 40}
CONFIG_NAME = {1: "cfg1 tiny (K=1000, J=500, R=5)", 2: "cfg2 paper-scale (K=1M, J=5000, R=10, ~63M nnz)",
               3: "cfg3 paper-scale (K=1M, J=5000, R=40, ~250M nnz)",
               4: "cfg4 largest (K=1M, J=5000, R=40, ~500M nnz)", 5: "cfg5 EHR skew (K=500K, J=1500, R=40)"}
METRIC = "spartan_als_nnz_per_s"


def load_fp64_peak():
    """Measured DFMA peak (scripts/fp64_peak.cu, profiles/fp64_peak_r01.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
            return float(json.load(f)["dfma_tflops"]), "measured (scripts/fp64_peak.cu)"
    except Exception:
        return 37.0, "fallback"


def iteration_flops(X, R):
    """SURVEY.md 8(d) F_iter: 6 nnz R + 12 sum(I_k) R^2 + 11 K R^3 (XV twice and X^T U';
    six I_k x R x R products; eig ~9R^3 + 2R^3 for the inverse square root)."""
    return 6.0 * X.nnz * R + 12.0 * X.n_rows * R * R + 11.0 * X.K * R ** 3


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(X, R):
    """Per-launch compulsory HBM bytes of each loop phase, for
    the kernels as designed.  CSR = 12 B/nnz + 8 B/row + 8 B/subject; CSC copy
    = 12 B/nnz + 8 B/column; per-subject packed C/S = 8 R(R+1)/2 B; E = 8 R^2 B;
    W rows 8 R B; U / Q rows 8 R B; V 8 J R B (L2-resident, counted once)."""
    K, J = X.K, X.J
    nnz, nr = X.nnz, X.n_rows
    nt = R * (R + 1) // 2
    csr = 12 * nnz + 8 * (nr + 1) + 8 * (K + 1)
    csc = 12 * nnz + 8 * (J + 1)
    q = 8 * nr * R
    w = 8 * K * R
    v = 8 * J * R
    gather_u = 8 * nnz * R  # M2 = X^T U: one U row per entry
    xv = q  # X V rows (NR x R) left by mode 3 for the next iteration's passes
    return {
        # small-R Q-free pipeline (steady state: the X V rows of the previous
        # mode-3 pass replace mode 2's CSR pass and mode 3's V_{t-1} gathers)
        "polar": 8 * K * (2 * nt + R),                  # C, W in; S out
        "mode2": xv + 8 * K * nt + w + q + csc + gather_u,  # X V rows, S, W in, U out; CSC + U rows in
        "mode3": csr + xv + xv + 8 * K * nt + w + w + 8 * K * nt + v,  # CSR, X V in and out, S, W in; m3, next C out
        "update_w": 2 * w,                              # m3 in, W out (NNLS)
        "fit": 2 * w,                                   # W, m3 in (gram + cross)
        # large-R pipeline: Procrustes reads the X V rows, writes Q, E in/out (warm start) ...
        "procrustes": xv + q + w + 2 * 8 * K * R * R,
        # ... mode 2 = Q in, U out, CSC + U rows in
        "mode2_large": 2 * q + csc + gather_u,
        # ... mode 3 = Q and the CSR in, X V rows and m3 out
        "mode3_large": q + csr + xv + w + v,
        # SURVEY.md §8d north-star iteration bytes (Q-based formulation)
        "iteration": 3 * csr + 3 * q + 4 * w + 4 * v,
    }


def setup_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def cpu_baseline(X, R, cfg_id, target_s=12.0, threads=None):
    """Oracle (CPU restatement of the reference, kind "port") on a bounded
    prefix of the same workload, all host threads."""
    import paper_1703_04219_b200 as p2g
    from tests.helpers import load_oracle, oracle_from_csr

    o = load_oracle()
    threads = threads or (os.cpu_count() or 1)
    probe = min(X.K, 2000)
    Xs = X.subset(0, probe)
    H0, V0, W0 = p2g.init_factors(102, Xs.K, Xs.J, R)
    t0 = time.perf_counter()
    o.fit_parafac2(oracle_from_csr(o, Xs), R, max_iters=1, tol=1e-300, nonneg=True, threads=threads, H0=H0, V0=V0,
                   W0=W0)
    dt = max(time.perf_counter() - t0, 1e-3)
    per_subject = dt / probe
    n = int(min(X.K, max(probe, target_s / 3.0 / per_subject)))
    Xs = X.subset(0, n)
    H0, V0, W0 = p2g.init_factors(102, Xs.K, Xs.J, R)
    T = oracle_from_csr(o, Xs)
    iters = 3
    t0 = time.perf_counter()
    r = o.fit_parafac2(T, R, max_iters=iters, tol=1e-300, nonneg=True, threads=threads, H0=H0, V0=V0, W0=W0)
    dt = time.perf_counter() - t0
    sec_iter = dt / iters
    return {"value": Xs.nnz / sec_iter, "unit": "nnz/s", "cores": threads, "kind": "port",
            "sample": f"first {n} of {X.K} subjects of {CONFIG_NAME[cfg_id].split(' (')[0]} "
                      f"({Xs.nnz} nnz), {iters} ALS iterations, oracle/p2_oracle.hpp -O3, {threads} threads",
            "sec_per_iter_sample": sec_iter, "est_sec_per_iter_full": sec_iter * X.nnz / Xs.nnz,
            "fit": r["fit"]}


def run_reference(args):
    world, rank, _ = (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if rank != 0:
        return 0
    import paper_1703_04219_b200 as p2g

    cfg_id = args.config
    R = args.rank or CONFIG_RANK[cfg_id]
    X = p2g.generate_baseline(cfg_id, R)
    from tests.helpers import load_oracle, oracle_from_csr

    o = load_oracle()
    threads = os.cpu_count() or 1
    # bounded sample: a prefix sized for ~args.ref_seconds of CPU per step
    probe = min(X.K, 2000)
    Xs = X.subset(0, probe)
    H0, V0, W0 = p2g.init_factors(102, Xs.K, Xs.J, R)
    t0 = time.perf_counter()
    o.fit_parafac2(oracle_from_csr(o, Xs), R, max_iters=1, tol=1e-300, threads=threads, H0=H0, V0=V0, W0=W0)
    per_subject = max(time.perf_counter() - t0, 1e-3) / probe
    n = int(min(X.K, max(probe, args.ref_seconds / per_subject)))
    Xs = X.subset(0, n)
    H0, V0, W0 = p2g.init_factors(102, Xs.K, Xs.J, R)
    T = oracle_from_csr(o, Xs)
    o.fit_parafac2(T, R, max_iters=max(args.warmup, 1), tol=1e-300, threads=threads, H0=H0, V0=V0, W0=W0)
    t0 = time.perf_counter()
    o.fit_parafac2(T, R, max_iters=args.steps, tol=1e-300, threads=threads, H0=H0, V0=V0, W0=W0)
    dt = time.perf_counter() - t0
    ms = dt / args.steps * 1e3
    value = Xs.nnz / (dt / args.steps)
    sample = (f"first {n} of {X.K} subjects of {CONFIG_NAME[cfg_id]} ({Xs.nnz} nnz) per step; "
              f"oracle port of the reference CPU path, {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": "nnz/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAME[cfg_id], "config_id": cfg_id, "rank": R, "K": X.K, "J": X.J,
                       "nnz": X.nnz, "sample_subjects": n, "sample_nnz": Xs.nnz},
            "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    world, rank, local = setup_dist()
    import paper_1703_04219_b200 as p2g

    cfg_id = args.config
    R = args.rank or CONFIG_RANK[cfg_id]
    t_gen = time.perf_counter()
    X = p2g.generate_baseline(cfg_id, R)
    t_gen = time.perf_counter() - t_gen
    H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
    nccl_id = None
    if world > 1:
        import torch
        import torch.distributed as dist

        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(p2g.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    ctx = p2g.Context(local, rank, world, nccl_id)
    ctx.load(X)
    kb, ke, nr, nz = ctx.shard_info()
    cfg = p2g.SolverConfig(rank=R, max_iters=args.steps, tol=1e-300, nonneg=True)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # warm-up (untimed), then exactly K timed steps
    ctx.bench_iterations(cfg, max(args.warmup, 1), H0, V0, W0, reset=True)
    ctx.kernel_times()  # (reset below via reset=True on the timed run's state)
    barrier()
    import torch

    torch.cuda.synchronize()
    launches0 = p2g.load_library().p2g_launch_count()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        ms, fits = ctx.bench_iterations(cfg, args.steps)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    barrier()
    launches = p2g.load_library().p2g_launch_count() - launches0
    ms_step = float(np.mean(ms))  # device time, already max over ranks inside the library
    value = X.nnz / (ms_step * 1e-3)
    ktimes = ctx.kernel_times()

    # roofline of the dominant kernel (largest share of the step)
    peak, peak_kind = load_peaks()
    ab = algorithmic_bytes(X.subset(kb, ke) if world > 1 else X, R)
    cand = {k: v for k, v in ktimes.items() if k in ("polar", "procrustes", "mode2", "mode3", "update_w")}
    dom = max(cand, key=lambda k: cand[k][0]) if cand else None
    roofline = None
    if dom:
        t_launch = cand[dom][0] * 1e-3
        akey = (dom + "_large") if (dom in ("mode2", "mode3") and R > 16) else dom
        achieved = ab[akey] / t_launch / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic_r01.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(f"cfg{cfg_id}", {}).get(dom)
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                    "algorithmic_bytes_per_launch": ab[akey], "ms_per_launch": cand[dom][0],
                    "share_of_step": sum(v[0] * v[1] for k, v in ktimes.items() if k == dom) /
                                     max(sum(v[0] * v[1] for v in ktimes.values()), 1e-12)}
    iter_gbs = ab["iteration"] / (ms_step * 1e-3) / 1e9

    # end-to-end through the public API: pinned host CSR -> load_csr -> fit -> factors back
    e2e = None
    if not args.no_e2e:
        pin = {}
        for name in ("subj_row_ptr", "row_ptr", "col_idx", "val"):
            a = getattr(X, name)
            t = torch.empty(a.shape, dtype={np.int64: torch.int64, np.int32: torch.int32,
                                            np.float64: torch.float64}[a.dtype.type], pin_memory=True)
            t.numpy()[...] = a
            pin[name] = t
        Xp = p2g.CSRTensor(X.J, pin["subj_row_ptr"].numpy(), pin["row_ptr"].numpy(), pin["col_idx"].numpy(),
                           pin["val"].numpy())
        # initial factors from pinned host memory too (column-major views)
        pinned_f = []
        for a in (H0, V0, W0):
            t = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
            v = t.numpy().reshape(a.shape[::-1]).T
            v[...] = a
            pinned_f.append((t, v))
        H0p, V0p, W0p = (v for _, v in pinned_f)
        kb_, ke_, _, _ = ctx.shard_info()
        outs = []
        for shp in ((R, R), (X.J, R), (ke_ - kb_, R)):
            t = torch.empty(shp[0] * shp[1], dtype=torch.float64, pin_memory=True)
            outs.append((t, t.numpy().reshape(shp[::-1]).T))
        e2e_iters = args.steps
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.load(Xp)
        t_load = time.perf_counter() - t0
        res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=e2e_iters, tol=1e-300, nonneg=True), H0p, V0p, W0p,
                      want_q=False, out=tuple(v for _, v in outs))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            import torch.distributed as dist

            tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        h2d = (X.subj_row_ptr.nbytes + X.row_ptr.nbytes + X.col_idx.nbytes + X.val.nbytes + H0.nbytes + V0.nbytes
               + W0.nbytes)
        d2h = res.H.nbytes + res.V.nbytes + res.W.nbytes + 8 * 2 * e2e_iters
        e2e = {"value": X.nnz * e2e_iters / dt, "unit": "nnz/s", "h2d_bytes_per_step": h2d // e2e_iters,
               "d2h_bytes_per_step": d2h // e2e_iters, "iterations_per_call": e2e_iters, "sec_per_call": dt,
               "load_s": t_load, "fit_s": dt - t_load,
               "fit_final": float(res.fit[-1])}

    # FP64 view of the step (the per-subject R x R work is FP64-issue bound)
    fpk, fpk_kind = load_fp64_peak()
    flops = iteration_flops(X, R)
    fp_tf = flops / (ms_step * 1e-3) / 1e12
    fp64 = {"bound": "fp64", "achieved": fp_tf, "peak": fpk, "unit": "TFLOP/s", "frac": fp_tf / fpk,
            "flops_per_iter": flops, "peak_kind": fpk_kind, "model": "SURVEY.md 8(d) F_iter"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(X, R, cfg_id)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "sec_per_iter": ms_step * 1e-3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md 8d; inputs > L2, no flush needed)",
            "config": {"workload": CONFIG_NAME[cfg_id], "config_id": cfg_id, "rank": R, "K": X.K, "J": X.J,
                       "nnz": X.nnz, "rows": X.n_rows, "nonneg": True, "iterations_timed": args.steps,
                       "l2": "inputs larger than L2 (CSR+Q >> 126 MB)", "parallelism": f"subject-shard x{world}"},
            "ms_per_iter_all": [float(x) for x in ms], "fit_trace": [float(x) for x in fits],
            "iteration_gbs_algorithmic": iter_gbs, "iteration_hbm_frac": iter_gbs / peak,
            "roofline": roofline, "roofline_fp64": fp64, "kernel_ms_per_launch": {k: v[0] for k, v in ktimes.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "wall_s_timed": wall,
            "clocks": clk.summary(), "gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
