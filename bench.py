#!/usr/bin/env python
"""SPARTan PARAFAC2-ALS benchmark (BASELINE.json metric: sec/iter & nnz/s at
1/2/4/8 B200, % of HBM roofline).

A "step" is one full PARAFAC2-ALS outer iteration (Procrustes + MTTKRP modes
1-3 + H/V/W updates + fit, solver.hpp:274-318) over the whole synthetic
workload.  Default workload: BASELINE.json configs[3] ("cfg4": K=1M
subjects, J=5000, R=40, ~500M nnz, fp64) -- the north star's named config and
the largest that fits one GPU -- generated on the host (seeded, SURVEY.md
§8d); inputs are far larger than L2 (CSR 6.2 GB + Q 18.7 GB vs 126 MB), so
no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl b200|reference]

Under torchrun (N>1) each rank owns the subjects partition_weighted gives it
(a per-rank share of one fixed workload -> "scaling": "strong").
``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port, built -O3 -march=native on the box; the reference itself cannot
be compiled here) on the host cores, rank 0 only.  The CPU legs
(``--impl reference`` and the ``cpu_baseline`` of the default run) generate
their inputs with the oracle's own restatement of the BASELINE generator and
never load libp2g.
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



def procrustes_flops(K, n_rows, R):
    """Algorithmic FP64 flops of one Procrustes launch (the per-subject dense
    R x R work of SURVEY.md 8(d)'s F_iter): four I_k x R x R products
    (B = X~ T, M = B^T B, F = B^T X~, Q = B Z: 8 sum(I_k) R^2) plus the
    symmetric eigensolve and inverse square root (9 R^3 + 2 R^3 per subject)."""
    return 8.0 * n_rows * R * R + 11.0 * K * R ** 3


def polar_flops(K, R):
    """k_polar_small (R <= 16): the R x R eigensolve + inverse square root and
    the m1 partial per subject (11 R^3 + 2 R^3)."""
    return 13.0 * K * R ** 3


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


def workload_config(cfg_id, R, K, J, nnz, rows, world):
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": CONFIG_NAME[cfg_id], "config_id": cfg_id, "rank": R, "K": int(K), "J": int(J),
            "nnz": int(nnz), "rows": int(rows), "nonneg": True, "fp": "f64",
            "l2": "inputs larger than L2 (CSR+Q >> 126 MB), no flush",
            "parallelism": f"subject-shard x{world}"}


# ---------------------------------------------------------------------------
# CPU legs: the oracle (a restatement of the reference's CPU path; the
# reference itself cannot be compiled).  They import the oracle
# module only -- never libp2g -- and generate their inputs with the oracle's
# restatement of the BASELINE generator (oracle/baseline_gen.hpp).
# ---------------------------------------------------------------------------
def load_cpu_oracle():
    """The oracle built -O3 -march=native on THIS host (make -C oracle native);
    falls back to the portable -march=x86-64-v3 test build if that fails."""
    native = os.path.join(ROOT, "oracle", "_build_native")
    build = "native"
    try:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native"], check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, timeout=600)
        path = native
    except Exception:
        path, build = os.path.join(ROOT, "oracle", "_build"), "portable"
    if path not in sys.path:
        sys.path.insert(0, path)
    import p2oracle  # noqa: E402

    return p2oracle, ("-O3 -march=native" if build == "native" else "-O3 -march=x86-64-v3")


def oracle_sample(o, cfg_id, R, n_subjects, threads):
    """The first n_subjects of config cfg_id as an oracle Tensor, and the D2
    initial factors of the FULL workload restricted to those subjects."""
    spec = o.baseline_spec(cfg_id, R)
    J, srp, rp, ci, v = o.baseline_generate(cfg_id, R, n_subjects, threads)
    T = o.Tensor.from_csr(J, srp, rp, ci, v)
    H0, V0, W0 = o.baseline_init(spec["seed"], spec["K"], J, R, n_subjects)
    return T, H0, V0, W0, int(rp[-1]), int(srp[-1])


def cpu_iteration_rate(o, cfg_id, R, threads, target_s, warmup, steps):
    """Times `steps` oracle ALS iterations (after `warmup`, one fit) on a
    subject prefix sized so one iteration takes about target_s.  Step time is
    the reference's own per-phase timers (solver.hpp:278-297: procrustes +
    project + cp).  One part of an iteration does not scale with the number
    of subjects: the V solve over J rows (nnls_rowwise, cp.hpp:117-121; the
    oracle times it as ms_v_update).  The full-workload iteration time is
    therefore estimated as t_V + (nnz_full / nnz_sample) (t_step - t_V)."""
    spec = o.baseline_spec(cfg_id, R)
    K = spec["K"]
    probe = min(K, 400 if R > 16 else 4000)
    T, H0, V0, W0, _, _ = oracle_sample(o, cfg_id, R, probe, threads)
    r = o.fit_parafac2(T, R, max_iters=2, tol=1e-300, nonneg=True, threads=threads, H0=H0, V0=V0, W0=W0)
    step = r["ms_procrustes"][1] + r["ms_project"][1] + r["ms_cp"][1]
    fixed = r["ms_v_update"][1]
    per_subject = max(step - fixed, 1e-3) * 1e-3 / probe
    n = int(min(K, max(probe, (target_s - fixed * 1e-3) / per_subject)))
    T, H0, V0, W0, nnz, rows = oracle_sample(o, cfg_id, R, n, threads)
    t0 = time.perf_counter()
    r = o.fit_parafac2(T, R, max_iters=warmup + steps, tol=1e-300, nonneg=True, threads=threads, H0=H0, V0=V0,
                       W0=W0)
    wall = time.perf_counter() - t0
    sl = slice(warmup, warmup + steps)
    ph = {k: [float(x) for x in r[k][sl]] for k in ("ms_procrustes", "ms_project", "ms_cp", "ms_v_update")}
    ms_steps = [a + b + c for a, b, c in zip(ph["ms_procrustes"], ph["ms_project"], ph["ms_cp"])]
    ms = float(np.mean(ms_steps))
    ms_fixed = float(np.mean(ph["ms_v_update"]))
    return {"n_subjects": n, "nnz": nnz, "rows": rows, "ms_per_iter": ms, "nnz_per_s": nnz / (ms * 1e-3),
            "ms_per_iter_all": ms_steps, "phase_ms_mean": {k: float(np.mean(v)) for k, v in ph.items()},
            "ms_v_update": ms_fixed, "wall_s_fit": wall, "iterations_in_fit": warmup + steps,
            "fit": [float(x) for x in r["fit"]]}


def full_estimate(m, full_nnz):
    """Full-workload seconds per iteration from a prefix sample (see
    cpu_iteration_rate)."""
    fixed = m["ms_v_update"] * 1e-3
    return fixed + (m["ms_per_iter"] * 1e-3 - fixed) * full_nnz / max(m["nnz"], 1)


def cpu_baseline(cfg_id, R, full_nnz, full_K, target_s=6.0):
    """`cpu_baseline` of the default (N=1) line: the oracle port on a bounded
    prefix of the same workload, all host threads, 1 warm-up + 2 timed
    iterations, extrapolated to the full workload (cpu_iteration_rate)."""
    o, flags = load_cpu_oracle()
    threads = os.cpu_count() or 1
    m = cpu_iteration_rate(o, cfg_id, R, threads, target_s, warmup=1, steps=2)
    t_full = full_estimate(m, full_nnz)
    return {"value": full_nnz / t_full, "unit": "nnz/s", "cores": threads, "kind": "port",
            "sample": (f"first {m['n_subjects']} of {full_K} subjects of {CONFIG_NAME[cfg_id].split(' (')[0]} "
                       f"({m['nnz']} nnz), iterations 2-3 of a fit from the same initial factors; "
                       f"oracle/p2_oracle.hpp {flags}, {threads} threads; time = the reference's per-phase timers; "
                       f"value = full nnz / (t_V + nnz_full/nnz_sample (t_iter - t_V)), t_V the J-row V solve"),
            "sec_per_iter_sample": m["ms_per_iter"] * 1e-3, "sample_value": m["nnz_per_s"],
            "phase_ms_mean": m["phase_ms_mean"], "est_sec_per_iter_full": t_full, "cpu_model": cpu_model()}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    o, flags = load_cpu_oracle()
    cfg_id = args.config
    R = args.rank or CONFIG_RANK[cfg_id]
    threads = os.cpu_count() or 1
    # the full workload's shape for the config line (same config as the GPU arm)
    J, srp, rp, _, _ = o.baseline_generate(cfg_id, R, 0, threads)
    K, rows, nnz = len(srp) - 1, int(srp[-1]), int(rp[-1])
    del srp, rp
    # each step: one oracle ALS iteration over a bounded prefix, sized so the
    # whole --steps K --warmup W run takes a few minutes
    per_step = min(args.ref_seconds, 150.0 / max(args.steps + args.warmup, 1))
    m = cpu_iteration_rate(o, cfg_id, R, threads, per_step, warmup=max(args.warmup, 0), steps=args.steps)
    t_full = full_estimate(m, nnz)
    value = nnz / t_full
    sample = (f"first {m['n_subjects']} of {K} subjects ({m['nnz']} nnz) per step, "
              f"{args.warmup} warm-up + {args.steps} timed iterations of one fit; oracle port of the reference CPU "
              f"path (oracle/p2_oracle.hpp {flags}), {threads} threads; step time = the reference's per-phase "
              f"timers (solver.hpp:278-297); value = full nnz / (t_V + nnz_full/nnz_sample (t_iter - t_V)), "
              f"t_V the J-row V solve")
    line = {"metric": METRIC, "value": value, "unit": "nnz/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3,
            "sec_per_iter": t_full, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, SURVEY.md 8d)",
            "config": workload_config(cfg_id, R, K, J, nnz, rows, world),
            "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "phase_ms_mean": m["phase_ms_mean"], "ms_per_iter_all": m["ms_per_iter_all"],
            "wall_s_fit": m["wall_s_fit"], "sample_ms_per_iter": m["ms_per_iter"], "sample_value": m["nnz_per_s"],
            "ms_v_update": m["ms_v_update"], "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def pinned_like(torch, a):
    t = torch.empty(a.shape, dtype={np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[
        a.dtype.type], pin_memory=True)
    t.numpy()[...] = a
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
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

    # roofline of the dominant kernel (largest share of the step), against
    # the bound that applies to it: FP64 for the per-subject R x R Procrustes
    # work, HBM for the streaming passes
    peak, peak_kind = load_peaks()
    fpk, fpk_kind = load_fp64_peak()
    Xs = X.subset(kb, ke) if world > 1 else X
    ab = algorithmic_bytes(Xs, R)
    cand = {k: v for k, v in ktimes.items() if k in ("polar", "procrustes", "mode2", "mode3", "update_w")}
    dom = max(cand, key=lambda k: cand[k][0]) if cand else None
    roofline = None
    if dom:
        t_launch = cand[dom][0] * 1e-3
        akey = (dom + "_large") if (dom in ("mode2", "mode3") and R > 16) else dom
        traffic = None
        for tname in ("traffic_r02.json", "traffic_r01.json"):
            tpath = os.path.join(ROOT, "profiles", tname)
            if traffic is None and os.path.exists(tpath):
                try:
                    traffic = json.load(open(tpath)).get(f"cfg{cfg_id}", {}).get(dom)
                except Exception:
                    traffic = None
        share = sum(v[0] * v[1] for k, v in ktimes.items() if k == dom) / \
            max(sum(v[0] * v[1] for v in ktimes.values()), 1e-12)
        hbm_view = {"achieved": ab[akey] / t_launch / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": ab[akey] / t_launch / 1e9 / peak, "algorithmic_bytes_per_launch": ab[akey]}
        if dom in ("procrustes", "polar"):
            fl = procrustes_flops(Xs.K, Xs.n_rows, R) if dom == "procrustes" else polar_flops(Xs.K, R)
            ach = fl / t_launch / 1e12
            roofline = {"bound": "fp64", "kernel": dom, "achieved": ach, "peak": fpk, "unit": "TFLOP/s",
                        "frac": ach / fpk, "traffic": traffic, "peak_kind": fpk_kind,
                        "algorithmic_flops_per_launch": fl,
                        "flop_model": ("8 sum(I_k) R^2 + 11 K R^3" if dom == "procrustes" else "13 K R^3"),
                        "ms_per_launch": cand[dom][0], "share_of_step": share, "hbm_view": hbm_view,
                        "note": "fp64 has no tcgen05 kind (SURVEY F8); peak = measured DFMA rate"}
            # the pipe that actually limits the R = 40 kernel: shared-memory wavefronts of
            # the Jacobi rounds.  Count = ncu's l1tex shared wavefronts of one full-size launch
            # (profiles/ncu_r02_full.txt, iteration 4), peak = one wavefront per SM and clock.
            try:
                tr = json.load(open(os.path.join(ROOT, "profiles", "traffic_r02.json"))).get(f"cfg{cfg_id}", {})
                wf, wf_ms = tr.get(dom + "_smem_wavefronts"), tr.get(dom + "_ncu_ms")
            except Exception:
                wf = wf_ms = None
            if wf and wf_ms and world == 1:
                props = torch.cuda.get_device_properties(local)
                wf_peak = props.multi_processor_count * (clk.summary().get("sm_mhz") or 1965.0) * 1e6
                roofline["smem_view"] = {"bound": "shared-memory pipe", "wavefronts_per_launch": wf,
                                         "ncu_ms_per_launch": wf_ms, "achieved": wf / (wf_ms * 1e-3),
                                         "peak": wf_peak, "unit": "wavefronts/s",
                                         "frac": wf / (wf_ms * 1e-3) / wf_peak,
                                         "note": "count and duration of the same ncu-captured launch (iteration 4; "
                                                 "the sweep count, hence both, is data dependent)"}
    iter_gbs = ab["iteration"] / (ms_step * 1e-3) / 1e9

    # end-to-end through the public API, every byte the reference's
    # fit_parafac2 hands back included: pinned host CSR -> load -> fit ->
    # H, V, W and every Q_k back to pinned host memory
    e2e = None
    if not args.no_e2e:
        pin = {name: pinned_like(torch, getattr(X, name)) for name in ("subj_row_ptr", "row_ptr", "col_idx", "val")}
        Xp = p2g.CSRTensor(X.J, pin["subj_row_ptr"].numpy(), pin["row_ptr"].numpy(), pin["col_idx"].numpy(),
                           pin["val"].numpy())
        pinned_f = []
        for a in (H0, V0, W0):
            t = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
            v = t.numpy().reshape(a.shape[::-1]).T
            v[...] = a
            pinned_f.append((t, v))
        H0p, V0p, W0p = (v for _, v in pinned_f)
        outs = []
        for shp in ((R, R), (X.J, R), (ke - kb, R)):
            t = torch.empty(shp[0] * shp[1], dtype=torch.float64, pin_memory=True)
            outs.append((t, t.numpy().reshape(shp[::-1]).T))
        qt = torch.empty(nr * R, dtype=torch.float64, pin_memory=True)
        qv = qt.numpy().reshape(nr, R)
        e2e_iters = args.steps
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.load(Xp)
        t_load = time.perf_counter() - t0
        res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=e2e_iters, tol=1e-300, nonneg=True), H0p, V0p, W0p,
                      out=tuple(v for _, v in outs), q_out=qv)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            import torch.distributed as dist

            tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        h2d = (X.subj_row_ptr.nbytes + X.row_ptr.nbytes + X.col_idx.nbytes + X.val.nbytes + H0.nbytes + V0.nbytes
               + W0.nbytes)
        # whole-job bytes: every rank returns its shard's Q_k and W rows (and H, V, the trace)
        d2h = (res.H.nbytes + res.V.nbytes + 8 * X.K * R + 8 * X.n_rows * R + 4 * X.K + 8 * 3 * e2e_iters)
        e2e = {"value": X.nnz * e2e_iters / dt, "unit": "nnz/s", "h2d_bytes_per_step": h2d // e2e_iters,
               "d2h_bytes_per_step": d2h // e2e_iters, "iterations_per_call": e2e_iters, "sec_per_call": dt,
               "load_s": t_load, "fit_s": dt - t_load, "q_bytes": 8 * X.n_rows * R,
               "what": "load(pinned CSR) + fit_parafac2 with every Q_k, H, V, W returned to pinned host memory",
               "fit_final": float(res.fit[-1])}
        del pin, Xp, qt, qv, outs

    # FP64 view of the whole step (SURVEY.md 8(d) F_iter)
    flops = iteration_flops(X, R)
    fp_tf = flops / (ms_step * 1e-3) / 1e12
    fp64 = {"bound": "fp64", "achieved": fp_tf, "peak": fpk, "unit": "TFLOP/s", "frac": fp_tf / fpk,
            "flops_per_iter": flops, "peak_kind": fpk_kind, "model": "SURVEY.md 8(d) F_iter"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg_id, R, X.nnz, X.K)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "sec_per_iter": ms_step * 1e-3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md 8d; inputs > L2, no flush needed)",
            "config": workload_config(cfg_id, R, X.K, X.J, X.nnz, X.n_rows, world),
            "ms_per_iter_all": [float(x) for x in ms], "fit_trace": [float(x) for x in fits],
            "iteration_gbs_algorithmic": iter_gbs, "iteration_hbm_frac": iter_gbs / peak,
            "roofline": roofline, "roofline_fp64_step": fp64,
            "kernel_ms_per_launch": {k: v[0] for k, v in ktimes.items()},
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
