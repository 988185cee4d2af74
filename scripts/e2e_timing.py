"""e2e phase split at a BASELINE config (P2G_TIMING prints the library's own laps)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_04219_b200 as p2g
cfg = int(os.environ.get("CFG", "2")); R = int(os.environ.get("RANK", "10")); iters = int(os.environ.get("ITERS", "5"))
X = p2g.generate_baseline(cfg, R)
H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg, R).seed), X.K, X.J, R)
pin = {}
for name in ("subj_row_ptr", "row_ptr", "col_idx", "val"):
    a = getattr(X, name)
    t = torch.empty(a.shape, dtype={np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[a.dtype.type], pin_memory=True)
    t.numpy()[...] = a
    pin[name] = t
Xp = p2g.CSRTensor(X.J, *(pin[n].numpy() for n in ("subj_row_ptr", "row_ptr", "col_idx", "val")))
ctx = p2g.Context(0)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.load(Xp); torch.cuda.synchronize(); t1 = time.perf_counter()
    res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=iters, tol=1e-300, nonneg=True), H0, V0, W0, want_q=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"rep {rep}: load {t1-t0:.3f}s fit({iters}) {t2-t1:.3f}s  wall ms/iter {np.round(res.ms, 1)}", flush=True)
