import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_04219_b200 as p2g
X = p2g.generate_baseline(2, 10)
H0, V0, W0 = p2g.init_factors(102, X.K, X.J, 10)
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
    res = ctx.fit(p2g.SolverConfig(rank=10, max_iters=5, tol=1e-300, nonneg=True), H0, V0, W0, want_q=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"load {t1-t0:.3f}s fit(5) {t2-t1:.3f}s  device ms/iter {np.round(res.ms, 2)}", flush=True)
