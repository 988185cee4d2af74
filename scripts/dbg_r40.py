"""R=40 prefixes of cfg3/cfg5: GPU fit vs oracle fit, flag histogram."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1703_04219_b200 as p2g
from helpers import load_oracle, oracle_from_csr

oracle = load_oracle()
ctx = p2g.Context(0)
iters = int(os.environ.get("ITERS", "6"))
for cfg_id, K in [(3, 3000), (5, 3000)]:
    R = 40
    X = p2g.generate_baseline(cfg_id, R, K=K)
    seed = int(p2g.baseline_spec(cfg_id, R).seed)
    H0, V0, W0 = p2g.init_factors(seed, X.K, X.J, R)
    print(f"cfg{cfg_id} K={K} nnz={X.nnz} rows={X.subj_row_ptr[-1]}", flush=True)
    ctx.load(X)
    Q, flags, m1 = ctx.procrustes(H0, V0, W0)
    print("  flags at init:", np.bincount(np.asarray(flags), minlength=4), flush=True)
    try:
        t = time.time()
        res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=iters, tol=1e-300, nonneg=True), H0, V0, W0)
        print("  gpu fit ok", np.round(res.fit, 8), f"{time.time()-t:.2f}s", flush=True)
    except Exception as e:
        print("  gpu fit FAILED:", type(e).__name__, e, flush=True)
    T = oracle_from_csr(oracle, X)
    try:
        t = time.time()
        ref = oracle.fit_parafac2(T, R, max_iters=iters, tol=1e-300, nonneg=True, threads=16, H0=H0, V0=V0, W0=W0)
        print("  oracle fit ok", np.round(ref["fit"], 8), f"{time.time()-t:.2f}s", flush=True)
    except Exception as e:
        print("  oracle fit FAILED:", type(e).__name__, e, flush=True)
