"""GPU vs oracle NNLS on the exact G/rhs of the oracle's R=40 iterations (cfg3/cfg5 prefixes)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1703_04219_b200 as p2g
from helpers import load_oracle, oracle_from_csr, rel_err

o = load_oracle()
ctx = p2g.Context(0)
for cfg_id in (3, 5):
    R = 40
    X = p2g.generate_baseline(cfg_id, R, K=3000)
    H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
    T = oracle_from_csr(o, X)
    ref = o.fit_parafac2(T, R, max_iters=4, tol=1e-300, nonneg=True, threads=16, H0=H0, V0=V0, W0=W0, dumps=True)
    for it, d in enumerate(ref["dumps"]):
        H, V, W = np.asarray(d["H"]), np.asarray(d["V"]), np.asarray(d["W"])
        nh = np.asarray(d["norm_h"]); nv = np.asarray(d["norm_v"])
        Wp = np.asarray(d["W_in"]) * nh[None, :]
        G2 = (Wp.T @ Wp) * (H.T @ H)
        G3 = (V.T @ V) * (H.T @ H)
        for name, G, B in (("V", G2, np.asarray(d["m2"])), ("W", G3, np.asarray(d["m3"]))):
            ev = np.linalg.eigvalsh(G)
            kappa = ev.max() / max(ev.min(), 1e-300)
            xo = o.nnls_rowwise(G, B, 16)
            try:
                xg = ctx.nnls_rowwise(G, B)
                msg = f"rel {rel_err(xg, xo):.2e}"
            except Exception as e:
                msg = f"FAILED {type(e).__name__}: {e}"
            print(f"cfg{cfg_id} it{it} {name}: kappa {kappa:.2e} rows {B.shape[0]} {msg}", flush=True)
