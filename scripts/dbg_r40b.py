"""R=40 cfg3/cfg5 prefixes: teacher-forced Procrustes and short fits vs the oracle."""
import os, sys
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
    ref = o.fit_parafac2(T, R, max_iters=3, tol=1e-300, nonneg=True, threads=16, H0=H0, V0=V0, W0=W0, dumps=True)
    ctx.load(X)
    for it, d in enumerate(ref["dumps"]):
        Q, flags, m1 = ctx.procrustes(d["H_in"], d["V_in"], d["W_in"])
        ofl = np.asarray(d["flags"])
        fl = np.asarray(flags)
        bad = np.where(np.isin(fl, (1, 3)) != np.isin(ofl, (1, 3)))[0]
        print(f"cfg{cfg_id} it{it}: Q rel {rel_err(Q, d['Q']):.2e} m1 rel {rel_err(m1, d['cp']['m1'] if 'cp' in d else d['m1']):.2e}"
              f" gpu flags {np.bincount(fl, minlength=4)} oracle flags {np.bincount(ofl, minlength=4)} deficient-mismatch {len(bad)}", flush=True)
    for n in (1, 2, 3):
        try:
            res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=n, tol=1e-300, nonneg=True), H0, V0, W0)
            print(f"  fit {n}: gpu {np.array(res.fit)} oracle {np.array(ref['fit'][:n])}", flush=True)
            d = ref["dumps"][n - 1]
            print(f"     H {rel_err(res.H, d['H']):.2e} V {rel_err(res.V, d['V']):.2e} W {rel_err(res.W, d['W']):.2e}", flush=True)
        except Exception as e:
            print(f"  fit {n}: FAILED {type(e).__name__}: {e}", flush=True)
