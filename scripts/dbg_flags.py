import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_04219_b200 as p2g
R = int(os.environ.get("RANK", "10")); cfg = int(os.environ.get("CFG", "2")); K = int(os.environ.get("K", "200000"))
X = p2g.generate_baseline(cfg, R, K=K)
H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg, R).seed), X.K, X.J, R)
ctx = p2g.Context(0)
ctx.load(X)
for it in range(1, 9):
    res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=it, tol=1e-300, nonneg=True), H0, V0, W0)
    print(it, "flags after iteration", np.bincount(np.asarray(res.flags), minlength=4), flush=True)
