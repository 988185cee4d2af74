"""Profiling driver: a K-subject prefix of a BASELINE config, N fit iterations."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_04219_b200 as p2g
cfg_id = int(os.environ.get("CFG", "3")); R = int(os.environ.get("RANK", "40"))
K = int(os.environ.get("K", "100000")); iters = int(os.environ.get("ITERS", "3"))
X = p2g.generate_baseline(cfg_id, R, K=K)
H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
ctx = p2g.Context(0)
ctx.load(X)
res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=iters, tol=1e-300, nonneg=True), H0, V0, W0, want_q=False)
print("fit", res.fit, "ms", res.ms)
