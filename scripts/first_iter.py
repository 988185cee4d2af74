"""Per-phase device ms of the first (cold) iteration vs a steady one."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_04219_b200 as p2g
cfg_id = int(os.environ.get("CFG", "2")); R = int(os.environ.get("RANK", "10"))
X = p2g.generate_baseline(cfg_id, R)
H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
ctx = p2g.Context(0)
ctx.load(X)
cfg = p2g.SolverConfig(rank=R, max_iters=1, tol=1e-300, nonneg=True)
for rep in range(2):
    ctx.kernel_times()
    ms, _ = ctx.bench_iterations(cfg, 1, H0, V0, W0, reset=True)
    k1 = ctx.kernel_times()
    ms2, _ = ctx.bench_iterations(cfg, 1)
    k2 = ctx.kernel_times()
    print("first", np.round(ms, 2), {k: round(v[0], 2) for k, v in sorted(k1.items(), key=lambda x: -x[1][0])})
    print("next ", np.round(ms2, 2), {k: round(v[0], 2) for k, v in sorted(k2.items(), key=lambda x: -x[1][0])})
