import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1703_04219_b200 as p2g
from helpers import load_oracle, oracle_from_csr
o = load_oracle(); ctx = p2g.Context(0)
R = 40
X = p2g.generate_baseline(5, R, K=1500)
H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(5, R).seed), X.K, X.J, R)
T = oracle_from_csr(o, X)
ref = o.fit_parafac2(T, R, max_iters=3, tol=1e-300, nonneg=True, threads=8, H0=H0, V0=V0, W0=W0, dumps=True)
ctx.load(X)
for it, d in enumerate(ref["dumps"]):
  Q, flags, m1   = ctx.procrustes(d["H_in"], d["V_in"], d["W_in"])
  H, V, W = (np.asarray(d[k]) for k in ("H_in", "V_in", "W_in"))
  Qo = np.asarray(d["Q"])
  rows = []
  for k in range(X.K):
      r0, r1 = X.subj_row_ptr[k], X.subj_row_ptr[k + 1]
      XV = np.zeros((r1 - r0, R))
      for r in range(r0, r1):
          p0, p1 = X.row_ptr[r], X.row_ptr[r + 1]
          XV[r - r0] = X.val[p0:p1] @ V[X.col_idx[p0:p1]]
      A = XV @ np.diag(W[k]) @ H.T
      U, s, Vt = np.linalg.svd(A, full_matrices=False)
      rho = int(np.count_nonzero(s * s > 1e-26 * s[0] ** 2))
      Ql = U[:, :rho] @ Vt[:rho]
      kapN = 1.0
      if rho < R:
          Ep = Vt[rho:].T
          LE = np.zeros((A.shape[0], R - rho)); LE[:R] = Ep
          N = LE - U[:, :rho] @ (U[:, :rho].T @ LE)
          Un, sn, Vnt = np.linalg.svd(N, full_matrices=False)
          kapN = sn[0] / sn[-1]
          Ql = Ql + (Un @ Vnt) @ Ep.T
      n = np.linalg.norm(Ql)
      eg = np.linalg.norm(Q[r0:r1] - Ql) / n
      eo = np.linalg.norm(Qo[r0:r1] - Ql) / n
      rows.append((max(eg, eo), k, s[0] / s[rho - 1], eg, eo, int(flags[k]), R - rho, kapN))
  rows.sort(reverse=True)
  for m, k, kap, eg, eo, f, nn, kapN in rows[:6]:
      print(f"it{it} k={k:5d} kappa={kap:9.3e} gpu-vs-lapack {eg:.2e} oracle-vs-lapack {eo:.2e} gpu flag {f} null {nn} kapN {kapN:.2e}")
