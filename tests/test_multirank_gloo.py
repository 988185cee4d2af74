"""Multi-rank (N > 1) path on CPU: world_size 2 over torch.distributed gloo.

Each rank owns the subjects partition_weighted(nnz_k + I_k, world) gives it
(the libp2g host partition, bit-exact with the reference's parallel.hpp:51-79)
and runs the PARAFAC2-ALS iteration exactly as the GPU design distributes it
(DESIGN.md §6): Procrustes, projection, mode-3 MTTKRP and the W NNLS stay
shard-local; the only collectives are sum-allreduces of M1 (R x R), M2 (J x R)
and [gram(W), cross] (R x R + 1); the H / V updates are replicated.  The
oracle supplies the per-shard math; the fit trajectory must equal the
single-process oracle's.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_tensor(o, X, kb, ke):
    sub = X.subset(kb, ke)
    return o.Tensor.from_csr(sub.J, sub.subj_row_ptr, sub.row_ptr, sub.col_idx, sub.val)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1703_04219_b200 as p2g
        from tests.helpers import load_oracle

        o = load_oracle()

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        R = 4
        X = p2g.generate_baseline(1, R, K=120)
        w = (X.subject_nnz() + X.rows_of()).astype(np.uint64)
        parts = p2g.partition_weighted(w, world)
        kb, ke = parts[rank]
        T = _shard_tensor(o, X, kb, ke)
        H, V, W0 = p2g.init_factors(7, X.K, X.J, R)
        W = W0[kb:ke].copy()
        norm_x = float(allreduce(np.array([T.frobenius_sq()]))[0])
        gramW = allreduce(o.gram(W))
        fits = []
        for _ in range(4):
            Qp, flags, _r = o.procrustes_all(T, H, V, W)
            P = o.project_slices(T, Qp)
            args = (P["rank"], P["n_cols"], P["blocks"], P["cols"])
            m1 = allreduce(o.mttkrp(*args, H, V, W, 1))                 # sync point 1
            G1 = o.hadamard(gramW, o.gram(V))
            Hn = m1 @ o.pinv_small(G1)
            nH = np.linalg.norm(Hn, axis=0)
            nH[nH == 0] = 1.0
            Hn = Hn / nH
            Wn = W * nH
            M2 = allreduce(o.mttkrp(*args, Hn, V, Wn, 2))               # sync point 2
            gWn = np.outer(nH, nH) * gramW
            Vn = o.nnls_rowwise(o.hadamard(gWn, o.gram(Hn)), M2)
            nV = np.linalg.norm(Vn, axis=0)
            nV[nV == 0] = 1.0
            Vn = Vn / nV
            m3 = o.mttkrp(*args, Hn, Vn, Wn, 3)                         # shard-local
            W = o.nnls_rowwise(o.hadamard(o.gram(Vn), o.gram(Hn)), m3)  # shard-local
            gc = allreduce(np.append(o.gram(W).ravel(), np.sum(W * m3)))  # sync point 3
            gramW = gc[:-1].reshape(R, R)
            model = np.sum(o.hadamard(o.gram(Hn), o.gram(Vn)) * gramW)
            fits.append(1.0 - max(0.0, norm_x - 2 * gc[-1] + model) / norm_x)
            H, V = Hn, Vn
        q.put((rank, parts, fits))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_iteration_matches_single_process(world, p2g, oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    # every rank agrees on the partition and (bit-identically) on the fits
    assert all(o_[1] == out[0][1] for o_ in out)
    assert all(o_[2] == out[0][2] for o_ in out)
    # partition is the reference's (bit-exact) and covers all subjects
    X = p2g.generate_baseline(1, 4, K=120)
    w = (X.subject_nnz() + X.rows_of()).tolist()
    assert out[0][1] == [tuple(t) for t in oracle.partition_weighted(w, world)]
    # single-process oracle, same inputs
    H, V, W = p2g.init_factors(7, X.K, X.J, 4)
    T = oracle.Tensor.from_csr(X.J, X.subj_row_ptr, X.row_ptr, X.col_idx, X.val)
    ref = oracle.fit_parafac2(T, 4, max_iters=4, tol=1e-300, nonneg=True, H0=H, V0=V, W0=W)
    assert np.abs(np.array(out[0][2]) - np.array(ref["fit"])).max() < 1e-10
