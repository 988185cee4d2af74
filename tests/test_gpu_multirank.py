"""libp2g's own multi-rank path (world_size 2), on one GPU.

Two processes, each with its own p2g context on cuda:0, joined by a gloo
process group that serves as the library's host-staged collective
(p2g_set_host_collective).  Each rank's kernels only wait on the host, never
on the other rank's kernels, so one GPU is safe (B200_PROFILING.md).  This
drives the code a multi-GPU run uses: partition_weighted sharding (load_csr
with the full tensor, and the shard-local load_shard), the per-iteration
allreduces of M1 / M2 / [gram(W), cross, error flags], the max-over-ranks
timing, and the collective error agreement.

Pins: the reference's thread-count invariance (test_solver.cpp:344-361, fits
at 1 vs 3 threads within 1e-9) -> 1 vs 2 ranks: fit trajectory within 1e-10,
H, V and the concatenated W within 1e-9.  A fault on one rank makes both
ranks raise (no hang).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {"cfg1": (1, 5, None), "cfg3": (3, 40, 400), "cfg2": (2, 10, 4000)}


def _worker(rank, world, port, outdir, case, mode):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    result = {}
    try:
        import paper_1703_04219_b200 as p2g

        cfg_id, R, K = CASES[case]
        X = p2g.generate_baseline(cfg_id, R, K=K)
        H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)

        def coll(buf, op):
            t = torch.from_numpy(buf)
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM)

        ctx = p2g.Context(0, rank, world, None)
        ctx.set_host_collective(coll)
        w = (X.subject_nnz() + X.rows_of()).astype(np.uint64)
        kb, ke = p2g.partition_weighted(w, world)[rank]
        cfg = p2g.SolverConfig(rank=R, max_iters=4, tol=1e-300, nonneg=True)
        try:
            if mode == "full":
                ctx.load(X)
                res = ctx.fit(cfg, H0, V0, W0)
            elif mode == "shard":
                ctx.load_shard(X.K, kb, ke, X.subset(kb, ke))
                res = ctx.fit(cfg, H0, V0, np.asfortranarray(W0[kb:ke]))
            elif mode == "fault":
                ctx.load(X)
                if rank == 1:
                    ctx.inject_fault(1, 2)
                res = ctx.fit(cfg, H0, V0, W0)
            elif mode == "short":  # only rank 1's shard holds a subject with I_k < R (its subject 3)
                S = X.subset(kb, ke)
                if rank == 1:
                    S = _truncate_subject(p2g, S, 3, R - 1)
                result["expect"] = kb + 3
                ctx.load_shard(X.K, kb, ke, S)
                res = ctx.fit(p2g.SolverConfig(rank=R, max_iters=2, tol=1e-300), H0, V0, W0[kb:ke])
            elif mode == "bench":
                ctx.load(X)
                ms, fits = ctx.bench_iterations(cfg, 3, H0, V0, W0, reset=True)
                result["ms"] = ms
                res = None
            if res is not None:
                kb2, ke2, _, _ = ctx.shard_info()
                result.update(fit=res.fit, H=res.H, V=res.V, W=res.W, kb=kb2, ke=ke2)
        except Exception as e:  # noqa: BLE001 - reported to the parent
            result["error"] = f"{type(e).__name__}: {e}"
        ctx.close()
    finally:
        np.save(os.path.join(outdir, f"r{rank}.npy"), result, allow_pickle=True)
        dist.destroy_process_group()


def _truncate_subject(p2g, S, j, rows):
    """S with subject j cut to its first `rows` rows (a shard-local edit)."""
    srp, rp = S.subj_row_ptr, S.row_ptr
    r0 = srp[j]
    keep = np.ones(S.n_rows, bool)
    keep[r0 + rows:srp[j + 1]] = False
    counts = np.diff(rp)[keep]
    ent = np.repeat(keep, np.diff(rp))
    new_srp = srp.copy()
    new_srp[j + 1:] -= srp[j + 1] - (r0 + rows)
    return p2g.CSRTensor(S.J, new_srp, np.concatenate([[0], np.cumsum(counts)]).astype(np.int64),
                         S.col_idx[ent].copy(), S.val[ent].copy())


def _run(case, mode):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d, case, mode), nprocs=2, join=True,
                           start_method="spawn")
        return [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True).item() for r in range(2)]


def _single(ctx, p2g, case):
    cfg_id, R, K = CASES[case]
    X = p2g.generate_baseline(cfg_id, R, K=K)
    H0, V0, W0 = p2g.init_factors(int(p2g.baseline_spec(cfg_id, R).seed), X.K, X.J, R)
    ctx.load(X)
    return ctx.fit(p2g.SolverConfig(rank=R, max_iters=4, tol=1e-300, nonneg=True), H0, V0, W0)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("case", ["cfg1", "cfg3", "cfg2"])
@pytest.mark.parametrize("mode", ["full", "shard"])
def test_two_ranks_match_one(ctx, p2g, case, mode):
    ref = _single(ctx, p2g, case)
    r0, r1 = _run(case, mode)
    assert "error" not in r0 and "error" not in r1, (r0.get("error"), r1.get("error"))
    assert r0["kb"] == 0 and r0["ke"] == r1["kb"] and r1["ke"] == ref.W.shape[0]
    # replicated state is bitwise identical on both ranks
    assert np.array_equal(r0["H"], r1["H"]) and np.array_equal(r0["V"], r1["V"])
    assert np.array_equal(r0["fit"], r1["fit"])
    assert np.abs(r0["fit"] - ref.fit).max() <= 1e-10
    assert _rel(r0["H"], ref.H) <= 1e-9 and _rel(r0["V"], ref.V) <= 1e-9
    assert _rel(np.vstack([r0["W"], r1["W"]]), ref.W) <= 1e-9


def test_fault_on_one_rank_raises_on_both():
    r0, r1 = _run("cfg1", "fault")
    for r in (r0, r1):
        assert r.get("error", "").startswith("NumericalError: NNLS did not converge"), r.get("error")


def test_validation_is_collective():
    """The I_k >= R check fails on rank 1 only; both ranks raise the same
    DataError naming the global subject (solver.hpp:116-122)."""
    r0, r1 = _run("cfg1", "short")
    assert r0.get("error") and r0["error"] == r1.get("error"), (r0.get("error"), r1.get("error"))
    assert r0["error"] == f"DataError: rank exceeds observations for subject {r1['expect']}: I_k = 4 < rank 5"


def test_bench_max_over_ranks():
    r0, r1 = _run("cfg1", "bench")
    assert "error" not in r0 and "error" not in r1
    assert np.array_equal(r0["ms"], r1["ms"]) and (r0["ms"] > 0).all()
