"""Multi-rank path on the CPU (world_size 2 and 3, gloo): the row partition of
the C ABI (afn_shard_rows, host arithmetic) and the exchange choreography of
the sharded apply / PCG (include/afn.h "Multi-GPU") are run
with the oracle as the per-rank compute and torch.distributed all-gathers as
the exchanges, and must reproduce the single-process oracle.

The GPU path executes the same steps with NCCL broadcasts (or, in the
emulated communicator, device copies; tests/test_gpu_dist.py)."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(buf, ranges_of, R):
    """All-gather each rank's owned index ranges of a same-layout array."""
    t = torch.from_numpy(np.ascontiguousarray(buf))
    got = [torch.empty_like(t) for _ in range(R)]
    dist.all_gather(got, t)
    out = buf.copy()
    for s in range(R):
        for a, b in ranges_of(s):
            out[a:b] = got[s].numpy()[a:b]
    return out


def _worker(rank, R, port, n, k, w, l, mu, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=R)
    try:
        import oracle as O
        import paper_2304_05460_b200 as afn
        from synth import gen_small

        # NCCL unique id bootstrap over the process group (no GPU needed)
        uid = afn.bootstrap_unique_id(dist)
        ids = [None] * R
        dist.all_gather_object(ids, uid)
        assert len(uid) == afn.COMM_ID_BYTES and all(i == ids[0] for i in ids)

        X, b = gen_small(n, 3, seed=5)
        B = O.build_afn(X, l, mu, k, w)  # replicated build (oracle)
        N2 = n - k
        V, L, G = B["V"], B["L"], B["G"].tocsr()
        Gt = G.T.tocsr()
        sh = [afn.shard_rows(n, k, R, s) for s in range(R)]
        a0, na, b0, nb = sh[rank]
        lo, hi = b0 - k, b0 - k + nb
        own = np.r_[a0:a0 + na, b0:b0 + nb]

        def vec_rng(s):
            return [(sh[s][0], sh[s][0] + sh[s][1]), (sh[s][2], sh[s][2] + sh[s][3])]

        def lm_rng(s):
            return [(sh[s][0], sh[s][0] + sh[s][1])]

        def rows2_rng(s):
            return [(sh[s][2] - k, sh[s][2] - k + sh[s][3])]

        def apply(r):  # the V-form apply of abi.cu apply_perm, one rank's share
            r = _exchange(r, lm_rng, R)
            t = sla.solve_triangular(L, r[:k], lower=True)
            u = np.zeros(N2)
            u[lo:hi] = r[k + lo:k + hi] - V[:, lo:hi].T @ t
            u = _exchange(u, rows2_rng, R)
            y = np.zeros(N2)
            y[lo:hi] = G[lo:hi] @ u
            y = _exchange(y, rows2_rng, R)
            z = np.zeros(n)
            z[k + lo:k + hi] = Gt[lo:hi] @ y
            kp = np.zeros((R, k))
            kp[rank] = V[:, lo:hi] @ z[k + lo:k + hi]
            kp = _exchange(kp.reshape(-1), lambda s: [(s * k, (s + 1) * k)], R).reshape(R, k)
            v = t.copy()
            for s in range(R):  # rank order
                v = v - kp[s]
            z[:k] = sla.solve_triangular(L.T, v, lower=False)
            return z

        def reduce(x):  # dot partials summed in rank order
            g = _exchange(np.eye(R)[rank] * x, lambda s: [(s, s + 1)], R)
            tot = 0.0
            for s in range(R):
                tot += g[s]
            return tot

        # ---- sharded apply == single-process apply
        rng = np.random.default_rng(rank + 100)
        rfull = np.random.default_rng(7).standard_normal(n)
        r = np.where(np.isin(np.arange(n), own), rfull, rng.standard_normal(n))  # junk off-shard
        z = apply(r)
        z = _exchange(z, vec_rng, R)
        zo = O.apply_afn(B, rfull)
        assert np.linalg.norm(z - zo) <= 1e-11 * np.linalg.norm(zo)

        # ---- sharded kernel matvec rows: union of shards = full matvec
        Xp = B["Xp"]
        qv = np.zeros(n)
        qv[own] = O.kmv_rows(Xp, l, mu, rfull, own)
        qv = _exchange(qv, vec_rng, R)
        assert np.linalg.norm(qv - O.kmv(Xp, l, mu, rfull)) <= 1e-13 * np.linalg.norm(qv)

        # ---- sharded PCG (abi.cu afn_pcg_solve) vs the oracle's PCG
        bp = b[B["perm"]]
        x = np.zeros(n)
        rr = bp.copy()
        nb_ = np.sqrt(reduce(rr[own] @ rr[own]))
        zz = apply(rr)
        rz = reduce(rr[own] @ zz[own])
        p = np.zeros(n)
        p[own] = zz[own]
        it = 0
        for it in range(1, 501):
            p = _exchange(p, vec_rng, R)
            qq = np.zeros(n)
            qq[own] = O.kmv_rows(Xp, l, mu, p, own)
            alpha = rz / reduce(p[own] @ qq[own])
            x[own] += alpha * p[own]
            rr[own] -= alpha * qq[own]
            if np.sqrt(reduce(rr[own] @ rr[own])) / nb_ <= 1e-4:
                break
            zz = apply(rr)
            rz_new = reduce(rr[own] @ zz[own])
            p[own] = zz[own] + (rz_new / rz) * p[own]
            rz = rz_new
        x = _exchange(x, vec_rng, R)
        ao, repo, _ = O.afn_pcg_solve(X, b, l, mu, k, w, B=B)
        a = np.empty(n)
        a[B["perm"]] = x
        q.put((rank, it, repo["iterations"], float(np.linalg.norm(a - ao) / np.linalg.norm(ao))))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e), 0.0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("R,n,k,w", [(2, 400, 40, 20), (3, 301, 31, 16)])
def test_sharded_apply_and_pcg_match_oracle(R, n, k, w):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, R, port, n, k, w, 1.0, 1e-3, q)) for r in range(R)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(R)]
    for p in procs:
        p.join(timeout=60)
    for rank, it, ito, err in res:
        assert it != "error", ito
        assert it == ito, (rank, it, ito)  # same iteration count as one process
        assert err <= 1e-9, err


def test_shard_rows_partition():
    """Every row of the permuted order is owned by exactly one rank, landmark
    and non-landmark blocks are contiguous and balanced (+-1)."""
    import paper_2304_05460_b200 as afn
    for n, k in [(1, 1), (10, 10), (1000, 100), (16384, 2000), (1048576, 8000), (7, 3)]:
        for R in (1, 2, 3, 8):
            cover = np.zeros(n, int)
            for s in range(R):
                a0, na, b0, nb = afn.shard_rows(n, k, R, s)
                assert 0 <= a0 and a0 + na <= k and k <= b0 and b0 + nb <= n
                cover[a0:a0 + na] += 1
                cover[b0:b0 + nb] += 1
                assert abs(na - k / R) < 1 and abs(nb - (n - k) / R) < 1
            assert (cover == 1).all()
    with pytest.raises(afn.AfnError):
        afn.shard_rows(10, 11, 2, 0)
