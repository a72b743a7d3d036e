"""world_size-2 gloo tests (CPU) of the multi-rank host logic: member sharding, the gs_comm
allreduce hook implementation (host-buffer mode), and the sharded barycenter decomposition
(barycenter.cpp:75-86 split across ranks) emulated with the oracle's filter applies."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_00805_b200.distributed import TorchAllreduce, member_shard  # noqa: F401


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_member_shard_partition():
    for m in (1, 2, 7, 8, 16, 33):
        for world in (1, 2, 3, 4, 8):
            if world > m:
                continue
            spans = [member_shard(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _emulated_sharded_barycenter(fo, a, members, alphas, lo, hi, hook, max_iter, tol):
    """The engine's sharded sweep order (gs_cheb.cu gs_barycenter) on the CPU oracle."""
    import pyoracle as po  # noqa: F401  (filter applies come from fo)
    n = a.size
    M = members[lo:hi]
    al = alphas[lo:hi]
    W = np.ones_like(M)
    apply = lambda X: fo.apply(np.ascontiguousarray((a[:, None] * X.T)))  # n x m_local
    phi = apply(W).T
    bary = np.full(n, 1.0 / n)
    it = conv = 0
    err = np.inf
    for sweep in range(1, max_iter + 1):
        V = M / np.maximum(phi, 1e-300)
        psi = apply(V).T
        lb = np.zeros(n)
        for c in range(hi - lo):
            lb = lb + al[c] * np.log(np.minimum(np.maximum(psi[c], 1e-300), 1e300))
        hook(lb.ctypes.data, n, 0)  # allreduce(SUM) of the local log-sums
        bary = np.exp(lb - lb.max())
        bary = bary / bary.sum()
        W = bary[None, :] / np.maximum(psi, 1e-300)
        phi = apply(W).T
        e = np.array([max(np.abs(V[c] * phi[c] - M[c]).sum() for c in range(hi - lo))])
        hook(e.ctypes.data, 1, 1)  # allreduce(MAX) of the marginal error
        err, it = float(e[0]), sweep
        if err <= tol:
            conv = 1
            break
    b = bary / bary.sum()
    return b, it, conv, err


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests")):
            sys.path.insert(0, p)
        import pyoracle as po
        from helpers import random_connected_graph, random_distribution
        from paper_2211_00805_b200.rng import Rng

        hook = TorchAllreduce(device_buffers=False)
        x = np.arange(5, dtype=np.float64) * (rank + 1)
        assert hook(x.ctypes.data, 5, 0) == 0
        assert np.array_equal(x, np.arange(5) * sum(r + 1 for r in range(world)))
        y = np.array([float(rank)])
        hook(y.ctypes.data, 1, 1)
        assert y[0] == world - 1

        n, m = 60, 5
        r, c, v = random_connected_graph(n, 9)
        A = po.from_triplets(n, r, c, v)
        L, lam, _ = po.laplacian(A, 1)
        fo = po.Filter(L, 1, lam, 0.8, 30)
        rng = Rng(8)
        members = np.array([random_distribution(n, rng) for _ in range(m)])
        alphas = np.full(m, 1.0 / m)
        a = np.full(n, 1.0 / n)
        lo, hi = member_shard(m, world, rank)
        b, it, conv, err = _emulated_sharded_barycenter(fo, a, members, alphas, lo, hi, hook, 400, 1e-8)
        ref = po.barycenter(fo, a, members, None, 400, 1e-8)
        q.put((rank, float(np.abs(b - ref["barycenter"]).max() / ref["barycenter"].max()),
               it, ref["iterations"], conv, int(ref["converged"]), hook.calls))
    except BaseException as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_barycenter_gloo_world2():
    world = 2
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for res in out:
        assert len(res) == 7, res
        rank, rel, it, it_ref, conv, conv_ref, calls = res
        assert rel <= 1e-12, res
        assert it == it_ref and conv == conv_ref
        assert calls == 2 + 2 * it


def _part_worker(rank, world, port, q):
    """Row-partitioned Chebyshev apply (heat.cpp:116-131 split by rows) on the
    partition plan of tests/helpers.py, with the halo exchange through TorchComm.alltoallv
    (gloo, host buffers): the rows must match the oracle's unpartitioned apply."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for p in (root, os.path.join(root, "oracle"), os.path.join(root, "tests")):
            sys.path.insert(0, p)
        import pyoracle as po
        import scipy.sparse as sp
        from helpers import partition_plan, random_connected_graph
        from paper_2211_00805_b200.distributed import TorchComm

        n, B = 90, 2
        r, c, v = random_connected_graph(n, 13)
        L, lam, _ = po.laplacian(po.from_triplets(n, r, c, v), 0)
        fo = po.Filter(L, 0, lam, 1.0, 30)
        Ls = fo.scaled
        order = np.random.default_rng(3).permutation(n).astype(np.int32)  # any locality order
        plan = partition_plan(Ls.offs, Ls.cols, Ls.vals, order, world)[rank]
        nl, nh = plan["re"] - plan["rb"], plan["nh"]
        Lloc = sp.csr_matrix((plan["vals"], plan["cols"], plan["offs"]), shape=(nl, nl + nh))
        hook = TorchComm(device_buffers=False)

        def exchange(T):  # fill the halo rows of T (nl + nh rows) from their owners
            send = np.ascontiguousarray(np.concatenate([T[rows] for rows in plan["send_rows"]]))
            recv = np.empty((nh, B))
            sb = [len(rows) * B * 8 for rows in plan["send_rows"]]
            rb = [int(k) * B * 8 for k in plan["recv"]]
            assert hook.alltoallv(send.ctypes.data, sb, recv.ctypes.data, rb) == 0
            T[nl:] = recv

        X = np.random.default_rng(5).standard_normal((n, B))
        b, K = fo.coeffs, fo.degree
        T0 = np.zeros((nl + nh, B))
        T0[:nl] = X[plan["vertices"]]
        exchange(T0)
        T1 = np.zeros_like(T0)
        T1[:nl] = Lloc @ T0 - T0[:nl]
        acc = 0.5 * b[0] * T0[:nl] + b[1] * T1[:nl]
        Tm2, Tm1 = T0, T1
        for k in range(2, K + 1):
            exchange(Tm1)
            Tk = np.zeros_like(T0)
            Tk[:nl] = 2.0 * (Lloc @ Tm1 - Tm1[:nl]) - Tm2[:nl]
            acc = acc + b[k] * Tk[:nl]
            Tm2, Tm1 = Tm1, Tk
        ref = fo.apply(X)[plan["vertices"]]
        q.put((rank, float(np.abs(acc - ref).max() / np.abs(ref).max()), hook.a2a_calls, nh))
    except BaseException as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_row_partitioned_apply_gloo_world2():
    world = 2
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for res in out:
        assert len(res) == 4, res
        rank, err, calls, nh = res
        assert err <= 1e-12, res
        assert calls == 30 and nh > 0
