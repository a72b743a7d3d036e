"""GPU: the member-sharded barycenter through the NCCL allreduce hook (world_size 1 here -- the
gpurun box has one GPU; the multi-rank host logic is covered by test_distributed_cpu.py)."""
import socket

import numpy as np
import pytest

from helpers import engine_filter, random_connected_graph, random_distribution, rel

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_barycenter_nccl_world1(ctx):
    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200.distributed import sharded_sinkhorn_barycenter
    from paper_2211_00805_b200.rng import Rng

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        n, m = 150, 6
        r, c, v = random_connected_graph(n, 31)
        f, _ = engine_filter(r, c, v, n, 1, 0.7, 30)
        rng = Rng(77)
        fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(m)])
        a = np.full(n, 1.0 / n)
        ref = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(300, 1e-9))
        out = sharded_sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(300, 1e-9))
        assert out.iterations == ref.iterations and out.converged == ref.converged
        assert rel(out.barycenter.weights, ref.barycenter.weights) <= 1e-14
        for k in range(m):
            assert rel(out.scalings[k][0], ref.scalings[k][0]) <= 1e-14
    finally:
        dist.destroy_process_group()


def test_engine_nccl_comm_world1_graph_captured(ctx):
    """The engine's own NCCL communicator (gs_nccl_comm_create) at world 1: the sharded
    barycenter equals the unsharded one, and the sweeps are graph-captured with the collectives
    inside (the hooks run only while the two-sweep graph is captured, not once per sweep)."""
    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200.distributed import NcclComm, sharded_sinkhorn_barycenter
    from paper_2211_00805_b200.rng import Rng

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        n, m = 180, 5
        r, c, v = random_connected_graph(n, 41)
        f, _ = engine_filter(r, c, v, n, 1, 0.7, 30)
        rng = Rng(78)
        fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(m)])
        a = np.full(n, 1.0 / n)
        ref = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(300, 1e-11))
        comm = NcclComm(f._ctx)
        out = sharded_sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(300, 1e-11), comm=comm)
        assert out.iterations == ref.iterations and out.converged == ref.converged
        assert out.iterations > 20
        assert rel(out.barycenter.weights, ref.barycenter.weights) <= 1e-14
        for k in range(m):
            assert rel(out.scalings[k][0], ref.scalings[k][0]) <= 1e-14
        # 1 validation allreduce + 2 captured sweeps x (log-sum, error) = 5, whatever the sweep count
        assert comm.calls() == 5, comm.calls()
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rpc", [None, "4"])
@pytest.mark.parametrize("ranks", [2, 4])
def test_member_sharded_barycenter_threads(ctx, monkeypatch, ranks, rpc):
    """Member-sharded barycenter with 2 / 4 ranks (host threads on one GPU, each with its own
    engine context; tests/part_comm.py hooks) against the unsharded engine run: the log-sum is
    re-associated across ranks (barycenter.cpp:75-78), so results agree to <= 1e-12.
    GS_RPC=4 puts the 2-member shards on the large-shared-memory kernel k_cheb_lane, whose
    once-per-device function attribute several host threads then race to set."""
    if rpc:
        monkeypatch.setenv("GS_RPC", rpc)
    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200.distributed import sharded_sinkhorn_barycenter
    from paper_2211_00805_b200.rng import Rng
    from part_comm import ThreadGroup

    n, m = 220, 8
    r, c, v = random_connected_graph(n, 43)
    rng = Rng(79)
    members = [random_distribution(n, rng) for _ in range(m)]
    a = np.full(n, 1.0 / n)
    f0, _ = engine_filter(r, c, v, n, 1, 0.7, 30)
    ref = gs.sinkhorn_barycenter(f0, gs.DistributionFamily([gs.Distribution(x) for x in members]), a,
                                 gs.SinkhornParams(400, 1e-10))
    g = ThreadGroup(ranks)

    def body(rank, comm):
        ctx_r = gs.Context(0)
        f, _ = engine_filter(r, c, v, n, 1, 0.7, 30, ctx=ctx_r)
        fam = gs.DistributionFamily([gs.Distribution(x) for x in members])
        return sharded_sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(400, 1e-10), comm=comm)

    outs = g.run(body)
    for k, out in enumerate(outs):
        assert out.iterations == ref.iterations and out.converged == ref.converged
        assert rel(out.barycenter.weights, ref.barycenter.weights) <= 1e-12
        from paper_2211_00805_b200.distributed import member_shard
        lo, hi = member_shard(m, ranks, k)
        for j in range(lo, hi):
            assert rel(out.scalings[j][0], ref.scalings[j][0]) <= 1e-12


def test_member_sharded_validation_is_collective(ctx):
    """One rank's member fails validation (a negative weight): every rank raises the same errc and
    none waits forever in a collective (rank-local failures must be agreed)."""
    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi
    from paper_2211_00805_b200.distributed import member_shard
    from part_comm import ThreadGroup
    from paper_2211_00805_b200.rng import Rng
    import ctypes as C

    n, m, ranks = 120, 4, 2
    r, c, v = random_connected_graph(n, 47)
    rng = Rng(80)
    members = np.stack([random_distribution(n, rng) for _ in range(m)])
    a = np.full(n, 1.0 / n)
    g = ThreadGroup(ranks)

    def body(rank, comm):
        ctx_r = gs.Context(0)
        f, _ = engine_filter(r, c, v, n, 1, 0.7, 30, ctx=ctx_r)
        lo, hi = member_shard(m, ranks, rank)
        local = members[lo:hi].copy()
        if rank == 1:
            local[0, 3] = -local[0, 3]  # only rank 1 sees a bad member
        al = np.full(hi - lo, 1.0 / m)
        out = np.empty(n)
        it = np.zeros(1, np.int32)
        cv = np.zeros(1, np.int32)
        er = np.zeros(1)
        rc = ctx_r.lib.gs_barycenter(ctx_r.handle, f._h, a.ctypes.data, local.ctypes.data, hi - lo,
                                     al.ctypes.data, 100, 1e-9, _capi.GS_MEM_HOST, C.byref(comm.comm),
                                     out.ctypes.data, None, None, it.ctypes.data, cv.ctypes.data,
                                     er.ctypes.data)
        return rc, ctx_r.lib.gs_last_error(ctx_r.handle).decode()

    outs = g.run(body)
    assert outs[0][0] == outs[1][0] == 10, outs  # errc::invalid_argument + 1 on every rank
    assert "negative" in outs[1][1] and "another rank" in outs[0][1]


def test_row_partition_engine_nccl_world1_graph_captured(ctx):
    """Row-partitioned Sinkhorn through the engine's NCCL comm at world 1: sweeps are captured
    as CUDA graphs with the collectives inside (the comm is GS_COMM_GRAPH_SAFE) and v / w are
    bit-identical to the unpartitioned run."""
    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200.distributed import NcclComm, partitioned_sinkhorn
    from paper_2211_00805_b200.rng import Rng

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        n, P = 400, 3
        r, c, v = random_connected_graph(n, 53)
        f, _ = engine_filter(r, c, v, n, 1, 0.7, 30)
        rng = Rng(81)
        mus = [gs.Distribution(random_distribution(n, rng)) for _ in range(P)]
        nus = [gs.Distribution(random_distribution(n, rng)) for _ in range(P)]
        a = np.full(n, 1.0 / n)
        params = gs.SinkhornParams(300, 1e-10)
        ref = gs.geodesic_sinkhorn_batch(f, mus, nus, a, params)
        comm = NcclComm(f._ctx)
        part, res = partitioned_sinkhorn(f, mus, nus, a, params, comm=comm)
        vid = part.vertices
        for p in range(P):
            assert res[p].iterations == ref[p].iterations
            assert np.array_equal(res[p].v, ref[p].v[vid]) and np.array_equal(res[p].w, ref[p].w[vid])
            assert rel(res[p].cost, ref[p].cost) <= 1e-13
        # captured once: the hooks ran only while the two-sweep graph was built (plus the
        # validation / setup reductions), not once per sweep
        assert comm.calls() < 40, comm.calls()
        comm.close()
    finally:
        dist.destroy_process_group()
