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
