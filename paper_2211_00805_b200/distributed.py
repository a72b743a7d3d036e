"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL on NVLink/NVSwitch).

The only real exchange on the hot path is the member-sharded barycenter
(configs 2 and 4): every rank owns a contiguous share of the family's members and, per sweep,
  * allreduce(SUM) of the n-vector sum_i alpha_i ln clamp(psi_i) over ranks
    (barycenter.cpp:75-78; the reference's member-order sum is re-associated across ranks), and
  * allreduce(MAX) of the per-rank marginal error (barycenter.cpp:86),
after which every rank computes the same barycenter. Row-partitioned runs (config 3; the graph
split into contiguous row ranges, RowPartition) add one halo exchange per Chebyshev step
(`gs_comm.alltoallv`) and allreduces of the per-column reductions. The engine calls both through
the C ABI hooks; `TorchComm` implements them with torch.distributed on the engine's stream (NCCL
for device buffers, gloo for host buffers). Distance pairs (config 1) need no collective: ranks
run independent pair shards.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _capi
from .geosink import (BarycenterResult, Distribution, DistributionFamily, HeatFilter,
                      RowPartition, SinkhornParams, _f64, _ptr, _stack)


def member_shard(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous share [lo, hi) of m members for `rank` (sizes differ by at most one)."""
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3}


class _CudaBytes:
    """__cuda_array_interface__ byte view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "|u1",
                                         "data": (ptr or 0, False), "version": 3}


class TorchComm:
    """gs_comm hooks over torch.distributed (allreduce + alltoallv). Keeps the ctypes callbacks
    alive; an exception inside a hook is stored in `error` and re-raised by the caller."""

    def __init__(self, group=None, device_buffers: bool = True):
        import torch
        import torch.distributed as dist

        self._torch, self._dist, self._group = torch, dist, group
        self._device = device_buffers
        self.calls = 0
        self.error: Optional[BaseException] = None

        def _hook(user, buf, count, op, stream):
            try:
                self.calls += 1
                rop = dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX
                if self._device:
                    t = torch.as_tensor(_CudaArray(buf, count), device="cuda")
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                        dist.all_reduce(t, op=rop, group=self._group)
                else:
                    arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double)), shape=(count,))
                    t = torch.from_numpy(arr)
                    dist.all_reduce(t, op=rop, group=self._group)
                return 0
            except BaseException as e:  # surfaced by the caller after the engine returns
                self.error = e
                return 1

        def _a2a(user, sendbuf, send_bytes, recvbuf, recv_bytes, nranks, stream):
            try:
                self.a2a_calls += 1
                sb = [int(send_bytes[q]) for q in range(nranks)]
                rb = [int(recv_bytes[q]) for q in range(nranks)]
                if self._device:
                    snd = torch.as_tensor(_CudaBytes(sendbuf, sum(sb)), device="cuda")
                    rcv = torch.as_tensor(_CudaBytes(recvbuf, sum(rb)), device="cuda")
                    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                        dist.all_to_all_single(rcv, snd, output_split_sizes=rb,
                                               input_split_sizes=sb, group=self._group)
                else:
                    snd = torch.from_numpy(_host_bytes(sendbuf, sum(sb)))
                    rcv = torch.from_numpy(_host_bytes(recvbuf, sum(rb)))
                    dist.all_to_all_single(rcv, snd, output_split_sizes=rb, input_split_sizes=sb,
                                           group=self._group)
                return 0
            except BaseException as e:
                self.error = e
                return 1

        self.a2a_calls = 0
        self._cb = _capi.ALLREDUCE_FN(_hook)
        self._cb_a2a = _capi.ALLTOALLV_FN(_a2a)
        self.comm = _capi.GsComm(self._cb, None, self._cb_a2a)

    def __call__(self, buf_ptr: int, count: int, op: int, stream: int = 0) -> int:
        """Invoke the allreduce hook directly (used by host-side tests)."""
        return self._cb(None, buf_ptr, count, op, stream)

    def alltoallv(self, send_ptr: int, send_bytes, recv_ptr: int, recv_bytes, stream: int = 0) -> int:
        """Invoke the alltoallv hook directly (used by host-side tests)."""
        k = len(send_bytes)
        sb = (C.c_int64 * k)(*send_bytes)
        rb = (C.c_int64 * k)(*recv_bytes)
        return self._cb_a2a(None, send_ptr, sb, recv_ptr, rb, k, stream)


TorchAllreduce = TorchComm  # earlier name (allreduce-only hook)


class NcclComm:
    """The engine's own NCCL communicator (gs_nccl_comm_create, csrc/gs_nccl.cu): NCCL calls on
    the engine's stream, no host callback inside the sweep loop, CUDA-graph capture kept
    (GS_COMM_GRAPH_SAFE). torch.distributed is only the bootstrap that broadcasts rank 0's
    ncclUniqueId. `comm` is the gs_comm* to hand to the engine."""

    def __init__(self, ctx, group=None):
        import torch.distributed as dist

        self._ctx = ctx
        lib = ctx.lib
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        uid = C.create_string_buffer(_capi.GS_NCCL_UNIQUE_ID_BYTES)
        if rank == 0:
            ctx.check(lib.gs_nccl_unique_id(uid))
        box = [bytes(uid.raw)]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(box, src=src, group=group)
        uid = C.create_string_buffer(box[0], _capi.GS_NCCL_UNIQUE_ID_BYTES)
        self._ptr = C.c_void_p()
        ctx.check(lib.gs_nccl_comm_create(ctx.handle, uid, world, rank, C.byref(self._ptr)))
        self.world, self.rank = world, rank
        self.error = None

    @property
    def comm(self):
        return self._ptr

    def calls(self) -> int:
        """Host-side hook invocations so far (a captured sweep graph replays its collectives
        without invoking the hooks again)."""
        return int(self._ctx.lib.gs_nccl_comm_calls(self._ptr))

    def close(self):
        if self._ptr:
            self._ctx.lib.gs_nccl_comm_destroy(self._ptr)
            self._ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _comm_arg(hook):
    """The gs_comm* argument for a hook object (TorchComm / RankComm struct or NcclComm)."""
    return hook.comm if isinstance(hook, NcclComm) else C.byref(hook.comm)


def _host_bytes(ptr: int, count: int) -> np.ndarray:
    if count == 0:
        return np.zeros(0, np.uint8)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(count,))


def partitioned_sinkhorn(filter: HeatFilter, mus, nus, a, params: SinkhornParams = SinkhornParams(),
                         group=None, comm=None, **kw):
    """geodesic_sinkhorn_batch with the graph's rows split over the ranks of `group` (one halo
    exchange per Chebyshev step). Every rank passes the full inputs and gets (partition, results)
    where results[p].v / .w hold the rows listed by partition.vertices. `comm`: None (torch hooks)
    or an NcclComm (the engine's own NCCL communicator)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    part = RowPartition(filter, world, rank)
    vid = part.vertices
    take = lambda d: (d.weights if isinstance(d, Distribution) else _f64(d))[vid]
    hook = comm if comm is not None else TorchComm(group, device_buffers=True)
    try:
        res = part.sinkhorn([take(m) for m in mus], [take(v) for v in nus], _f64(a)[vid], params,
                            comm=hook.comm, **kw)
    except Exception:
        if hook.error is not None:
            raise hook.error
        raise
    return part, res


def sharded_sinkhorn_barycenter(filter: HeatFilter, family: DistributionFamily, a,
                                params: SinkhornParams = SinkhornParams(),
                                group=None, comm=None) -> BarycenterResult:
    """sinkhorn_barycenter (barycenter.cpp:45-99) with the members sharded over the ranks of
    `group`; every rank passes the full family and gets the full barycenter plus the scalings
    of its own members (others are None). `comm`: None (torch.distributed hooks), an NcclComm
    (the engine's NCCL communicator; sweeps stay CUDA-graph captured) or any object with a
    gs_comm `comm` attribute."""
    import torch.distributed as dist

    from .geosink import Error, errc

    ctx = filter._ctx
    n = filter.size()
    family.validate(n)
    world = dist.get_world_size(group) if comm is None or isinstance(comm, (TorchComm, NcclComm)) else comm.g.n
    rank = dist.get_rank(group) if comm is None or isinstance(comm, (TorchComm, NcclComm)) else comm.rank
    m = len(family.members)
    if world > m:  # every shard needs a member: an empty shard cannot take part in the sweeps
        raise Error(errc.invalid_argument,
                    f"InvalidArgument: {m} members cannot be sharded over {world} ranks")
    lo, hi = member_shard(m, world, rank)
    al = family.resolved_alphas()[lo:hi].copy()
    local = _stack(family.members[lo:hi], n)
    a = _f64(a)
    bary = np.empty(n)
    V = np.empty((hi - lo, n))
    W = np.empty((hi - lo, n))
    it = np.zeros(1, np.int32)
    conv = np.zeros(1, np.int32)
    err = np.zeros(1)
    hook = comm if comm is not None else TorchComm(group, device_buffers=True)
    rc = ctx.lib.gs_barycenter(ctx.handle, filter._h, _ptr(a), _ptr(local), hi - lo, _ptr(al),
                               int(params.max_iter), float(params.tol), _capi.GS_MEM_HOST,
                               _comm_arg(hook), _ptr(bary), _ptr(V), _ptr(W), _ptr(it),
                               _ptr(conv), _ptr(err))
    if hook.error is not None:
        raise hook.error
    ctx.check(rc)
    scal = [None] * m
    for c in range(lo, hi):
        scal[c] = (V[c - lo].copy(), W[c - lo].copy())
    return BarycenterResult(Distribution(bary, validate=False), scal, int(it[0]), bool(conv[0]),
                            float(err[0]))
