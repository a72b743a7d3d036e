"""Test infrastructure: an in-process stand-in for a process group, so the row-partitioned engine
path (gs_part_*) can run several parts on ONE GPU. Each part is a host thread driving its own
engine context (own CUDA stream); the gs_comm hooks rendezvous on host barriers after
synchronising the caller's stream, then move bytes with device-to-device copies. No kernel ever
waits on another part's kernel (the GPU is never asked to co-schedule dependent grids).

The same hooks in production are distributed.TorchComm (NCCL / gloo, one process per GPU).
"""
from __future__ import annotations

import threading

import torch

from paper_2211_00805_b200 import _capi


class _Dev:
    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr or 0, False), "version": 3}


def _view(ptr, count, typestr="<f8"):
    return torch.as_tensor(_Dev(ptr, count, typestr), device="cuda")


class ThreadGroup:
    def __init__(self, nparts: int, timeout: float = 120.0):
        self.n = nparts
        self.barrier = threading.Barrier(nparts, timeout=timeout)
        self.slots = [None] * nparts

    def comm(self, rank: int) -> "RankComm":
        return RankComm(self, rank)

    def run(self, fn):
        """Run fn(rank, comm) on one thread per part; returns the per-rank results (or raises
        the first exception)."""
        out = [None] * self.n
        errs = [None] * self.n

        def body(r):
            try:
                torch.cuda.set_device(0)
                out[r] = fn(r, self.comm(r))
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errs[r] = e
                self.barrier.abort()

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(600)
        for e in errs:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in errs:
            if e is not None:
                raise e
        return out


class RankComm:
    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank = group, rank
        self.error = None
        self.calls = 0
        self.a2a_calls = 0
        self._stream = torch.cuda.Stream()

        def allreduce(user, buf, count, op, stream):
            try:
                self.calls += 1
                torch.cuda.ExternalStream(stream).synchronize()
                g = self.g
                mine = _view(buf, count)
                g.slots[self.rank] = mine
                g.barrier.wait()
                with torch.cuda.stream(self._stream):
                    res = g.slots[0].clone()
                    for q in range(1, g.n):  # rank order, identical on every rank
                        res = res + g.slots[q] if op == 0 else torch.maximum(res, g.slots[q])
                self._stream.synchronize()
                g.barrier.wait()
                with torch.cuda.stream(self._stream):
                    mine.copy_(res)
                self._stream.synchronize()
                return 0
            except BaseException as e:  # noqa: BLE001
                self.error = e
                self.g.barrier.abort()
                return 1

        def alltoallv(user, sendbuf, send_bytes, recvbuf, recv_bytes, nranks, stream):
            try:
                self.a2a_calls += 1
                torch.cuda.ExternalStream(stream).synchronize()
                g = self.g
                sb = [int(send_bytes[q]) for q in range(nranks)]
                rb = [int(recv_bytes[q]) for q in range(nranks)]
                g.slots[self.rank] = (sendbuf, sb)
                g.barrier.wait()
                off = 0
                with torch.cuda.stream(self._stream):
                    for q in range(nranks):
                        if rb[q]:
                            qptr, qsb = g.slots[q]
                            if qsb[self.rank] != rb[q]:
                                raise RuntimeError(f"rank {q} sends {qsb[self.rank]} bytes, "
                                                   f"rank {self.rank} expects {rb[q]}")
                            src = _view(qptr + sum(qsb[:self.rank]), rb[q], "|u1")
                            _view(recvbuf + off, rb[q], "|u1").copy_(src)
                        off += rb[q]
                self._stream.synchronize()
                g.barrier.wait()
                return 0
            except BaseException as e:  # noqa: BLE001
                self.error = e
                self.g.barrier.abort()
                return 1

        self._cbs = (_capi.ALLREDUCE_FN(allreduce), _capi.ALLTOALLV_FN(alltoallv))
        self.comm = _capi.GsComm(self._cbs[0], None, self._cbs[1])
