"""CPU: the windowed step kernel's host plan (paper_2211_00805_b200/csrc/gs_win.cu), checked
without a device. The kernel (gs_win.cuh) folds every CSR entry from the ring slot the plan
assigns it; these tests replay the producer/consumer protocol on the host and check that the
slot holds the entry's neighbour row under every interleaving the kernel allows (the producer
runs up to `stages - 1` blocks ahead of the consumers)."""
import ctypes as C

import numpy as np
import pytest

import pyoracle as po


def _lib():
    from paper_2211_00805_b200 import _capi
    return _capi.load()


def _graph(n, k=10, seed=1):
    from paper_2211_00805_b200 import workloads
    workloads.set_rng_class(po.Rng)
    roll = workloads.swiss_roll(n, seed)
    A, _ = po.knn_graph(roll.points, k, 1, 0.0)
    L, _, _ = po.laplacian(A, 0)
    return n, np.ascontiguousarray(L.offs, np.int32), np.ascontiguousarray(L.cols, np.int32)


def _plan(n, offs, cols, row_bytes, nctas):
    lib = _lib()
    p = C.c_void_p()
    sizes = np.zeros(7, np.int64)
    rc = lib.gs_win_plan_host(n, offs.ctypes.data, cols.ctypes.data, row_bytes, nctas, C.byref(p),
                              sizes.ctypes.data)
    if rc != 0:
        return rc, None
    W, nct, nb, nl, stages, lmax, npad = (int(x) for x in sizes)
    blk = np.zeros((nb, 8), np.int32)
    cta = np.zeros(nct + 1, np.int32)
    loads = np.zeros(nl, np.int32)
    poffs = np.zeros(n + 1, np.int32)
    slot = np.zeros(npad, np.uint16)
    own = np.zeros(n, np.uint16)
    lib.gs_win_plan_arrays(p, blk.ctypes.data, cta.ctypes.data, loads.ctypes.data, poffs.ctypes.data,
                           slot.ctypes.data, own.ctypes.data)
    lib.gs_win_plan_destroy(p)
    # padded CSR: row r starts at poffs[r] & ~3 and has poffs[r] & 3 padding entries at its end
    start = poffs & ~3
    assert np.all(start % 4 == 0) and start[-1] == npad
    assert np.array_equal(np.diff(start) - (poffs[:-1] & 3), np.diff(offs))
    # padded index of every real entry
    pidx = np.concatenate([start[r] + np.arange(offs[r + 1] - offs[r]) for r in range(n)]).astype(np.int64)
    return 0, dict(W=W, nctas=nct, stages=stages, lmax=lmax, blk=blk, cta=cta, loads=loads,
                   slot=slot, own=own, start=start, pidx=pidx)


def _replay(n, offs, cols, P):
    """The producer issues block j once block wait(j) is consumed (blk[:, 7]); consumers finish
    blocks in order. While block b is being read, every block up to jmax(b) -- the longest prefix
    whose waits are all < b -- may already have been issued. For every b and every issued prefix
    in [b, jmax(b)], each entry's ring slot holds its column and each row's own slot the row."""
    W, S = P["W"], P["stages"]
    blk, cta, loads = P["blk"], P["cta"], P["loads"]
    covered = np.zeros(n, bool)
    for c in range(P["nctas"]):
        b0, b1 = cta[c], cta[c + 1]
        wait = blk[b0:b1, 7]
        # the metadata stages bound the lead, and no block waits on itself or a later block
        assert np.all(wait >= np.arange(b0, b1) - S) and np.all(wait < np.arange(b0, b1))
        ring = np.full(W, -1, np.int64)
        applied = b0  # blocks whose loads are in the ring
        for b in range(b0, b1):
            row0, nrows, lbeg, nl, slot0, e0, e1, _ = blk[b]
            assert nl % 4 == 0 and nl <= P["lmax"] and slot0 % 4 == 0
            jmax = b
            while jmax + 1 < b1 and wait[jmax + 1 - b0] < b:
                jmax += 1
            for last_issued in range(b, jmax + 1):
                while applied <= last_issued:
                    s0, lb, nlb = blk[applied][4], blk[applied][2], blk[applied][3]
                    for i in range(nlb):
                        ring[(s0 + i) % W] = loads[lb + i]
                    applied += 1
                rows = np.arange(row0, row0 + nrows)
                assert np.all(ring[P["own"][rows]] == rows)
                assert e0 == P["start"][row0] and e1 == P["start"][row0 + nrows]
                ent = np.arange(offs[row0], offs[row0 + nrows])
                assert np.all(ring[P["slot"][P["pidx"][ent]]] == cols[ent])
            covered[row0:row0 + nrows] = True
    assert covered.all()
    # blocks tile each CTA's rows in order
    assert blk[0][0] == 0 and np.all(blk[1:, 0] == blk[:-1, 0] + blk[:-1, 1])


@pytest.mark.parametrize("row_bytes,nctas", [(512, 8), (256, 3), (128, 16)])
def test_win_plan_replay(row_bytes, nctas):
    n, offs, cols = _graph(3000)
    rc, P = _plan(n, offs, cols, row_bytes, nctas)
    assert rc == 0
    _replay(n, offs, cols, P)


def test_win_plan_on_bisection_order():
    n, offs, cols = _graph(4000)
    lib = _lib()
    order = np.zeros(n, np.int32)
    assert lib.gs_win_bisect_order_host(n, offs.ctypes.data, cols.ctypes.data, 32, order.ctypes.data) == 0
    assert np.array_equal(np.sort(order), np.arange(n))
    # renumber rows, keep every row's entries in the original column order (as gs_permute_graph)
    newpos = np.empty(n, np.int64)
    newpos[order] = np.arange(n)
    deg = np.diff(offs)[order]
    o2 = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    c2 = np.concatenate([newpos[cols[offs[v]:offs[v + 1]]] for v in order]).astype(np.int32)
    rc, P = _plan(n, o2, c2, 512, 4)
    assert rc == 0
    _replay(n, o2, c2, P)
    # the bisection order needs fewer loads than the caller's order
    rc0, P0 = _plan(n, offs, cols, 512, 4)
    assert len(P["loads"]) < len(P0["loads"])


def test_win_plan_rejects_oversized_row():
    # a star: vertex 0 adjacent to everybody -> one row needs more loads than a block holds
    n = 400
    rows = [[0] + list(range(1, n))] + [[0, i] for i in range(1, n)]
    offs = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    cols = np.concatenate(rows).astype(np.int32)
    rc, _ = _plan(n, offs, cols, 512, 2)
    from paper_2211_00805_b200 import _capi
    assert rc == _capi.GS_ERR_UNSUPPORTED
