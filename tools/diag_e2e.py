import sys, time, os, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2211_00805_b200 as gs
from paper_2211_00805_b200 import _capi, workloads
import bench
class A: pass
args = A(); args.config = 0; args.n = 2000; args.pairs = 1; args.sweeps = 100
cfg = bench.make_config(args)
ctx = gs.Context(0)
A_, sigma = gs.knn_gaussian_graph(cfg.roll.points, 10, ctx=ctx)
lap = gs.laplacian(A_, gs.LaplacianKind.combinatorial)
f = gs.HeatFilter(lap, 1.0, 30)
n, P = 2000, 1
lib = ctx.lib
def run(mem, pin):
    if mem == 1:
        dev = torch.device('cuda')
        M = torch.from_numpy(cfg.mus).to(dev); N = torch.from_numpy(cfg.nus).to(dev); a = torch.full((n,), 1/n, dtype=torch.float64, device=dev)
        outs = [torch.empty((P, n), dtype=torch.float64, device=dev) for _ in range(2)] + [torch.empty(P, dtype=torch.float64, device=dev) for _ in range(2)] + [torch.empty(P, dtype=torch.int32, device=dev) for _ in range(2)] + [torch.empty(P, dtype=torch.float64, device=dev)]
    else:
        mk = (lambda t: t.pin_memory()) if pin else (lambda t: t)
        M = mk(torch.from_numpy(cfg.mus)); N = mk(torch.from_numpy(cfg.nus)); a = mk(torch.full((n,), 1/n, dtype=torch.float64))
        outs = [mk(torch.empty((P, n), dtype=torch.float64)) for _ in range(2)] + [torch.empty(P, dtype=torch.float64) for _ in range(2)] + [torch.empty(P, dtype=torch.int32) for _ in range(2)] + [torch.empty(P, dtype=torch.float64)]
    fp, fs = C.c_int(), C.c_int()
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rc = lib.gs_sinkhorn(ctx.handle, f._h, a.data_ptr(), M.data_ptr(), N.data_ptr(), P, 100, 5e-324, 2, mem, *[o.data_ptr() for o in outs], C.byref(fp), C.byref(fs))
        torch.cuda.synchronize(); print(mem, pin, rep, rc, round((time.perf_counter()-t0)*1000, 2), 'ms')
run(1, False); run(0, True); run(0, False)
