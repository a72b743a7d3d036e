#!/usr/bin/env python
"""Benchmark of the Chebyshev-Sinkhorn hot path (BASELINE.json config 1) on B200.

One "step" = one full batched geodesic Sinkhorn run (geodesic_sinkhorn_batch,
proj/src/transport.cpp:144-239): 64 source/target pairs on a 200,000-vertex swiss-roll kNN graph,
200 sweeps, each sweep = two 30-step Chebyshev heat applications over the 64-column batch.

  value  : sweeps/s over the whole job (N ranks x 200 sweeps x K steps / max-over-ranks time),
           inputs resident in HBM, device pointers through the C ABI.
  e2e    : the same metric through the public API with host buffers (H2D of mu/nu/a and D2H of
           v/w/cost/kl inside the timed region).
  roofline: the dominant kernel (k_cheb_step) -- algorithmic bytes per launch (SURVEY.md §8(d):
           nnz*(8+4) + 4(n+1) + 5*n*B*8) / its average CUDA-event duration in the timed region.
  cpu_baseline: the oracle restatement (oracle/, -O3 -march=native OpenMP) on this host, bounded
           sample of the same batch on the GPU-built graph.

Multi-GPU (torchrun): weak scaling, each rank runs its own 64 pairs on a replica of the graph,
no data-path collective (pairs are independent); timing is max over ranks.
`--impl reference` times the CPU reference path (the oracle port; the reference C++ library
cannot be built here) on the same config, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Chebyshev-Sinkhorn iterations/sec and achieved HBM GB/s vs peak, 1/2/4/8 B200"
UNIT = "sweeps/s"
TOL_RUN_ALL = 5e-324  # smallest positive double: the loop never exits early


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm),
                "reasons": sorted(reasons)}


class _StdoutToStderr:
    """Route fd 1 to stderr while NCCL initialises (its version banner would corrupt the single
    JSON line the driver reads from stdout)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _max_rel(a, b):
    ok = np.isfinite(a) & np.isfinite(b) & (b != 0)
    return float(np.max(np.abs(a[ok] - b[ok]) / np.abs(b[ok]))) if ok.any() else None


def algorithmic_bytes_per_step(n, nnz, B, sv=8):
    """matrix values + int32 indices + int32 offsets + 5 vector streams."""
    return nnz * (sv + 4) + 4 * (n + 1) + 5 * n * B * sv


# --------------------------------------------------------------------------- CPU legs
def cpu_sinkhorn_sample(L_host, lam, cfg, sweeps, native=True):
    """Time `sweeps` batched sweeps of the oracle on the GPU-built Laplacian; returns sweeps/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    lib = po.lib(native=native)
    Lo = po.CSR(L_host[0], L_host[1], L_host[2], L_host[3])
    fo = po.Filter(Lo, 0, lam, cfg.t, cfg.degree)
    n = cfg.roll.s.size
    a = np.full(n, 1.0 / n)
    t0 = time.perf_counter()
    res = po.sinkhorn_batch(fo, a, cfg.mus, cfg.nus, sweeps, TOL_RUN_ALL, flags=1, L=lib)
    dt = time.perf_counter() - t0
    return sweeps / dt, dt, res


def run_reference(args):
    """--impl reference: the CPU reference path (oracle port, all host threads), rank 0 only.
    Inputs come from the oracle's own Rng (oracle/pyoracle.py), so this arm never loads the
    product library."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from paper_2211_00805_b200 import workloads

    workloads.set_rng_class(po.Rng)
    lib = po.lib(native=True)
    cfg = make_config(args)
    t0 = time.perf_counter()
    A, sigma = po.knn_graph(cfg.roll.points, cfg.k, 1, 0.0)
    L, lam, rounds = po.laplacian(A, 0)
    fo = po.Filter(L, 0, lam, cfg.t, cfg.degree)
    setup_s = time.perf_counter() - t0
    n = args.n
    a = np.full(n, 1.0 / n)
    sweeps = max(2, args.ref_sweeps)

    def step():
        po.sinkhorn_batch(fo, a, cfg.mus, cfg.nus, sweeps, TOL_RUN_ALL, flags=1, L=lib)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = args.steps * sweeps / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(args),
        "operator": {"nnz_adjacency": int(A.nnz), "lambda_max_bound": lam, "lambda_rounds": rounds,
                     "sigma": sigma, "setup_s": setup_s, "built_by": "oracle (CPU kNN)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sweeps} sweeps of the {args.pairs}-pair batch per step on the full "
                                   f"n={n} graph (oracle restatement, OpenMP, -march=native)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": _product_lib_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


def _product_lib_mapped():
    """True when libgeosink_b200.so is mapped into this process (the reference arm must not)."""
    try:
        with open("/proc/self/maps") as f:
            return "libgeosink_b200" in f.read()
    except OSError:
        return None


def make_config(args, rank=0):
    from paper_2211_00805_b200 import workloads
    if args.config == 0:
        # config 0: one pair of s-bumps at 2pi / 4pi (width 0.5) on the n=2000 roll, 100 sweeps
        roll = workloads.swiss_roll(args.n, 1)
        mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)[None, :]
        nu = workloads.bump_in_s(roll, 4 * math.pi, 0.5)[None, :]
        return workloads.Config1(roll, mu, nu, sweeps=args.sweeps)
    return workloads.config1(args.n, args.pairs, seed=1, pair_seed=2 + 1000 * rank)


def config_dict(args):
    """The workload definition, identical in both arms (operator details that depend on how the
    graph was built -- lambda, sigma, timings -- live under "operator")."""
    return {
        "workload": (f"config{args.config}: swiss roll n={args.n}, k=10 symmetrised kNN, Gaussian weights "
                     f"sigma=median eps_10, combinatorial L, t=1, K=30, {args.pairs} pairs x "
                     f"{args.sweeps} sweeps (2 x {args.pairs}-column applies per sweep), fp64"),
        "n": args.n, "pairs": args.pairs, "sweeps_per_run": args.sweeps, "degree": 30,
        "stagnation_abort": "disabled (bench-only, DESIGN.md)",
        "tol": "5e-324 (all sweeps run)",
        "l2": "working set > 0.8 GB >> 126 MB L2; no flush needed between steps",
    }


# --------------------------------------------------------------------------- GPU arm
def run_engine(args):
    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi, workloads

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
    ctx = gs.Context(local)
    # a dedicated non-blocking stream shared by torch and the engine (the legacy default stream
    # serialises stream-ordered allocations and cannot be graph-captured)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib

    # ---- setup: graph build + Laplacian + lambda + filter, all on the device -------------------
    cfg = make_config(args, rank)
    t0 = time.perf_counter()
    A, sigma = gs.knn_gaussian_graph(cfg.roll.points, cfg.k, ctx=ctx)
    t_graph = time.perf_counter() - t0
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, cfg.t, cfg.degree)
    if os.environ.get("GS_BENCH_ORDER"):  # experiment: host-computed locality order
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import orders
        kind = os.environ["GS_BENCH_ORDER"]
        Ls = filt.scaled_laplacian()
        o = (orders.morton3(cfg.roll.points) if kind == "morton" else
             orders.bisect_order(Ls.row_offsets(), Ls.col_indices(), args.n,
                                 int(os.environ.get("GS_BENCH_LEAF", "64"))))
        filt.set_vertex_order(o, 0)
    t_prep = time.perf_counter() - t0 - t_graph
    n, P = args.n, args.pairs
    nnz_L = lap.matrix.stored_entries()

    dev = torch.device("cuda", local)
    M = torch.from_numpy(cfg.mus).to(dev)
    N = torch.from_numpy(cfg.nus).to(dev)
    a = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    ov = torch.empty((P, n), dtype=torch.float64, device=dev)
    ow = torch.empty_like(ov)
    oc = torch.empty(P, dtype=torch.float64, device=dev)
    ok = torch.empty_like(oc)
    oi = torch.empty(P, dtype=torch.int32, device=dev)
    occ = torch.empty_like(oi)
    oe = torch.empty_like(oc)
    import ctypes as C
    fp, fs = C.c_int(), C.c_int()
    flags = _capi.GS_FLAG_NO_STAGNATION_ABORT

    def step():
        ctx.check(lib.gs_sinkhorn(ctx.handle, filt._h, a.data_ptr(), M.data_ptr(), N.data_ptr(), P,
                                  args.sweeps, TOL_RUN_ALL, flags, _capi.GS_MEM_DEVICE,
                                  ov.data_ptr(), ow.data_ptr(), oc.data_ptr(), ok.data_ptr(),
                                  oi.data_ptr(), occ.data_ptr(), oe.data_ptr(), C.byref(fp),
                                  C.byref(fs)))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    l0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = ctx.launch_count() - l0
    # step-kernel launches per run: the initial apply plus 2 applies per sweep, K = 30 steps each
    steps_per_run = (1 + 2 * args.sweeps) * 30
    steps_total = args.steps * steps_per_run
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    value = world * args.sweeps * args.steps / (elapsed_ms / 1000.0)

    # ---- per-launch kernel time: one extra run of the same workload with per-kernel launches
    # (no CUDA graphs) and an event pair around EVERY step-kernel launch; the graph-replayed timed
    # region above cannot be split into launches. share_of_step = summed step-kernel time / that
    # run's own elapsed time, which must be <= 1.
    os.environ["GS_GRAPH"] = "0"
    ctx.set_timing(True)
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    step()
    k1.record(stream)
    torch.cuda.synchronize()
    step_n, step_ms = ctx.timing(0)
    epi_n, epi_ms = ctx.timing(1)
    ctx.set_timing(False)
    del os.environ["GS_GRAPH"]
    kt_elapsed = k0.elapsed_time(k1)
    share = step_ms / max(kt_elapsed, 1e-9)
    if args.config == 0:  # one persistent launch runs every sweep: time per Chebyshev step
        step_n = steps_per_run
    assert share <= 1.0 + 1e-6, ("step-kernel time exceeds its run", step_ms, kt_elapsed)

    # ---- roofline of the dominant kernel ------------------------------------------------------
    peak, peak_kind = peaks()
    bytes_step = algorithmic_bytes_per_step(n, nnz_L, P)
    avg_step_ms = step_ms / max(step_n, 1)
    achieved = bytes_step / (avg_step_ms / 1000.0) / 1e9
    # lower bound from the graph-replayed timed region: every step launch's bytes over the whole
    # elapsed time (finalize / control / epilogue kernels included)
    lb_achieved = bytes_step * steps_total / (elapsed_ms / 1000.0) / 1e9
    traffic = None
    ncu_info = None
    prof = os.path.join(ROOT, "profiles", "cheb_step_traffic.json")
    if args.config == 1 and os.path.exists(prof):  # ncu counters of the config-1 step kernel
        try:
            with open(prof) as f:
                ncu_info = json.load(f)
            traffic = ncu_info.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the public API with host buffers --------------------------------------------
    Mh = torch.from_numpy(cfg.mus).pin_memory()
    Nh = torch.from_numpy(cfg.nus).pin_memory()
    ah = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
    vh = torch.empty((P, n), dtype=torch.float64).pin_memory()
    wh = torch.empty_like(vh).pin_memory()
    ch = np.empty(P)
    kh = np.empty(P)
    ih = np.empty(P, np.int32)
    cvh = np.empty(P, np.int32)
    eh = np.empty(P)

    def step_host():
        ctx.check(lib.gs_sinkhorn(ctx.handle, filt._h, ah.data_ptr(), Mh.data_ptr(), Nh.data_ptr(),
                                  P, args.sweeps, TOL_RUN_ALL, flags, _capi.GS_MEM_HOST,
                                  vh.data_ptr(), wh.data_ptr(), ch.ctypes.data, kh.ctypes.data,
                                  ih.ctypes.data, cvh.ctypes.data, eh.ctypes.data, C.byref(fp),
                                  C.byref(fs)))

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    step_host()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    barrier()
    e2e_value = world * args.sweeps * e2e_steps / e2e_s
    h2d = 2 * P * n * 8 + n * 8
    d2h = 2 * P * n * 8 + P * (8 + 8 + 4 + 4 + 8)

    def run_sk(Mt, Nt, sweeps, flg, tol=TOL_RUN_ALL):
        """One engine call on device inputs (P_ = rows of Mt); returns host results or the errc."""
        P_ = Mt.shape[0]
        v_ = torch.empty((P_, n), dtype=torch.float64, device=dev)
        w_ = torch.empty_like(v_)
        c_ = torch.empty(P_, dtype=torch.float64, device=dev)
        k_ = torch.empty_like(c_)
        e_ = torch.empty_like(c_)
        i_ = torch.empty(P_, dtype=torch.int32, device=dev)
        cv_ = torch.empty_like(i_)
        fp_, fs_ = C.c_int(-1), C.c_int(-1)
        rc = lib.gs_sinkhorn(ctx.handle, filt._h, a.data_ptr(), Mt.data_ptr(), Nt.data_ptr(), P_,
                             sweeps, tol, flg, _capi.GS_MEM_DEVICE, v_.data_ptr(), w_.data_ptr(),
                             c_.data_ptr(), k_.data_ptr(), i_.data_ptr(), cv_.data_ptr(),
                             e_.data_ptr(), C.byref(fp_), C.byref(fs_))
        torch.cuda.synchronize()
        if rc != 0:
            return {"errc": lib.gs_last_error(ctx.handle).decode(),
                    "rc": int(rc), "fail_pair": fp_.value, "fail_sweep": fs_.value}
        return {"v": v_.cpu().numpy(), "w": w_.cpu().numpy(), "cost": c_.cpu().numpy(),
                "iterations": i_.cpu().numpy()}

    # well-posed companion pairs on the same graph (workloads.bump_mixture_companions: every
    # target bump within the K-hop reach of its source bump, so the reference converges instead
    # of raising Disconnected; SURVEY §7 hard part 1)
    cmus, cnus = workloads.bump_mixture_companions(cfg.roll, P, seed=7 + 1000 * rank)
    Mc = torch.from_numpy(cmus).to(dev)
    Nc = torch.from_numpy(cnus).to(dev)

    # ---- fp32 mode (config 1 is specified "fp64 and fp32"; DESIGN.md §4 "Precision") ----------
    fp32 = None
    if not args.no_fp32:
        flags32 = flags | _capi.GS_FLAG_FP32
        r64 = run_sk(Mc, Nc, args.sweeps, flags)
        r32 = run_sk(Mc, Nc, args.sweeps, flags32)  # also the warm-up of the 32-bit instantiation
        torch.cuda.synchronize()
        barrier()
        ctx.set_timing(True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        k32 = max(1, min(args.steps, 2))

        def step32():
            ctx.check(lib.gs_sinkhorn(ctx.handle, filt._h, a.data_ptr(), Mc.data_ptr(), Nc.data_ptr(),
                                      P, args.sweeps, TOL_RUN_ALL, flags32, _capi.GS_MEM_DEVICE,
                                      ov.data_ptr(), ow.data_ptr(), oc.data_ptr(), ok.data_ptr(),
                                      oi.data_ptr(), occ.data_ptr(), oe.data_ptr(), C.byref(fp),
                                      C.byref(fs)))

        e0.record(stream)
        for _ in range(k32):
            step32()
        e1.record(stream)
        torch.cuda.synchronize()
        n32, ms32 = ctx.timing(0)
        ctx.set_timing(False)
        el32 = max_over_ranks(e0.elapsed_time(e1))
        bytes32 = nnz_L * (4 + 4) + 4 * (n + 1) + 5 * n * P * 4
        c64 = r64.get("cost")
        c32 = r32.get("cost")
        # config 1 as specified, reference semantics (stagnation abort on): the 32-bit mode must
        # stop at the same pair with the same errc as fp64
        spec64 = run_sk(M, N, args.sweeps, 0, tol=1e-9)
        spec32 = run_sk(M, N, args.sweeps, _capi.GS_FLAG_FP32, tol=1e-9)
        strip = lambda r: {k: r[k] for k in ("rc", "fail_pair", "fail_sweep", "errc") if k in r} or \
            {"rc": 0, "iterations": int(r["iterations"].max())}
        fp32 = {"storage": "32-bit words: sign + fp64 exponent + 20 fraction bits (DESIGN.md §4)",
                "inputs": f"{P} well-posed companion pairs on the same graph, {args.sweeps} sweeps",
                "value": world * args.sweeps * k32 / (el32 / 1000.0), "unit": UNIT, "steps": k32,
                "avg_step_kernel_ms": ms32 / max(n32, 1) if n32 else None,
                "bytes_per_launch": bytes32,
                "max_rel_cost_vs_fp64": _max_rel(c32, c64) if c32 is not None and c64 is not None else None,
                "tolerance": 1e-4,
                "finite_costs": int(np.isfinite(c32).sum()) if c32 is not None else 0, "pairs": int(P),
                "as_specified_abort_on": {"fp64": strip(spec64), "fp32": strip(spec32),
                                          "same_outcome": strip(spec64) == strip(spec32)}}

    # ---- CPU baseline (rank 0, N = 1) and results parity ----------------------------------------
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as po
        offs = lap.matrix.row_offsets().copy()
        cols = lap.matrix.col_indices().copy()
        vals = lap.matrix.values().copy()
        sweeps = args.cpu_sweeps
        v, dt, ref = cpu_sinkhorn_sample((n, offs, cols, vals), lap.lambda_max_bound, cfg, sweeps)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"{sweeps} sweep(s) of the same {P}-pair batch on the GPU-built n={n} "
                         f"graph, oracle restatement -O3 -march=native OpenMP ({dt:.1f} s)"}
        # (1) the timed workload itself, first sweep(s), all 64 pairs: bit-identical v / w
        r1 = run_sk(M, N, sweeps, flags)
        parity = {"against": "oracle restatement (oracle/), same GPU-built Laplacian, same inputs",
                  "timed_workload": {"sweeps": sweeps, "pairs": int(P),
                                     "v_w_bit_identical": bool(np.array_equal(r1["v"], ref["v"]) and
                                                               np.array_equal(r1["w"], ref["w"])),
                                     "max_rel_cost": _max_rel(r1["cost"], ref["cost"])}}
        # (2) all sweeps on well-posed companion pairs (reference semantics, abort on): every
        # cost within 1e-9 relative, v / w bit-identical
        pp = min(P, args.parity_pairs)
        lib_o = po.lib(native=True)
        fo = po.Filter(po.CSR(n, offs, cols, vals), 0, lap.lambda_max_bound, cfg.t, cfg.degree)
        t0p = time.perf_counter()
        refc = po.sinkhorn_batch(fo, np.full(n, 1.0 / n), cmus[:pp], cnus[:pp], args.sweeps, 1e-9,
                                 flags=0, L=lib_o)
        dtp = time.perf_counter() - t0p
        rc_ = run_sk(Mc[:pp].contiguous(), Nc[:pp].contiguous(), args.sweeps, 0, tol=1e-9)
        parity["companion_full_run"] = {
            "pairs": pp, "max_sweeps": args.sweeps, "tol": 1e-9,
            "iterations_engine": rc_["iterations"].tolist(),
            "iterations_oracle": refc["iterations"].tolist(),
            "v_w_bit_identical": bool(np.array_equal(rc_["v"], refc["v"]) and np.array_equal(rc_["w"], refc["w"])),
            "max_rel_cost": _max_rel(rc_["cost"], refc["cost"]), "tolerance": 1e-9,
            "oracle_s": dtp}

    legs = None
    if args.config == 1 and not args.no_legs:
        legs = partitioned_legs(args, ctx, stream, world, rank, local)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_dict(args),
            "operator": {"nnz_adjacency": int(A.stored_entries()), "nnz_L": int(nnz_L),
                         "lambda_max_bound": lap.lambda_max_bound, "lambda_rounds": lap.power_rounds,
                         "sigma": sigma, "graph_build_s": t_graph, "prepare_s": t_prep,
                         "built_by": "engine (device kNN)",
                         "parallelism": f"replicas x{world} (pairs per rank)",
                         "column_sweeps_per_s": value * P},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": ("k_cheb_win<double, 64, *> (windowed Chebyshev step: one CTA per SM, "
                                    "neighbour rows staged by TMA gather4 into a shared-memory ring)"
                                    if args.config == 1 else
                                    "k_sk_persist (every sweep in one 16-CTA cluster kernel, T pushed between "
                                    "CTAs with st.async; latency-bound: the 0.39 MB working set lives in shared "
                                    "memory; avg_launch_ms = kernel time per Chebyshev step)"),
                         "bytes_per_launch": bytes_step, "avg_launch_ms": avg_step_ms,
                         "launches_timed": step_n,
                         "timing": "event pair around every step launch of one full run with "
                                   "per-kernel launches (GS_GRAPH=0)",
                         "share_of_step": share,
                         "lower_bound_from_timed_region": {
                             "achieved": lb_achieved, "frac": lb_achieved / peak,
                             "how": "step launches x bytes / elapsed of the graph-replayed timed region"},
                         "ncu": ncu_info},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "epilogue_kernels": {"launches": epi_n, "ms": epi_ms},
            "cpu_baseline": cpu,
            "parity": parity,
            "fp32_mode": fp32,
            "partitioned": legs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- N-GPU data planes
def partitioned_legs(args, ctx, stream, world, rank, local):
    """Strong-scaling legs of the two partitioned data planes, run after the main
    measurement at every N, so a 1/2/4/8-GPU sweep of the default bench sees both:
      * member_sharded: config-2 shape (R^30 mixture, 20 clusters, k = 15, t = 0.5, K = 30,
        8 members) at n = --legs-bary-n; members split over the ranks, per sweep one allreduce of
        the n-vector log-sum and one of the (error, status) pair over the engine's NCCL comm,
        sweeps CUDA-graph captured with the collectives inside;
      * row_partitioned: config-3 shape (swiss roll, k = 10, t = 1, K = 30, fp32, one pair) at
        n = --legs-rows-n; rows split over the ranks, one neighbour-only halo exchange per
        Chebyshev step (ncclSend/Recv), column reductions allreduced.
    At N = 1 both run unpartitioned (no comm). Times are device events, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi, workloads
    from paper_2211_00805_b200.distributed import NcclComm, member_shard

    dev = torch.device("cuda", local)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    comm = NcclComm(ctx) if world > 1 else None
    out = {}
    # ---- member-sharded barycenter ------------------------------------------------------------
    n, m, sweeps = args.legs_bary_n, 8, args.legs_sweeps
    cfg = workloads.config2(n, m)
    A, _ = gs.knn_gaussian_graph(cfg.mix.points, cfg.k, ctx=ctx)
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, cfg.t, cfg.degree)
    lo, hi = member_shard(m, world, rank)
    Ml = torch.from_numpy(np.ascontiguousarray(cfg.members[lo:hi])).to(dev)
    al = torch.full((hi - lo,), 1.0 / m, dtype=torch.float64, device=dev)
    a = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    bary = torch.empty(n, dtype=torch.float64, device=dev)
    it, cv, er = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1)

    def run_bary():
        ctx.check(ctx.lib.gs_barycenter_ex(ctx.handle, filt._h, a.data_ptr(), Ml.data_ptr(), hi - lo,
                                           al.data_ptr(), sweeps, TOL_RUN_ALL, _capi.GS_MEM_DEVICE,
                                           comm.comm if comm else None, 0, bary.data_ptr(), None,
                                           None, it.ctypes.data, cv.ctypes.data, er.ctypes.data))

    ms = timed(run_bary, 2)
    out["member_sharded"] = {
        "workload": f"config-2 shape: R^30 mixture n={n}, k=15, t=0.5, K=30, {m} members x {sweeps} sweeps",
        "value": 2 * sweeps / (ms / 1000.0), "unit": "barycenter sweeps/s", "scaling": "strong",
        "members_per_rank": hi - lo, "comm": "engine NCCL (graph-captured allreduce)" if comm else "none (1 rank)"}
    del filt, lap, A
    # ---- row-partitioned fp32 Sinkhorn --------------------------------------------------------
    n = args.legs_rows_n
    roll = workloads.swiss_roll(n, 1)
    A, _ = gs.knn_gaussian_graph(roll.points, 10, ctx=ctx)
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, 1.0, 30)
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5)
    part = gs.RowPartition(filt, world, rank, ctx=ctx) if world > 1 else None
    vid = part.vertices.astype(np.int64) if part is not None else np.arange(n)
    Md = torch.from_numpy(mu[vid].copy()).to(dev)
    Nd = torch.from_numpy(nu[vid].copy()).to(dev)
    ad = torch.full((vid.size,), 1.0 / n, dtype=torch.float64, device=dev)
    vd = torch.empty(vid.size, dtype=torch.float64, device=dev)
    wd = torch.empty_like(vd)
    dsc = torch.empty(3, dtype=torch.float64, device=dev)
    dsi = torch.empty(2, dtype=torch.int32, device=dev)
    fp, fs = C.c_int(), C.c_int()
    flags = _capi.GS_FLAG_NO_STAGNATION_ABORT | _capi.GS_FLAG_FP32

    def run_rows():
        p0, pi = dsc.data_ptr(), dsi.data_ptr()
        outs = (vd.data_ptr(), wd.data_ptr(), p0, p0 + 8, pi, pi + 4, p0 + 16, C.byref(fp), C.byref(fs))
        if part is None:
            rc = ctx.lib.gs_sinkhorn(ctx.handle, filt._h, ad.data_ptr(), Md.data_ptr(), Nd.data_ptr(), 1,
                                     sweeps, TOL_RUN_ALL, flags, _capi.GS_MEM_DEVICE, *outs)
        else:
            rc = ctx.lib.gs_part_sinkhorn(ctx.handle, part._h, comm.comm, ad.data_ptr(), Md.data_ptr(),
                                          Nd.data_ptr(), 1, sweeps, TOL_RUN_ALL, flags,
                                          _capi.GS_MEM_DEVICE, *outs)
        ctx.check(rc)

    ms = timed(run_rows, 2)
    out["row_partitioned"] = {
        "workload": f"config-3 shape: swiss roll n={n}, k=10, t=1, K=30, fp32 (32-bit words), 1 pair x {sweeps} sweeps",
        "value": 2 * sweeps / (ms / 1000.0), "unit": "sweeps/s", "scaling": "strong",
        "rows_per_rank": int(vid.size),
        "comm": "engine NCCL (neighbour-only send/recv halo per step)" if comm else "none (1 rank)"}
    if comm:
        comm.close()
    return out


# --------------------------------------------------------------------------- config 2 (barycenter)
def run_engine_bary(args):
    """Config 2: member-sharded barycenter. Every rank builds the same graph; members are split
    over the ranks; per sweep one NCCL allreduce(SUM) of the n-vector log-sum and one
    allreduce(MAX) of the marginal error (paper_2211_00805_b200/distributed.py). Strong scaling:
    the 8-member family is fixed, value = barycenter sweeps/s."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi, workloads
    from paper_2211_00805_b200.distributed import NcclComm, member_shard

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    with _StdoutToStderr():
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % _free_port(),
                                    rank=0, world_size=1, device_id=torch.device("cuda", local))
        dist.barrier()
    ctx = gs.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    cfg = workloads.config2(args.n, args.members)
    t0 = time.perf_counter()
    A, sigma = gs.knn_gaussian_graph(cfg.mix.points, cfg.k, ctx=ctx)
    t_graph = time.perf_counter() - t0
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, cfg.t, cfg.degree)
    if os.environ.get("GS_BENCH_ORDER") == "bisect":  # experiment: host-computed locality order
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import orders
        Ls = filt.scaled_laplacian()
        offs = Ls.row_offsets()
        o = orders.bisect_order(offs, Ls.col_indices(), args.n, int(os.environ.get("GS_BENCH_LEAF", "64")))
        win = 256  # degree-sorted windows, as the narrow layout's default order
        deg = np.diff(offs)[o]
        o2 = o.copy()
        for w0 in range(0, len(o), win):
            seg = o[w0:w0 + win]
            o2[w0:w0 + win] = seg[np.argsort(-deg[w0:w0 + win], kind="stable")]
        filt.set_vertex_order(o2, 1)
    n, m = args.n, args.members
    lo, hi = member_shard(m, world, rank)
    dev = torch.device("cuda", local)
    Mloc = torch.from_numpy(np.ascontiguousarray(cfg.members[lo:hi])).to(dev)
    al = torch.full((hi - lo,), 1.0 / m, dtype=torch.float64, device=dev)
    a = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    bary = torch.empty(n, dtype=torch.float64, device=dev)
    Vo = torch.empty((hi - lo, n), dtype=torch.float64, device=dev)
    Wo = torch.empty_like(Vo)
    it = np.zeros(1, np.int32)
    conv = np.zeros(1, np.int32)
    err = np.zeros(1)
    # the engine's own NCCL communicator: allreduces on the engine stream, sweeps stay
    # graph-captured; one rank has nothing to reduce and runs without a comm
    hook = NcclComm(ctx) if world > 1 else None
    comm_arg = hook.comm if world > 1 else None

    def step():
        rc = lib.gs_barycenter_ex(ctx.handle, filt._h, a.data_ptr(), Mloc.data_ptr(), hi - lo,
                                  al.data_ptr(), args.sweeps, TOL_RUN_ALL, _capi.GS_MEM_DEVICE,
                                  comm_arg, 0, bary.data_ptr(), Vo.data_ptr(),
                                  Wo.data_ptr(), it.ctypes.data, conv.ctypes.data, err.ctypes.data)
        ctx.check(rc)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ctx.set_timing(True)
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    step_n, step_ms = ctx.timing(0)
    ctx.set_timing(False)
    launches = ctx.launch_count() - l0
    elapsed = max_over_ranks(e0.elapsed_time(e1))
    value = args.sweeps * args.steps / (elapsed / 1000.0)
    peak, peak_kind = peaks()
    nnz_L = lap.matrix.stored_entries()
    B = hi - lo
    bytes_step = algorithmic_bytes_per_step(n, nnz_L, B)
    avg = step_ms / max(step_n, 1)

    # ---- e2e through the C ABI with host buffers (members, alphas, a in; bary, V, W out) ---------
    Mh = torch.from_numpy(np.ascontiguousarray(cfg.members[lo:hi])).pin_memory()
    alh = torch.full((hi - lo,), 1.0 / m, dtype=torch.float64).pin_memory()
    ah = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
    bh = torch.empty(n, dtype=torch.float64).pin_memory()
    Vh = torch.empty((hi - lo, n), dtype=torch.float64).pin_memory()
    Wh = torch.empty_like(Vh).pin_memory()

    def step_host():
        rc = lib.gs_barycenter_ex(ctx.handle, filt._h, ah.data_ptr(), Mh.data_ptr(), hi - lo,
                                  alh.data_ptr(), args.sweeps, TOL_RUN_ALL, _capi.GS_MEM_HOST,
                                  comm_arg, 0, bh.data_ptr(), Vh.data_ptr(),
                                  Wh.data_ptr(), it.ctypes.data, conv.ctypes.data, err.ctypes.data)
        ctx.check(rc)

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    dist.barrier()
    e2e = {"value": args.sweeps * e2e_steps / e2e_s, "unit": "barycenter sweeps/s",
           "h2d_bytes_per_step": (hi - lo) * n * 8 + (hi - lo) * 8 + n * 8,
           "d2h_bytes_per_step": n * 8 + 2 * (hi - lo) * n * 8 + 4 + 4 + 8, "steps": e2e_steps}
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as po
        L = lap.matrix
        Lo = po.CSR(n, L.row_offsets().copy(), L.col_indices().copy(), L.values().copy())
        fo = po.Filter(Lo, 0, lap.lambda_max_bound, cfg.t, cfg.degree)
        t1 = time.perf_counter()
        ref = po.barycenter(fo, np.full(n, 1.0 / n), cfg.members, None, 1, TOL_RUN_ALL,
                            L=po.lib(native=True))
        dt = time.perf_counter() - t1
        cpu = {"value": 1.0 / dt, "unit": "barycenter sweeps/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"1 barycenter sweep of the 8-member family on the GPU-built n={n} graph ({dt:.1f} s)"}
        # results parity at full size: the engine's sweep on the same operator and family
        rc = lib.gs_barycenter_ex(ctx.handle, filt._h, ah.data_ptr(), Mh.data_ptr(), hi - lo,
                                  alh.data_ptr(), 1, TOL_RUN_ALL, _capi.GS_MEM_HOST, comm_arg, 0,
                                  bh.data_ptr(), Vh.data_ptr(), Wh.data_ptr(), it.ctypes.data,
                                  conv.ctypes.data, err.ctypes.data)
        ctx.check(rc)
        bary = bh.numpy().copy()
        parity = {"sweeps": 1, "against": "oracle restatement, same GPU-built Laplacian, same family",
                  "max_rel_barycenter": _max_rel(bary, ref["barycenter"]),
                  "max_rel_V": _max_rel(Vh.numpy(), ref["V"]), "max_rel_W": _max_rel(Wh.numpy(), ref["W"])}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "barycenter sweeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config2: {n} points in R^30 (20-component mixture), k=15 "
                                   f"Gaussian-median graph, t=0.5, K=30, m={m} members sharded "
                                   f"over {world} rank(s), {args.sweeps} sweeps",
                       "nnz_L": int(nnz_L), "lambda_max_bound": lap.lambda_max_bound,
                       "lambda_rounds": lap.power_rounds, "graph_build_s": t_graph,
                       "members_per_rank": B, "allreduce_calls": hook.calls() if hook is not None else 0,
                       "parallelism": f"member sharding x{world}, NCCL allreduce per sweep" if world > 1
                       else "one rank: no collective, sweeps replayed as a CUDA graph"},
            "roofline": {"bound": "hbm", "achieved": bytes_step / (avg / 1000.0) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_step / (avg / 1000.0) / 1e9 / peak,
                         "traffic": None, "peak_kind": peak_kind, "bytes_per_launch": bytes_step,
                         "avg_launch_ms": avg, "launches_timed": step_n},
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks, "cpu_baseline": cpu,
            "parity": parity,
            "iterations": int(it[0]), "marginal_error": float(err[0]),
        }), flush=True)
    dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- config 4 (barycentric distance)
def run_engine_bary_dist(args):
    """Config 4: barycentric distance (barycenter.cpp:101-107) on n = 4e6 points in R^30 (40
    clusters), k = 15, t = 0.5, K = 30: the barycenters of two 16-member groups (200 sweeps each,
    members sharded over the ranks with one allreduce pair per sweep, as config 2), then the
    geodesic Sinkhorn distance between them (200 sweeps, every rank). One step = one evaluation;
    value = evaluations/s (strong scaling)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi, workloads
    from paper_2211_00805_b200.distributed import NcclComm, member_shard

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    with _StdoutToStderr():
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%d" % _free_port(),
                                    rank=0, world_size=1, device_id=torch.device("cuda", local))
        dist.barrier()
    ctx = gs.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    n, m = args.n, args.members
    t0 = time.perf_counter()
    cfg = workloads.config4(n, m)
    t_data = time.perf_counter() - t0
    t0 = time.perf_counter()
    A, sigma = gs.knn_gaussian_graph(cfg.mix.points, cfg.k, ctx=ctx)
    t_graph = time.perf_counter() - t0
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, cfg.t, cfg.degree)
    lo, hi = member_shard(m, world, rank)
    B = hi - lo
    dev = torch.device("cuda", local)
    Ga = torch.from_numpy(np.ascontiguousarray(cfg.group_a[lo:hi])).to(dev)
    Gb = torch.from_numpy(np.ascontiguousarray(cfg.group_b[lo:hi])).to(dev)
    al = torch.full((B,), 1.0 / m, dtype=torch.float64, device=dev)
    a = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    ba = torch.empty(n, dtype=torch.float64, device=dev)
    bb = torch.empty_like(ba)
    Vo = torch.empty((B, n), dtype=torch.float64, device=dev)
    Wo = torch.empty_like(Vo)
    vd = torch.empty(n, dtype=torch.float64, device=dev)
    wd = torch.empty_like(vd)
    dsc = torch.empty(3, dtype=torch.float64, device=dev)
    dsi = torch.empty(2, dtype=torch.int32, device=dev)
    it, conv, err = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1)
    hook = NcclComm(ctx) if world > 1 else None  # the engine's own NCCL communicator
    comm_arg = hook.comm if world > 1 else None
    fp, fs = C.c_int(), C.c_int()
    flags = _capi.GS_FLAG_NO_STAGNATION_ABORT

    def bary(M, out):
        rc = lib.gs_barycenter_ex(ctx.handle, filt._h, a.data_ptr(), M.data_ptr(), B, al.data_ptr(),
                                  args.sweeps, TOL_RUN_ALL, _capi.GS_MEM_DEVICE, comm_arg, 0,
                                  out.data_ptr(), Vo.data_ptr(), Wo.data_ptr(), it.ctypes.data,
                                  conv.ctypes.data, err.ctypes.data)
        ctx.check(rc)

    def step():
        bary(Ga, ba)
        bary(Gb, bb)
        p0, pi = dsc.data_ptr(), dsi.data_ptr()
        ctx.check(lib.gs_sinkhorn(ctx.handle, filt._h, a.data_ptr(), ba.data_ptr(), bb.data_ptr(), 1,
                                  args.sweeps, TOL_RUN_ALL, flags | _capi.GS_FLAG_SINGLE,
                                  _capi.GS_MEM_DEVICE, vd.data_ptr(), wd.data_ptr(), p0, p0 + 8,
                                  pi, pi + 4, p0 + 16, C.byref(fp), C.byref(fs)))

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ctx.set_timing(True, period=args.timing_period)
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    step_n, step_ms = ctx.timing(0)
    ctx.set_timing(False)
    launches = ctx.launch_count() - l0
    elapsed = max_over_ranks(e0.elapsed_time(e1))
    value = args.steps / (elapsed / 1000.0)
    distance = float(dsc[0].item())
    # ---- per-launch step time of the barycenter alone (B = members per rank), one extra run with
    # per-kernel launches and an event pair around every step launch
    os.environ["GS_GRAPH"] = "0"
    ctx.set_timing(True)
    bary(Ga, ba)
    torch.cuda.synchronize()
    step_n, step_ms = ctx.timing(0)
    ctx.set_timing(False)
    del os.environ["GS_GRAPH"]
    # ---- reference semantics for the distance (abort on): barycentric_distance raises
    # Disconnected when the two barycenters' mass sits in different graph components
    # (barycenter.cpp:101-107 -> transport.cpp:132-134)
    rc_ab = lib.gs_sinkhorn(ctx.handle, filt._h, a.data_ptr(), ba.data_ptr(), bb.data_ptr(), 1,
                            args.sweeps, 1e-9, _capi.GS_FLAG_SINGLE, _capi.GS_MEM_DEVICE,
                            vd.data_ptr(), wd.data_ptr(), dsc.data_ptr(), dsc.data_ptr() + 8,
                            dsi.data_ptr(), dsi.data_ptr() + 4, dsc.data_ptr() + 16, C.byref(fp),
                            C.byref(fs))
    torch.cuda.synchronize()
    distance_ref = ({"rc": int(rc_ab), "errc": lib.gs_last_error(ctx.handle).decode(),
                     "fail_sweep": fs.value} if rc_ab else {"rc": 0, "cost": float(dsc[0].item())})
    # ---- e2e: the same evaluation through gs.barycentric_distance-equivalent host-buffer calls ----
    Gah = torch.from_numpy(np.ascontiguousarray(cfg.group_a[lo:hi])).pin_memory()
    Gbh = torch.from_numpy(np.ascontiguousarray(cfg.group_b[lo:hi])).pin_memory()
    alh = torch.full((B,), 1.0 / m, dtype=torch.float64).pin_memory()
    ah = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
    bah = torch.empty(n, dtype=torch.float64).pin_memory()
    bbh = torch.empty_like(bah).pin_memory()
    Vh = torch.empty((B, n), dtype=torch.float64).pin_memory()
    Wh = torch.empty_like(Vh).pin_memory()
    vh = torch.empty(n, dtype=torch.float64).pin_memory()
    wh = torch.empty_like(vh).pin_memory()
    cost_h, kl_h, err_h = np.zeros(1), np.zeros(1), np.zeros(1)
    it_h, cv_h = np.zeros(1, np.int32), np.zeros(1, np.int32)

    def step_host():
        for M, out in ((Gah, bah), (Gbh, bbh)):
            rc = lib.gs_barycenter_ex(ctx.handle, filt._h, ah.data_ptr(), M.data_ptr(), B, alh.data_ptr(),
                                      args.sweeps, TOL_RUN_ALL, _capi.GS_MEM_HOST, comm_arg, 0,
                                      out.data_ptr(), Vh.data_ptr(), Wh.data_ptr(), it.ctypes.data,
                                      conv.ctypes.data, err.ctypes.data)
            ctx.check(rc)
        ctx.check(lib.gs_sinkhorn(ctx.handle, filt._h, ah.data_ptr(), bah.data_ptr(), bbh.data_ptr(), 1,
                                  args.sweeps, TOL_RUN_ALL, flags | _capi.GS_FLAG_SINGLE,
                                  _capi.GS_MEM_HOST, vh.data_ptr(), wh.data_ptr(), cost_h.ctypes.data,
                                  kl_h.ctypes.data, it_h.ctypes.data, cv_h.ctypes.data, err_h.ctypes.data,
                                  C.byref(fp), C.byref(fs)))

    torch.cuda.synchronize()
    dist.barrier()
    t1 = time.perf_counter()
    step_host()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t1)
    e2e = {"value": 1.0 / e2e_s, "unit": "barycentric distances/s",
           "h2d_bytes_per_step": 2 * (B * n * 8 + B * 8 + n * 8) + 2 * n * 8 + n * 8,
           "d2h_bytes_per_step": 2 * (n * 8 + 2 * B * n * 8 + 16) + 2 * n * 8 + 32, "steps": 1}
    cpu4 = None
    parity4 = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:  # bounded sample: one barycenter sweep of group A (16 members) of the oracle
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import pyoracle as po
            L = lap.matrix
            Lo = po.CSR(n, L.row_offsets().copy(), L.col_indices().copy(), L.values().copy())
            fo = po.Filter(Lo, 0, lap.lambda_max_bound, cfg.t, cfg.degree)
            t2 = time.perf_counter()
            ref = po.barycenter(fo, np.full(n, 1.0 / n), cfg.group_a, None, 1, TOL_RUN_ALL,
                                L=po.lib(native=True))
            dt = time.perf_counter() - t2
            # one evaluation = 2 x sweeps barycenter sweeps of m members + sweeps one-pair sweeps
            est = 2 * args.sweeps * dt + args.sweeps * dt / m
            cpu4 = {"value": 1.0 / est, "unit": "barycentric distances/s", "cores": os.cpu_count(),
                    "kind": "port",
                    "sample": f"1 barycenter sweep of group A ({m} members) on the GPU-built n={n} graph "
                              f"({dt:.1f} s), extrapolated to one evaluation (2 x {args.sweeps} barycenter "
                              f"sweeps + {args.sweeps} one-pair sweeps at 1/{m} of a barycenter sweep)"}
            # results parity at full size: the engine's sweep on the same operator and family
            rc = lib.gs_barycenter_ex(ctx.handle, filt._h, ah.data_ptr(), Gah.data_ptr(), B, alh.data_ptr(),
                                      1, TOL_RUN_ALL, _capi.GS_MEM_HOST, comm_arg, 0, bah.data_ptr(),
                                      Vh.data_ptr(), Wh.data_ptr(), it.ctypes.data, conv.ctypes.data,
                                      err.ctypes.data)
            ctx.check(rc)
            parity4 = {"sweeps": 1, "against": "oracle restatement, same GPU-built Laplacian, group A",
                       "max_rel_barycenter": _max_rel(bah.numpy(), ref["barycenter"]),
                       "max_rel_V": _max_rel(Vh.numpy(), ref["V"]),
                       "max_rel_W": _max_rel(Wh.numpy(), ref["W"]), "tolerance": 1e-9}
        except Exception as e:  # host memory / time limits: report why
            cpu4 = {"value": None, "unit": "barycentric distances/s", "cores": os.cpu_count(),
                    "kind": "port", "sample": f"not run: {type(e).__name__}: {e}"}
    peak, peak_kind = peaks()
    nnz_L = lap.matrix.stored_entries()
    bytes_step = algorithmic_bytes_per_step(n, nnz_L, B)
    avg = step_ms / max(step_n, 1)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "barycentric distances/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"config4: {n} points in R^30 (40-component mixture), k=15 "
                                   f"Gaussian-median graph, t=0.5, K=30; two {m}-member barycenters "
                                   f"x {args.sweeps} sweeps (members sharded over {world} rank(s)) + "
                                   f"their geodesic Sinkhorn distance ({args.sweeps} sweeps)",
                       "nnz_L": int(nnz_L), "graph_build_s": t_graph, "data_s": t_data,
                       "members_per_rank": B,
                       "distance_abort_off": distance,
                       "distance_reference_semantics": distance_ref,
                       "sweeps_per_step": {"barycenter": 2 * args.sweeps, "distance": args.sweeps},
                       "parallelism": (f"member sharding x{world}, NCCL allreduce per sweep"
                                       if world > 1 else "one rank: no collective, CUDA-graph sweeps")},
            "roofline": {"bound": "hbm", "achieved": bytes_step / (avg / 1000.0) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_step / (avg / 1000.0) / 1e9 / peak,
                         "traffic": None, "peak_kind": peak_kind, "bytes_per_launch": bytes_step,
                         "avg_launch_ms": avg, "launches_timed": step_n,
                         "kernel": f"barycenter step (B = {B}), event pair around every launch of one "
                                   "barycenter run with per-kernel launches"},
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks, "cpu_baseline": cpu4,
            **({"parity": parity4} if parity4 else {}),
        }), flush=True)
    dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- config 3 (row partitions)
def run_engine_rows(args):
    """Config 3: n = 2e7 swiss roll, k = 10 Gaussian-median graph (grid kNN), combinatorial L,
    t = 1, K = 30, fp32, one pair (config 0's bumps at 2 pi / 4 pi), 100 sweeps. Rows are
    partitioned over the ranks (gs_part_*: contiguous nnz-balanced ranges of the CM order, one halo
    exchange per Chebyshev step through NCCL all_to_all_single, allreduced column reductions);
    strong scaling, value = sweeps/s. One rank runs the unpartitioned path (the same rows, sweeps
    replayed as CUDA graphs)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import _capi, workloads
    from paper_2211_00805_b200.distributed import NcclComm

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        with _StdoutToStderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
    ctx = gs.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    n = args.n
    t0 = time.perf_counter()
    roll = workloads.swiss_roll(n, 1)
    A, sigma = gs.knn_gaussian_graph(roll.points, 10, ctx=ctx)
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    filt = gs.HeatFilter(lap, 1.0, 30)
    if os.environ.get("GS_BENCH_ORDER") == "morton":  # experiment: host-computed locality order
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import orders
        o = orders.morton3(roll.points)
        filt.set_vertex_order(o, 0)
        filt.set_vertex_order(o, 1)
    setup_s = time.perf_counter() - t0
    # config 3's pair as specified (bumps at 2 pi and 4 pi) lies beyond the K = 30 hop reach: the
    # reference raises Disconnected and the 32-bit mode the same errc (fp64 with the abort off
    # returns -inf); the timed pair is its well-posed companion, nu at 2 pi + 0.5
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5)
    a = np.full(n, 1.0 / n)
    flags = _capi.GS_FLAG_NO_STAGNATION_ABORT | _capi.GS_FLAG_FP32
    dev = torch.device("cuda", local)
    hook = None
    comm = None
    part = None
    if world > 1:
        part = gs.RowPartition(filt, world, rank, ctx=ctx)
        vid = part.vertices.astype(np.int64)
        hook = NcclComm(ctx)  # the engine's own NCCL communicator (neighbour-only halo exchange)
        comm = hook.comm
        nnz_loc = part.nnz_local
    else:
        vid = np.arange(n)
        nnz_loc = lap.matrix.stored_entries()
    nl = vid.size
    Md = torch.from_numpy(mu[vid].copy()).to(dev)
    Nd = torch.from_numpy(nu[vid].copy()).to(dev)
    ad = torch.from_numpy(a[vid].copy()).to(dev)
    vd = torch.empty(nl, dtype=torch.float64, device=dev)
    wd = torch.empty_like(vd)
    cost, kl, err = np.empty(1), np.empty(1), np.empty(1)
    it, conv = np.empty(1, np.int32), np.empty(1, np.int32)
    fp, fs = C.c_int(), C.c_int()

    dsc = torch.empty(3, dtype=torch.float64, device=dev)  # cost, kl, err (device-mode outputs)
    dsi = torch.empty(2, dtype=torch.int32, device=dev)    # iterations, converged

    def run(mem, M, N, av, v, w):
        if mem == _capi.GS_MEM_DEVICE:
            p0, pi = dsc.data_ptr(), dsi.data_ptr()
            small = (p0, p0 + 8, pi, pi + 4, p0 + 16)
        else:
            small = (cost.ctypes.data, kl.ctypes.data, it.ctypes.data, conv.ctypes.data,
                     err.ctypes.data)
        outs = (v, w, *small, C.byref(fp), C.byref(fs))
        if part is None:
            rc = lib.gs_sinkhorn(ctx.handle, filt._h, av, M, N, 1, args.sweeps, TOL_RUN_ALL, flags,
                                 mem, *outs)
        else:
            rc = lib.gs_part_sinkhorn(ctx.handle, part._h, comm, av, M, N, 1, args.sweeps,
                                      TOL_RUN_ALL, flags, mem, *outs)
        ctx.check(rc)

    def step():
        run(_capi.GS_MEM_DEVICE, Md.data_ptr(), Nd.data_ptr(), ad.data_ptr(), vd.data_ptr(),
            wd.data_ptr())

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ctx.set_timing(True, period=args.timing_period)
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    step_n, step_ms = ctx.timing(0)
    ctx.set_timing(False)
    launches = ctx.launch_count() - l0
    elapsed = max_over_ranks(e0.elapsed_time(e1))
    value = args.sweeps * args.steps / (elapsed / 1000.0)
    peak, peak_kind = peaks()
    bytes_step = algorithmic_bytes_per_step(nl, nnz_loc, 1, sv=4)
    avg = step_ms / max(step_n, 1)
    # ---- e2e through the C ABI with host buffers ------------------------------------------------
    Mh = torch.from_numpy(mu[vid].copy()).pin_memory()
    Nh = torch.from_numpy(nu[vid].copy()).pin_memory()
    ah = torch.from_numpy(a[vid].copy()).pin_memory()
    vh = torch.empty(nl, dtype=torch.float64).pin_memory()
    wh = torch.empty_like(vh).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    barrier()
    t1 = time.perf_counter()
    for _ in range(e2e_steps):
        run(_capi.GS_MEM_HOST, Mh.data_ptr(), Nh.data_ptr(), ah.data_ptr(), vh.data_ptr(), wh.data_ptr())
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t1)
    barrier()
    e2e = {"value": args.sweeps * e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 3 * nl * 8, "d2h_bytes_per_step": 2 * nl * 8 + 8 + 8 + 4 + 4 + 8,
           "steps": e2e_steps}
    cpu = None
    parity3 = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:  # bounded sample: one K = 30 fp64 apply (half a sweep) of the oracle on this graph
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import pyoracle as po
            L = lap.matrix
            Lo = po.CSR(n, L.row_offsets().copy(), L.col_indices().copy(), L.values().copy())
            fo = po.Filter(Lo, 0, lap.lambda_max_bound, 1.0, 30)
            x = mu.copy()
            t2 = time.perf_counter()
            yo = fo.apply(x)
            dt = time.perf_counter() - t2
            cpu = {"value": 0.5 / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"one K=30 fp64 apply (half a sweep) of the oracle on the GPU-built "
                             f"n={n} graph, OpenMP ({dt:.1f} s)"}
            # full-size parity of the apply (outside every timed region): the engine's fp64 apply
            # against the oracle's bit for bit, its 32-bit mode within the north star's 1e-4
            y64 = filt.apply(x)
            y32 = filt.apply(x, fp32=True)
            scale = float(np.max(np.abs(yo)))
            parity3 = {"against": "oracle restatement (oracle/), one K=30 apply of mu on the same "
                                  f"GPU-built n={n} operator",
                       "fp64_apply_bit_identical": bool(np.array_equal(y64, yo)),
                       "fp32_mode_apply_max_abs_over_max": float(np.max(np.abs(y32 - yo)) / scale),
                       "tolerance": 1e-4}
        except Exception as e:  # host memory / time limits: report why
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                   "sample": f"not run: {type(e).__name__}"}
    # DRAM bytes of the dominant kernel per launch from the committed ncu capture (one rank)
    traffic3, ncu3 = None, None
    prof3 = os.path.join(ROOT, "profiles", "lane_step_traffic.json")
    if world == 1 and os.path.exists(prof3):
        try:
            with open(prof3) as fh:
                ncu3 = json.load(fh)
            traffic3 = ncu3.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic3, ncu3 = None, None
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"config3: swiss roll n={n}, k=10 Gaussian-median graph (grid "
                                   f"kNN), combinatorial L, t=1, K=30, fp32 (32-bit words), 1 pair "
                                   f"(bumps at 2pi and 2pi+0.5: the well-posed companion), "
                                   f"{args.sweeps} sweeps, rows partitioned over {world} rank(s)",
                       "nnz_L": int(lap.matrix.stored_entries()), "rows_local": int(nl),
                       "nnz_local": int(nnz_loc),
                       "halo_rows": int(part.n_halo) if part is not None else 0,
                       "setup_s": setup_s, "sigma": sigma, "lambda_max_bound": lap.lambda_max_bound,
                       "stagnation_abort": "disabled (bench-only, DESIGN.md)",
                       "l2": "working set > 2 GB >> 126 MB L2; no flush needed between steps",
                       "parallelism": (f"row partitions x{world}, engine NCCL halo (neighbour send/recv) per step, graph-captured sweeps"
                                       if world > 1 else "one rank: unpartitioned rows, CUDA-graph sweeps")},
            "roofline": {"bound": "hbm", "achieved": bytes_step / (avg / 1000.0) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_step / (avg / 1000.0) / 1e9 / peak,
                         "traffic": traffic3, "peak_kind": peak_kind, "bytes_per_launch": bytes_step,
                         "avg_launch_ms": avg, "launches_timed": step_n,
                         "kernel": ("k_cheb_lane<float, 1, *> (one row per lane, per-warp CSR slices staged in "
                                    "shared memory by bulk copies)" if world == 1 else
                                    "k_cheb_lane<float, 1, *> on the part's interior / boundary row ranges"),
                         **({"ncu": ncu3} if ncu3 else {})},
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks, "cpu_baseline": cpu,
            "iterations": int(it[0]), "marginal_error": float(err[0]),
            **({"parity": parity3} if parity3 else {}),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    p_ = s_.getsockname()[1]
    s_.close()
    return p_


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--pairs", type=int, default=64)
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sweeps", type=int, default=1)
    ap.add_argument("--ref-sweeps", type=int, default=2)
    ap.add_argument("--parity-pairs", type=int, default=4)
    ap.add_argument("--no-legs", action="store_true", help="skip the partitioned data-plane legs")
    ap.add_argument("--legs-bary-n", type=int, default=200_000)
    ap.add_argument("--legs-rows-n", type=int, default=2_000_000)
    ap.add_argument("--legs-sweeps", type=int, default=40)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--members", type=int, default=8)
    ap.add_argument("--timing-period", type=int, default=1,
                    help="event-time every Nth engine launch inside the timed region (sweeps "
                         "replayed as CUDA graphs are not split into launches: the timed launches "
                         "are each call's initial apply)")
    args = ap.parse_args()
    # N GPUs of one node: one process per GPU. Without a launcher around us, re-exec under
    # torch.distributed.run (127.0.0.1 rendezvous); under one, the launcher's world must be N.
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world_env}"}))
        return 2
    if args.config == 0 and "--steps" not in sys.argv:
        args.steps = 100  # ~0.6 s timed region, long enough for the clock sampler
    if args.config == 0:  # BASELINE.json configs[0]: n=2000, one pair, 100 sweeps
        if args.n == 200_000:
            args.n = 2000
        if args.pairs == 64:
            args.pairs = 1
        if args.sweeps == 200:
            args.sweeps = 100
    if args.config == 2:
        if args.n == 200_000:
            args.n = 1_000_000
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 2 reference arm needs an "
                              "O(n^2 d) CPU kNN at n=1e6; use the default config"}))
            return 0
        return run_engine_bary(args)
    if args.config == 4:
        if args.n == 200_000:
            args.n = 4_000_000
        if args.members == 8:
            args.members = 16
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 4 reference arm needs an "
                              "O(n^2 d) CPU kNN at n=4e6; use the default config"}))
            return 0
        return run_engine_bary_dist(args)
    if args.config == 3:
        if args.n == 200_000:
            args.n = 20_000_000
        if args.sweeps == 200:
            args.sweeps = 100
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 3 reference arm needs an "
                              "O(n^2) CPU kNN at n=2e7; use the default config"}))
            return 0
        return run_engine_rows(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
