"""CPU-only checks of the product library and host logic (no kernel launches here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "geosink_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(gs_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2211_00805_b200 import _capi
    lib = _capi.load()
    names = _declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers exactly the declared surface
    assert set(_capi.SIGNATURES) == set(names)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2211_00805_b200", "lib", "libgeosink_b200.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2211_00805_b200 import Context, _capi
    with pytest.raises(_capi.EngineUnavailable):
        Context(0)


def test_host_rng_and_workloads_deterministic():
    from paper_2211_00805_b200 import workloads
    a = workloads.swiss_roll(1000, 1)
    b = workloads.swiss_roll(1000, 1)
    assert np.array_equal(a.points, b.points)
    assert a.s.min() >= 1.5 * np.pi and a.s.max() < 4.5 * np.pi
    assert a.h.min() >= 0 and a.h.max() < 20
    mus, nus = workloads.bump_mixture_pairs(a, 4, 2)
    assert mus.shape == (4, 1000) and np.allclose(mus.sum(1), 1, atol=1e-14)
    mix = workloads.gaussian_mixture(2000, 30, 20, 3)
    mem = workloads.cluster_subset_members(mix, 8, 4, 0.6, 4)
    assert mem.shape == (8, 2000) and np.allclose(mem.sum(1), 1, atol=1e-14)
    for m in mem:  # each member supported on at most 4 clusters
        assert len(np.unique(mix.labels[m > 0])) <= 4


def test_python_api_host_validation():
    from paper_2211_00805_b200 import Distribution, DistributionFamily, Error, errc
    with pytest.raises(Error) as e:
        Distribution(np.full(3, 0.5))
    assert e.value.code == errc.invalid_argument
    with pytest.raises(Error):
        Distribution(np.array([1.5, -0.5]))
    u = Distribution.uniform(4)
    assert abs(u.weights.sum() - 1) <= 1e-15
    ind = Distribution.indicator(5, [1, 3])
    assert ind.weights[1] == 0.5 and ind.weights[0] == 0.0
    fam = DistributionFamily([Distribution.uniform(4)], alphas=np.array([0.5, 0.5]))
    with pytest.raises(Error) as e:
        fam.validate(4)
    assert e.value.code == errc.length_mismatch
    with pytest.raises(Error):
        DistributionFamily([]).validate(4)


def test_reference_arm_json_contract():
    """bench.py --impl reference (the CPU oracle arm) prints one JSON line with the contract's
    keys on a small instance of the config-1 workload."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--n", "3000",
                        "--pairs", "4", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["product_library_loaded"] is False  # inputs drawn with the oracle's Rng
