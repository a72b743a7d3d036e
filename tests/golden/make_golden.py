"""Generates the committed golden fixtures (run in the dev container, where /root/reference and
scipy exist; the GPU box only reads the .npz files):

  rng_reference.npz  outputs of the reference's own rng.hpp (compiled into oracle/_ref by
                     oracle/Makefile `ref`) for several seeds: bits, uniforms, normals, below
  bessel_ive.npz     2 (-1)^k e^{-t} I_k(t) from scipy.special.ive (independent of the oracle)
                     at the t values of tests/test_heat.cpp:87-100 and the BASELINE configs
  heat_dense.npz     exact e^{-tL} (numpy eigh) for acceptance-criterion-1 graphs
                     (tests/acceptance/acceptance.cpp:73-97), to pin the filter restatement

Usage: python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rng_fixture():
    import pyoracle as po
    R = po.ref_rng()
    assert R is not None, "build oracle/_ref first: make -C oracle ref"
    out = {}
    for seed in (0, 1, 42, 0x5EED1A4B, 2**63 + 5):
        b = np.empty(700, np.uint64)
        R.ref_rng_bits(seed, 700, b)
        u = np.empty(700)
        R.ref_rng_uniform(seed, 700, u)
        z = np.empty(701)
        R.ref_rng_normal(seed, 701, z)
        w = np.empty(300, np.uint64)
        R.ref_rng_below(seed, 97, 300, w)
        out[f"bits_{seed}"] = b
        out[f"uniform_{seed}"] = u
        out[f"normal_{seed}"] = z
        out[f"below97_{seed}"] = w
    out["seed_mix"] = np.array([R.ref_rng_seed_mix(a, b) for a in (0, 1, 7, 2**40) for b in (0, 3, 11)],
                               np.uint64)
    np.savez_compressed(os.path.join(HERE, "rng_reference.npz"), **out)


def bessel_fixture():
    from scipy.special import ive
    out = {}
    for t in (0.3, 0.5, 1.0, 2.0, 5.0, 7.0, 7.95, 13.06, 15.33, 20.0, 50.3):
        deg = 4 * int(np.ceil(t)) + 30
        k = np.arange(deg + 1)
        sign = np.where(k % 2 == 0, 1.0, -1.0)
        out[f"t_{t}"] = 2.0 * sign * ive(k, t)
    np.savez_compressed(os.path.join(HERE, "bessel_ive.npz"), **out)


def heat_fixture():
    import pyoracle as po
    from helpers import acceptance_graph
    out = {}
    for n in (20, 100):
        r, c, v = acceptance_graph(n, 1000 + n)
        A = po.from_triplets(n, r, c, v)
        for kind in (0, 1):
            L, lam, _ = po.laplacian(A, kind)
            w, U = np.linalg.eigh(L.to_dense())
            for t in (0.1, 1.0, 5.0):
                out[f"H_{n}_{kind}_{t}"] = (U * np.exp(-t * w)) @ U.T
    np.savez_compressed(os.path.join(HERE, "heat_dense.npz"), **out)


if __name__ == "__main__":
    rng_fixture()
    bessel_fixture()
    heat_fixture()
    print("golden fixtures written to", HERE)
