"""mccann_interpolate (transport.cpp:326-376): host sampling over plan rows, checked against a
plain-loop restatement with the same geosink::Rng draws, plus the reference's validation and the
s = 0 / s = 1 endpoints. (Plan rows come from the device in use -- tests/test_gpu_parity.py.)"""
import numpy as np
import pytest

import paper_2211_00805_b200 as gs
from paper_2211_00805_b200.rng import Rng


def _loop_restatement(src, tgt, rows, s, num, seed):
    m_src, m_tgt = len(rows), len(rows[0])
    mass = []
    for r in rows:
        acc = 0.0
        for x in r:
            acc += max(x, 0.0)
        mass.append(acc)
    cum, acc = [], 0.0
    for x in mass:
        acc += x
        cum.append(acc)
    total = cum[-1]
    rng = Rng(seed)
    counts = [0] * m_src
    for _ in range(num):
        u = rng.uniform() * total
        i = next((k for k, c in enumerate(cum) if not c < u), m_src)
        counts[min(i, m_src - 1)] += 1
    out = []
    for i in range(m_src):
        if counts[i] == 0:
            continue
        rc, acc = [], 0.0
        for x in rows[i]:
            acc += max(x, 0.0)
            rc.append(acc)
        for _ in range(counts[i]):
            u = rng.uniform() * rc[-1]
            j = next((k for k, c in enumerate(rc) if not c < u), m_tgt)
            out.append([(1.0 - s) * a + s * b for a, b in zip(src[i], tgt[min(j, m_tgt - 1)])])
    return np.array(out)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_mccann_matches_loop_restatement(seed):
    g = np.random.default_rng(seed)
    src, tgt = g.standard_normal((9, 3)), g.standard_normal((7, 3))
    plan = g.random((9, 7)) - 0.1  # some negative entries: clamped at zero like the reference
    plan = np.maximum(plan, -0.05)
    plan /= np.maximum(plan, 0).sum()
    rows = [list(r) for r in plan]
    got = gs.mccann_interpolate(src, tgt, lambda i: plan[i], 0.3, 25, seed)
    ref = _loop_restatement(src.tolist(), tgt.tolist(), rows, 0.3, 25, seed)
    assert np.array_equal(got, ref)


def test_mccann_endpoints_and_validation():
    g = np.random.default_rng(0)
    src, tgt = g.standard_normal((4, 2)), g.standard_normal((5, 2))
    plan = np.full((4, 5), 1.0 / 20)
    at0 = gs.mccann_interpolate(src, tgt, lambda i: plan[i], 0.0, 30, 7)
    assert all(any(np.array_equal(p, x) for x in src) for p in at0)
    at1 = gs.mccann_interpolate(src, tgt, lambda i: plan[i], 1.0, 30, 7)
    assert all(any(np.array_equal(p, y) for y in tgt) for p in at1)
    cases = [
        (lambda: gs.mccann_interpolate(src, g.standard_normal((5, 3)), lambda i: plan[i], 0.5, 3, 1), gs.errc.size_mismatch),
        (lambda: gs.mccann_interpolate(src, tgt, lambda i: plan[i], 1.5, 3, 1), gs.errc.invalid_argument),
        (lambda: gs.mccann_interpolate(src, tgt, lambda i: plan[i], 0.5, 0, 1), gs.errc.invalid_argument),
        (lambda: gs.mccann_interpolate(src, tgt, lambda i: plan[i] * 0.5, 0.5, 3, 1), gs.errc.degenerate_plan),
        (lambda: gs.mccann_interpolate(src, tgt, lambda i: plan[i][:3], 0.5, 3, 1), gs.errc.length_mismatch),
        (lambda: gs.mccann_interpolate(np.zeros((0, 2)), tgt, lambda i: plan[i], 0.5, 3, 1), gs.errc.dimension_mismatch),
    ]
    for fn, code in cases:
        with pytest.raises(gs.Error) as e:
            fn()
        assert e.value.code == code
