"""geosink::Rng (proj/include/geosink/rng.hpp:13-68) over the engine's host-side gs_rng_* ABI."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi


class Rng:
    def __init__(self, seed: int):
        self._lib = _capi.load()
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self._h = self._lib.gs_rng_create(self.seed)

    def fork(self, stream: int) -> "Rng":
        return Rng(self.seed_mix(self.seed, stream))

    def bits(self) -> int:
        return int(self._lib.gs_rng_bits(self._h))

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        if lo is None:
            return float(self._lib.gs_rng_uniform(self._h))
        return float(self._lib.gs_rng_uniform_range(self._h, lo, hi))

    def normal(self) -> float:
        return float(self._lib.gs_rng_normal(self._h))

    def below(self, n: int) -> int:
        return int(self._lib.gs_rng_below(self._h, n))

    @staticmethod
    def seed_mix(a: int, b: int) -> int:
        return int(_capi.load().gs_rng_seed_mix(a & 0xFFFFFFFFFFFFFFFF, b & 0xFFFFFFFFFFFFFFFF))

    def pattern(self, count: int, spec) -> np.ndarray:
        """Draw `count` values cycling through spec = [(kind, lo, hi), ...] (see gs_rng_fill_pattern):
        kind 'u' = uniform(lo, hi), 'n' = hi * normal() (+ lo), 'b' = below(hi)."""
        kinds = np.array([{"u": 0, "n": 1, "b": 2}[k] for k, _, _ in spec], np.int32)
        lo = np.array([float(l) for _, l, _ in spec], np.float64)
        hi = np.array([float(h) for _, _, h in spec], np.float64)
        out = np.empty(count, np.float64)
        self._lib.gs_rng_fill_pattern(self._h, out.ctypes.data, count, kinds.ctypes.data,
                                      lo.ctypes.data, hi.ctypes.data, len(spec))
        return out

    def normals(self, count: int) -> np.ndarray:
        return self.pattern(count, [("n", 0.0, 1.0)])

    def __del__(self):
        try:
            self._lib.gs_rng_destroy(self._h)
        except Exception:
            pass
