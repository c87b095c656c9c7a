"""Counter-based random numbers for the synthetic tables (master seed 180608384,
per-column seeds derived by SplitMix64).

`splitmix64` / `derive_seed` run on Python ints (exact, host only). `h32` is a stateless
32-bit hash of (seed, row index) written with int64 torch ops whose intermediates never exceed
2^49, so it is exact and identical on CPU and CUDA (no reliance on signed-overflow wrapping).
"""

from __future__ import annotations

import torch

MASTER_SEED = 180608384
_M64 = (1 << 64) - 1
_M32 = 0xFFFFFFFF


def splitmix64(x: int) -> int:
    """One SplitMix64 output for state x (Steele, Lea & Flood 2014), Python-int exact."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def derive_seed(*parts) -> int:
    """Derive a 32-bit seed from the master seed and a path of names/ints."""
    s = splitmix64(MASTER_SEED)
    for p in parts:
        if isinstance(p, str):
            for ch in p.encode():
                s = splitmix64(s ^ ch)
        else:
            s = splitmix64(s ^ (int(p) & _M64))
    return s & _M32


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 tensors holding values in [0, 2^32); exact (< 2^49)."""
    lo = c & 0xFFFF
    hi = (c >> 16) & 0xFFFF
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def _lowbias32(x: torch.Tensor) -> torch.Tensor:
    # C. Wellons' "lowbias32" integer hash; x holds values in [0, 2^32).
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def h32(seed: int, idx: torch.Tensor) -> torch.Tensor:
    """Stateless hash of row indices (int64 tensor, values < 2^32) → int64 values in [0, 2^32)."""
    s1 = seed & _M32
    s2 = splitmix64(seed) & _M32
    x = (idx & _M32) ^ s1
    x = _lowbias32(x)
    x = _lowbias32(x ^ s2)
    return x


def uniform_int(seed: int, idx: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """Integers in [lo, hi] (inclusive) by multiply-shift of h32; requires hi - lo < 2^31."""
    rng = hi - lo + 1
    assert 0 < rng < (1 << 31)
    return lo + ((h32(seed, idx) * rng) >> 32)
