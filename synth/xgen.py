"""Counter-based feature generator (SURVEY.md §8(d) "Concrete synthetic inputs").

x[r, c] = 2^-19 * (u0 + u1 + u2 + u3 - 2^21), u_j uniform 20-bit integers drawn
from SplitMix64 at counter 4*(r*F + c) + j under a per-seed key.  The integer
fits in 22 bits, so x is exact in fp32 (no rounding anywhere) and lies on a
2^-19 lattice in [-4, 4): Irwin-Hall, bell-shaped, std ~= 1.15.  Because the
formula is integer-only, numpy (host) and torch (any device) produce the same
bits for any row range, which is what lets the oracle regenerate exactly the
rows it checks.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + np.uint64(_GOLDEN))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def _seed_key(seed: int) -> int:
    return int(splitmix64_np(np.array([seed & _MASK64], dtype=np.uint64))[0])


def gen_x(seed: int, row0: int, n_rows: int, n_features: int) -> np.ndarray:
    """Rows [row0, row0+n_rows) of the seed's matrix, fp32 row-major (host)."""
    out = np.empty((n_rows, n_features), dtype=np.float32)
    key = np.uint64(_seed_key(seed))
    step = max(1, (1 << 22) // max(1, n_features))
    for a in range(0, n_rows, step):
        b = min(n_rows, a + step)
        idx = (np.arange(row0 + a, row0 + b, dtype=np.uint64)[:, None] * np.uint64(n_features)
               + np.arange(n_features, dtype=np.uint64)[None, :])
        with np.errstate(over="ignore"):
            base = key + idx * np.uint64(4)
            s = np.zeros(idx.shape, dtype=np.int64)
            for j in range(4):
                s += (splitmix64_np(base + np.uint64(j)) >> np.uint64(44)).astype(np.int64)
        out[a:b] = ((s - (1 << 21)).astype(np.float32)) * np.float32(2.0 ** -19)
    return out


def _i64(v: int) -> int:
    v &= _MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _splitmix64_torch(x):
    import torch
    def lsr(z, s):
        return (z >> s) & ((1 << (64 - s)) - 1)
    z = x + _i64(_GOLDEN)
    z = (z ^ lsr(z, 30)) * _i64(_M1)
    z = (z ^ lsr(z, 27)) * _i64(_M2)
    return z ^ lsr(z, 31)


def gen_x_torch(seed: int, row0: int, n_rows: int, n_features: int, device="cpu", out=None):
    """Same matrix as :func:`gen_x`, generated with torch int64 ops on ``device``."""
    import torch
    if out is None:
        out = torch.empty((n_rows, n_features), dtype=torch.float32, device=device)
    key = _i64(_seed_key(seed))
    cols = torch.arange(n_features, dtype=torch.int64, device=out.device)
    step = max(1, (1 << 24) // max(1, n_features))
    for a in range(0, n_rows, step):
        b = min(n_rows, a + step)
        rows = torch.arange(row0 + a, row0 + b, dtype=torch.int64, device=out.device)
        idx = rows[:, None] * n_features + cols[None, :]
        base = idx * 4 + key
        s = torch.zeros_like(idx)
        for j in range(4):
            s += (_splitmix64_torch(base + j) >> 44) & ((1 << 20) - 1)
        out[a:b] = (s - (1 << 21)).to(torch.float32) * (2.0 ** -19)
    return out


_SPECIALS = np.array([np.nan, np.inf, -np.inf, 0.0, -0.0,
                      np.float32(1.4e-45), np.float32(-1.4e-45),
                      np.float32(1.17549435e-38)], dtype=np.float32)


def inject_specials(x: np.ndarray, seed: int, rate: float = 1e-3) -> np.ndarray:
    """Correctness variant only: overwrite ~rate of the entries with NaN, +-inf,
    +-0 and subnormals; never used in timed runs."""
    x = x.copy()
    n = x.size
    idx = np.arange(n, dtype=np.uint64)
    h = splitmix64_np(idx + np.uint64(_seed_key(seed ^ 0x5eed)))
    hit = (h >> np.uint64(40)).astype(np.float64) / float(1 << 24) < rate
    pick = ((h >> np.uint64(8)) & np.uint64(0xFF)).astype(np.int64) % len(_SPECIALS)
    flat = x.reshape(-1)
    flat[hit] = _SPECIALS[pick[hit]]
    return x


# iris-like column ranges (BASELINE.json configs[0])
IRIS_RANGES = ((4.3, 7.9), (2.0, 4.4), (1.0, 6.9), (0.1, 2.5))


def iris_like_x(seed: int = 1, n_rows: int = 150) -> np.ndarray:
    """150x4 values on the 0.1 lattice inside iris's per-column ranges, fp32."""
    out = np.empty((n_rows, 4), dtype=np.float32)
    key = _seed_key(seed)
    for c, (lo, hi) in enumerate(IRIS_RANGES):
        steps = int(round((hi - lo) * 10)) + 1
        h = splitmix64_np(np.arange(n_rows, dtype=np.uint64) * np.uint64(4) + np.uint64(c)
                          + np.uint64(key))
        k = (h >> np.uint64(11)).astype(np.int64) % steps
        out[:, c] = np.float32(np.round(lo + 0.1 * k, 1))
    return out
