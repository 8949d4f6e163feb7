"""Counter-based splitmix64 RNG (reading R7).

u64(seed, stream, idx) = splitmix64( splitmix64(seed ^ stream*K) + idx )   (mod 2^64)
U01 = (u64 >> 11) * 2^-53   (double in [0, 1))
"""
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_KSTREAM = np.uint64(0xD1B54A32D192ED03)


def splitmix64(x):
    """Vectorised splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def _stream_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream & 0xFFFFFFFFFFFFFFFF) * _KSTREAM)
    return splitmix64(np.array([k], dtype=np.uint64))[0]


def u64(seed: int, stream: int, idx) -> np.ndarray:
    key = _stream_key(seed, stream)
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(key + idx)


def u01(seed: int, stream: int, n_or_idx) -> np.ndarray:
    """U[0,1) doubles for counters 0..n-1 (or an explicit counter array)."""
    idx = np.arange(n_or_idx, dtype=np.uint64) if np.isscalar(n_or_idx) else n_or_idx
    return (u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(seed: int, stream: int, n: int, lo: float, hi: float) -> np.ndarray:
    """U[lo, hi) in float64 (callers round once to float32 where a float32 is wanted)."""
    return lo + (hi - lo) * u01(seed, stream, n)


def normal(seed: int, stream: int, n: int) -> np.ndarray:
    """Standard normals by Box-Muller from counters 2i, 2i+1 of the stream."""
    idx = np.arange(2 * n, dtype=np.uint64)
    u = u01(seed, stream, idx).reshape(n, 2)
    u1 = 1.0 - u[:, 0]  # (0, 1]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u[:, 1])
