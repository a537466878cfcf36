"""Order-independent fingerprints of a pair multiset, vectorised with numpy (test helper).

The definition is oracle/sj_oracle.c's (orc_grid_digest):
    F_a(S) = sum_x mix_a(x) mod 2^64,  F_b(S) = sum_x mix_b(x) mod 2^64,
    F_c(cnt) = sum_i mix_a(i << 32 | cnt_i) mod 2^64,
mix_a = SplitMix64's output function of x + 0x9E3779B97F4A7C15, mix_b = MurmurHash3 fmix64 of
x ^ 0xC2B2AE3D27D4EB4F.  tests/test_oracle_pins.py pins these numpy versions against the C oracle's
mixers, and those against the published reference values.  The CUDA library computes the same
F_a / F_b on the device (sj_result_fingerprint): a third, independent implementation.
"""
import numpy as np

_U = np.uint64


def mix_a(x: np.ndarray) -> np.ndarray:
    z = np.asarray(x, dtype=np.uint64) + _U(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
    return z ^ (z >> _U(31))


def mix_b(x: np.ndarray) -> np.ndarray:
    k = np.asarray(x, dtype=np.uint64) ^ _U(0xC2B2AE3D27D4EB4F)
    with np.errstate(over="ignore"):
        k ^= k >> _U(33)
        k *= _U(0xFF51AFD7ED558CCD)
        k ^= k >> _U(33)
        k *= _U(0xC4CEB9FE1A85EC53)
        k ^= k >> _U(33)
    return k


def _sum64(v: np.ndarray) -> int:
    # exact sum mod 2^64 (numpy's uint64 sum wraps, which is the definition)
    with np.errstate(over="ignore"):
        return int(np.sum(v, dtype=np.uint64))


def fingerprint(pairs: np.ndarray, chunk: int = 1 << 24) -> tuple:
    """(F_a, F_b) of an explicit array of packed pairs."""
    p = np.asarray(pairs, dtype=np.uint64)
    fa = fb = 0
    for s in range(0, len(p), chunk):
        c = p[s:s + chunk]
        fa = (fa + _sum64(mix_a(c))) % 2**64
        fb = (fb + _sum64(mix_b(c))) % 2**64
    return fa, fb


def count_fingerprint(counts: np.ndarray, base: int = 0) -> int:
    """F_c of per-query counts cnt[i - base] (queries base .. base + len - 1)."""
    c = np.asarray(counts).astype(np.uint64)
    ids = np.arange(base, base + len(c), dtype=np.uint64)
    return _sum64(mix_a((ids << _U(32)) | c))
