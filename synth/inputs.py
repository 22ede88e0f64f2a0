"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no pruning, no GEMM, no plan).
It only turns (config seed, tensor name, rank, element index) into numbers with
the value distributions SURVEY.md §8(d) fixes:

* X ~ N(0,1), G ~ N(0,1)                         (activations / upstream grads)
* W ~ U(-1/sqrt(d_in), +1/sqrt(d_in))            (SPEC S:307 initialisation)
* priority scores ~ lognormal(ln 1e-3, 1.0), fp32 (the paper's per-column
  weight-variation δ, Alg.1 l.4, is non-negative and heavy-tailed)

Every floating value is rounded to bf16 (round-to-nearest-even) and returned as
float64 holding that exact bf16 value, so the fp64 oracle and the bf16 GPU path
consume bit-identical inputs.

Generator: counter-based splitmix64.  Element (i, j) of a tensor with `cols`
columns uses counter i*cols + j, so any rank can generate just its own shard of
a dense tensor and the shards concatenate to the dense tensor exactly.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 240111469  # seed s = 240111469 + config index

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _fnv1a64(name: str) -> int:
    h = 0xCBF29CE484222325
    for b in name.encode():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def tensor_key(seed: int, name: str, rank: int = 0) -> np.uint64:
    k = np.array([(seed ^ _fnv1a64(name) ^ ((rank + 1) * 0x9E3779B97F4A7C15)) & 0xFFFFFFFFFFFFFFFF],
                 dtype=np.uint64)
    return _splitmix64(k)[0]


def _uniform01(key: np.uint64, counters: np.ndarray) -> np.ndarray:
    """Uniform doubles in (0, 1] from 53 random bits."""
    with np.errstate(over="ignore"):
        r = _splitmix64(counters.astype(np.uint64) + key)
    return ((r >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16 (ties to even), returned as float64."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def _grid_counters(rows: int, cols: int, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    ii = np.arange(r0, r1, dtype=np.uint64)[:, None]
    jj = np.arange(c0, c1, dtype=np.uint64)[None, :]
    return ii * np.uint64(cols) + jj


def normal(seed: int, name: str, rows: int, cols: int, rank: int = 0,
           r0: int = 0, r1: int | None = None, c0: int = 0, c1: int | None = None) -> np.ndarray:
    """bf16-rounded N(0,1) block [r0:r1, c0:c1] of a rows x cols tensor (Box-Muller)."""
    r1 = rows if r1 is None else r1
    c1 = cols if c1 is None else c1
    key = tensor_key(seed, name, rank)
    cnt = _grid_counters(rows, cols, r0, r1, c0, c1) * np.uint64(2)
    u1 = _uniform01(key, cnt)
    u2 = _uniform01(key, cnt + np.uint64(1))
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return round_bf16(z)


def uniform_sym(seed: int, name: str, rows: int, cols: int, bound: float, rank: int = 0,
                r0: int = 0, r1: int | None = None, c0: int = 0, c1: int | None = None) -> np.ndarray:
    """bf16-rounded U(-bound, +bound) block of a rows x cols tensor."""
    r1 = rows if r1 is None else r1
    c1 = cols if c1 is None else c1
    key = tensor_key(seed, name, rank)
    u = _uniform01(key, _grid_counters(rows, cols, r0, r1, c0, c1))
    return round_bf16((2.0 * u - 1.0) * bound)


def lognormal_scores(seed: int, name: str, n: int, rank: int = 0,
                     mu: float = float(np.log(1e-3)), sigma: float = 1.0,
                     levels: int = 0) -> np.ndarray:
    """fp32 priority scores ~ lognormal(mu, sigma), returned as float32.

    levels > 0 quantises the scores to that many distinct values (the tie-stress
    variant of config c3)."""
    key = tensor_key(seed, name, rank)
    cnt = np.arange(n, dtype=np.uint64) * np.uint64(2)
    u1 = _uniform01(key, cnt)
    u2 = _uniform01(key, cnt + np.uint64(1))
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    s = np.exp(mu + sigma * z)
    if levels > 0:
        lo, hi = s.min(), s.max()
        q = np.floor((s - lo) / (hi - lo + 1e-300) * levels)
        s = lo + q * (hi - lo) / levels
    return s.astype(np.float32)


def index_list(seed: int, name: str, n: int, k: int, rank: int = 0) -> np.ndarray:
    """k distinct indices of range(n), ascending (random-priority / ZERO-Rd case)."""
    key = tensor_key(seed, name, rank)
    u = _uniform01(key, np.arange(n, dtype=np.uint64))
    return np.sort(np.argsort(u, kind="stable")[:k]).astype(np.int32)
