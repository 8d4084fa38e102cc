"""Counter-based random streams, drop-in for hadamard_ga.rand (rand.py:1-156).

`RngStream` keeps the reference's (seed, stream_id, counter) addressing and
splitmix64 hashing exactly (rand.py:39-77); the vector draws run on the GPU
through libhga (hga_ref_uniform / hga_ref_permutation) and come back as numpy
arrays, bit-identical to the reference's.  Scalar draws (`next_u64`,
`uniform_int`) are a few integer operations and stay on the host -- they are
key arithmetic, like computing a kernel argument, not a data path.

The production GA does not use these streams: it draws from per-thread
Philox4x32-10 counters inside the kernels (csrc/generation.cu).  These are
the "reference-stream" mode that replays a reference run bit-for-bit.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _dev
from ._dev import check, lib

__all__ = ["MASK64", "RngStream", "random_seed", "shuffle_column", "stream_key", "mix64"]

MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_SEED_SALT = 0x5851F42D4C957F2D
_STREAM_SALT = 0x14057B7EF767814F


def mix64(x: int) -> int:
    """splitmix64 finalizer (rand.py:39-44)."""
    x &= MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def stream_key(seed: int, stream_id: int) -> int:
    """Per-stream key (rand.py:55-58)."""
    return mix64(mix64(seed ^ _SEED_SALT) ^ mix64((stream_id * _GOLDEN + _STREAM_SALT) & MASK64))


def random_seed() -> int:
    """Fresh 64-bit seed from OS entropy (rand.py:80-82)."""
    return int.from_bytes(os.urandom(8), "big")


def device_uniform(seed: int, stream_id: int, counter: int, lo: int, hi: int, n: int) -> torch.Tensor:
    """Device int64 tensor of RngStream(seed, stream_id, counter).uniform_array(lo, hi, n)."""
    dev = _dev.require_cuda()
    out = torch.empty(max(n, 0), dtype=torch.int64, device=dev)
    if n > 0:
        check(lib.hga_ref_uniform(seed & MASK64, stream_id & MASK64, counter, lo, hi, n, out.data_ptr(),
                                  _dev.stream_ptr()), "hga_ref_uniform")
    return out


def device_permutation(seed: int, stream_id: int, counter: int, n: int) -> torch.Tensor:
    """Device int64 tensor of RngStream(seed, stream_id, counter).permutation(n)."""
    dev = _dev.require_cuda()
    out = torch.empty(n, dtype=torch.int64, device=dev)
    wsb = int(lib.hga_ref_permutation_ws_bytes(n))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    check(lib.hga_ref_permutation(seed & MASK64, stream_id & MASK64, counter, n, out.data_ptr(), ws.data_ptr(),
                                  wsb, _dev.stream_ptr()), "hga_ref_permutation")
    return out


class RngStream:
    """One addressable stream: (seed, stream_id) plus a draw counter (rand.py:85-140)."""

    __slots__ = ("seed", "stream_id", "counter", "_key")

    def __init__(self, seed: int, stream_id: int = 0, counter: int = 0):
        self.seed = seed & MASK64
        self.stream_id = stream_id & MASK64
        self.counter = counter
        self._key = stream_key(self.seed, self.stream_id)

    def __repr__(self) -> str:
        return f"RngStream(seed={self.seed:#x}, stream_id={self.stream_id:#x}, counter={self.counter})"

    def next_u64(self) -> int:
        value = mix64((self._key + self.counter * _GOLDEN) & MASK64)
        self.counter += 1
        return value

    def uniform_int(self, lo: int, hi: int) -> int:
        if lo > hi:
            raise ValueError(f"empty range [{lo}, {hi}]")
        return lo + self.next_u64() % (hi - lo + 1)

    def uniform_array(self, lo: int, hi: int, n: int) -> np.ndarray:
        if lo > hi:
            raise ValueError(f"empty range [{lo}, {hi}]")
        if n < 0:
            raise ValueError("n must be nonnegative")
        out = device_uniform(self.seed, self.stream_id, self.counter, lo, hi, n).cpu().numpy()
        self.counter += n
        return out

    def permutation(self, n: int) -> np.ndarray:
        if n < 1:
            raise ValueError("n must be positive")
        out = device_permutation(self.seed, self.stream_id, self.counter, n).cpu().numpy()
        self.counter += n - 1
        return out


def shuffle_column(matrix: np.ndarray, col: int, stream: RngStream) -> np.ndarray:
    """Fisher-Yates of one column in place (rand.py:143-156).

    A single column is m-1 scalar draws; this is host-side convenience kept
    for API completeness (the population init shuffles every column on the
    GPU, see engine.init_population).
    """
    m = matrix.shape[0]
    if not 1 <= col < m:
        raise IndexError(f"column must be in [1, {m - 1}], got {col}")
    for i1 in range(m - 1):
        i2 = stream.uniform_int(i1, m - 1)
        matrix[i1, col], matrix[i2, col] = matrix[i2, col], matrix[i1, col]
    return matrix
