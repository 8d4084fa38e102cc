"""Sign-matrix math, drop-in for hadamard_ga.core (core.py:1-113).

`fitness_f1` / `fitness_f2` / `is_hadamard` run through the same fused GPU
penalty kernel as `engine.evaluate` (a batch of one), so a solution reported
by the GA is certified by the kernel path *and* can be re-checked with the
reference's own int32 `core.gram` by the caller.  `as_sign_matrix`,
`is_balanced` and `sylvester` are input validation / test-fixture helpers and
stay in numpy, as in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine

__all__ = [
    "SYLVESTER_MAX_POWER",
    "as_sign_matrix",
    "is_balanced",
    "gram",
    "fitness_f1",
    "fitness_f2",
    "fitness_sq",
    "orthogonal_pairs",
    "is_hadamard",
    "sylvester",
]

SYLVESTER_MAX_POWER = 10


def as_sign_matrix(matrix) -> np.ndarray:
    """Validate a square +1/-1 matrix and return it as int8 (core.py:29-40)."""
    q = np.asarray(matrix)
    if q.ndim != 2 or q.shape[0] != q.shape[1] or q.shape[0] < 1:
        raise ValueError(f"expected a square matrix, got shape {q.shape}")
    if not np.isin(q, (-1, 1)).all():
        bad = q[~np.isin(q, (-1, 1))].ravel()[0]
        raise ValueError(f"matrix entries must be +1 or -1, found {bad!r}")
    return q.astype(np.int8, copy=False)


def is_balanced(matrix) -> bool:
    """Population contract: order 4k, all-+1 first column, balanced columns (core.py:43-56)."""
    q = as_sign_matrix(matrix)
    m = q.shape[0]
    if m % 4 != 0:
        return False
    if not (q[:, 0] == 1).all():
        return False
    return bool((q[:, 1:].sum(axis=0, dtype=np.int64) == 0).all())


def gram(matrix) -> np.ndarray:
    """Column Gram matrix, exact int32 (core.py:59-67), computed on the GPU."""
    q = as_sign_matrix(matrix)
    t = torch.from_numpy(q.astype(np.float32)).cuda()
    g = (t.T @ t).round().to(torch.int32)  # |g| <= m < 2^24: exact in fp32
    return g.cpu().numpy()


def _one(matrix, name: str) -> int:
    q = as_sign_matrix(matrix)
    return int(engine.evaluate(q[None], name)[0])


def fitness_f1(matrix) -> int:
    """sum |G| - m^2 (core.py:70-78)."""
    return _one(matrix, "f1")


def fitness_f2(matrix) -> int:
    """nnz(G) - m (core.py:81-89)."""
    return _one(matrix, "f2")


def fitness_sq(matrix) -> int:
    """sum over i != j of g_ij^2."""
    return _one(matrix, "sq")


def orthogonal_pairs(matrix) -> int:
    """Number of column pairs i < j with g_ij = 0."""
    return _one(matrix, "orth")


def is_hadamard(matrix) -> bool:
    """G == m I (core.py:92-96)."""
    return fitness_f2(matrix) == 0


def sylvester(power: int, max_power: int = SYLVESTER_MAX_POWER) -> np.ndarray:
    """Order-2**power Hadamard matrix by doubling (core.py:99-113); fixture helper."""
    if power < 0:
        raise ValueError("power must be nonnegative")
    if power > max_power:
        raise ValueError(f"power {power} exceeds size limit {max_power}")
    h = np.ones((1, 1), dtype=np.int8)
    for _ in range(power):
        h = np.block([[h, h], [h, -h]]).astype(np.int8)
    return h
