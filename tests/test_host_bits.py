"""The host half of the bit-stream host step (csrc/host_bits.cpp) through
its C ABI (hga_host_pack_bits / hga_host_unpack_bits): no GPU needed.

hga_step_host_bits packs the caller's int8 (4N, m, m) population into a
flat bit stream (bit e set iff byte e is -1) on libhga's host thread pool,
validating every byte is +-1, and unpacks the new population from the
stream; these tests pin both against numpy (np.packbits, little bit order)
on sizes that split into many pool tasks and on ragged tails.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2208_14961_b200._lib import FLAG_NOT_SIGN, lib


def _pack_np(x: np.ndarray) -> np.ndarray:
    bits = np.packbits((x.reshape(-1) < 0).astype(np.uint8), bitorder="little")
    words = (x.size + 31) // 32
    return np.pad(bits, (0, 4 * words - bits.size)).view("<u4")


def _pack(x: np.ndarray) -> tuple[int, np.ndarray]:
    x = np.ascontiguousarray(x, dtype=np.int8)
    out = np.full((x.size + 31) // 32, 0xDEADBEEF, dtype=np.uint32)
    rc = lib.hga_host_pack_bits(x.ctypes.data, x.size, out.ctypes.data)
    return rc, out


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 4096 * 3 + 17, 40_000 * 400, 2_000_003])
def test_pack_matches_numpy_and_round_trips(n):
    rng = np.random.default_rng(n)
    x = rng.choice(np.array([-1, 1], dtype=np.int8), size=n)
    rc, words = _pack(x)
    assert rc == 0
    assert np.array_equal(words, _pack_np(x))
    back = np.zeros(n, dtype=np.int8)
    lib.hga_host_unpack_bits(words.ctypes.data, n, back.ctypes.data)
    assert np.array_equal(back, x)


@pytest.mark.parametrize("bad", [0, 2, -2, 127, -128, 3])
@pytest.mark.parametrize("where", ["first", "middle", "tail"])
def test_pack_rejects_entries_that_are_not_signs(bad, where):
    n = 1_000_037  # a partial last word
    x = np.ones(n, dtype=np.int8)
    pos = {"first": 0, "middle": n // 2 + 5, "tail": n - 1}[where]
    x[pos] = bad
    rc, _ = _pack(x)
    assert rc == FLAG_NOT_SIGN


def test_population_stream_layout():
    """Matrix k of an (n, m, m) population occupies stream bits
    [k m^2, (k+1) m^2), row-major: the layout k_bits_to_cols reads."""
    m, n = 20, 7
    rng = np.random.default_rng(3)
    pop = rng.choice(np.array([-1, 1], dtype=np.int8), size=(n, m, m))
    rc, words = _pack(pop)
    assert rc == 0
    for k, r, j in ((0, 0, 0), (3, 5, 7), (6, 19, 19), (1, 0, 19)):
        e = k * m * m + r * m + j
        assert ((int(words[e >> 5]) >> (e & 31)) & 1) == int(pop[k, r, j] < 0)


def test_empty_and_tiny():
    assert lib.hga_host_pack_bits(None, 0, None) == 0
    lib.hga_host_unpack_bits(None, 0, None)


@pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")
def test_pack_in_a_forked_child():
    """A child forked after the pool's workers started has none of them: the
    packer runs inline there instead of waiting for threads that do not exist."""
    import os

    x = np.random.default_rng(5).choice(np.array([-1, 1], dtype=np.int8), size=300_001)
    assert _pack(x)[0] == 0  # the parent's pool is running
    pid = os.fork()
    if pid == 0:  # child
        ok = False
        try:
            rc, words = _pack(x)
            back = np.zeros(x.size, dtype=np.int8)
            lib.hga_host_unpack_bits(words.ctypes.data, x.size, back.ctypes.data)
            ok = rc == 0 and np.array_equal(words, _pack_np(x)) and np.array_equal(back, x)
        finally:
            os._exit(0 if ok else 1)
    import time

    deadline = time.monotonic() + 60
    while True:  # never hang the suite on a child that deadlocked
        done, status = os.waitpid(pid, os.WNOHANG)
        if done:
            break
        if time.monotonic() > deadline:
            os.kill(pid, 9)
            os.waitpid(pid, 0)
            pytest.fail("forked child did not finish")
        time.sleep(0.01)
    assert os.WIFEXITED(status) and os.WEXITSTATUS(status) == 0
