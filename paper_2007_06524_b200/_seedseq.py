"""Vectorised numpy.random.SeedSequence over many seeds at once.

The reference derives every realization's seed with
``SeedSequence(entropy=master, spawn_key=(m,)).generate_state(1, uint64)``
(lattice.py:273-276) and keys its Philox stream with
``SeedSequence(seed).generate_state(2, uint64)`` (lattice.py:279-281): two
Python-level SeedSequence objects per realization, 16 ms for a config-3 batch --
the only host work of the seeds-to-solutions pipeline.  This module restates
SeedSequence's published hashing (O'Neill's ``seed_seq_fe``, as implemented in
numpy's bit_generator: pool of four 32-bit words, ``hashmix`` / ``mix`` with the
constants below) on uint32 arrays, one row per seed; the results are
bit-identical to numpy's (tests/test_host_api.py).
"""

from __future__ import annotations

import numpy as np

_POOL = 4
_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_SHIFT = np.uint32(16)
_M32 = 0xFFFFFFFF


class _Hash:
    """hashmix with its evolving multiplier (a scalar sequence independent of the data)."""

    def __init__(self, init):
        self.c = init

    def __call__(self, value):
        value = value ^ np.uint32(self.c)
        self.c = (self.c * _MULT_A) & _M32
        value = value * np.uint32(self.c)
        return value ^ (value >> _SHIFT)


def _mix(x, y):
    r = np.uint32(_MIX_L) * x - np.uint32(_MIX_R) * y
    return r ^ (r >> _SHIFT)


def _pool(words: np.ndarray) -> list:
    """Entropy pool of SeedSequence for each row of ``words`` ((B, k) uint32, k >= 4: the
    assembled entropy, zero-padded -- a missing word and a zero word hash alike)."""
    h = _Hash(_INIT_A)
    k = words.shape[1]
    mixer = [h(words[:, i].copy()) for i in range(_POOL)]
    for i_src in range(_POOL):
        for i_dst in range(_POOL):
            if i_src != i_dst:
                mixer[i_dst] = _mix(mixer[i_dst], h(mixer[i_src]))
    for i_src in range(_POOL, k):
        for i_dst in range(_POOL):
            mixer[i_dst] = _mix(mixer[i_dst], h(words[:, i_src].copy()))
    return mixer


def _generate32(pool: list, n_words: int) -> np.ndarray:
    c = _INIT_B
    out = np.empty((pool[0].shape[0], n_words), dtype=np.uint32)
    for i in range(n_words):
        v = pool[i % _POOL] ^ np.uint32(c)
        c = (c * _MULT_B) & _M32
        v = v * np.uint32(c)
        out[:, i] = v ^ (v >> _SHIFT)
    return out


def _words64(x: np.ndarray, n: int) -> np.ndarray:
    """Little-endian 32-bit words of non-negative integers < 2^64, zero-padded to n columns."""
    x = np.asarray(x, dtype=np.uint64)
    w = np.zeros((x.shape[0], n), dtype=np.uint32)
    w[:, 0] = (x & np.uint64(_M32)).astype(np.uint32)
    w[:, 1] = (x >> np.uint64(32)).astype(np.uint32)
    return w


def derive_seeds(master_seed: int, indices) -> np.ndarray:
    """``[derive_seed(master_seed, m) for m in indices]`` as a uint64 array (lattice.py:273-276)."""
    idx = np.asarray(indices, dtype=np.uint64).reshape(-1)
    master = int(master_seed)
    if master < 0 or master >= 1 << 128 or (idx.size and int(idx.max()) >= 1 << 32):
        # outside the vectorised word layout: numpy itself
        return np.array([np.random.SeedSequence(entropy=master, spawn_key=(int(m),)).generate_state(1, np.uint64)[0]
                         for m in idx], dtype=np.uint64)
    with np.errstate(over="ignore"):
        words = np.zeros((idx.shape[0], _POOL + 1), dtype=np.uint32)
        for i in range(_POOL):  # the run entropy, padded to the pool size because a spawn key follows
            words[:, i] = (master >> (32 * i)) & _M32
        words[:, _POOL] = idx.astype(np.uint32)
        st = _generate32(_pool(words), 2)
    return st[:, 0].astype(np.uint64) | (st[:, 1].astype(np.uint64) << np.uint64(32))


def philox_keys(seeds) -> np.ndarray:
    """(B, 2) uint64 keys ``SeedSequence(seed).generate_state(2, uint64)`` (lattice.py:279-281)."""
    s = np.asarray([int(v) for v in seeds], dtype=object)
    if any(v < 0 or v >= 1 << 64 for v in s):
        return np.stack([np.random.SeedSequence(int(v)).generate_state(2, np.uint64) for v in s]
                        ).astype(np.uint64).reshape(-1, 2)
    with np.errstate(over="ignore"):
        st = _generate32(_pool(_words64(s.astype(np.uint64), _POOL)), 4)
    lo = st[:, 0::2].astype(np.uint64)
    hi = st[:, 1::2].astype(np.uint64)
    return (lo | (hi << np.uint64(32))).reshape(-1, 2)
