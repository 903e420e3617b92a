"""Host-side SplitMix64 seeding helpers (mirror of the reference's rng API).

The device kernels carry their own SplitMix64 (`Prg` in csrc/common.cuh); this host copy
serves the public API (`Prg`, `derive_round_seed`, ...) and one-time input
preparation (the TAG_SHUFFLE shard permutation).  Stream conventions follow
reference rng.py:1-136:

* draw i (1-based) of a stream seeded with s is scramble(s + i*GOLDEN);
* per-(client, round) seed = mix64(run_seed ^ (cid << 32 | round));
* named streams (shuffle / synthetic / master sampling) = mix64(run_seed ^ TAG).
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
TAG_SHUFFLE = 0x8000000000000001
TAG_SYNTH = 0x8000000000000002
TAG_MASTER = 0x8000000000000003


def _scramble(z: int) -> int:
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def mix64(z: int) -> int:
    """The SplitMix64 finaliser applied to z + GOLDEN (rng.py:37-42)."""
    return _scramble((z + GOLDEN) & MASK64)


def _scramble_vec(ctr: np.ndarray) -> np.ndarray:
    z = (ctr ^ (ctr >> np.uint64(30))) * np.uint64(MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


class Prg:
    """SplitMix64 stream (rng.py:45-118): scalar and block draws interleave."""

    __slots__ = ("_state", "seed0")

    def __init__(self, seed: int):
        self._state = seed & MASK64
        self.seed0 = self._state

    def next_u64(self) -> int:
        self._state = (self._state + GOLDEN) & MASK64
        return _scramble(self._state)

    def u64_block(self, n: int) -> np.ndarray:
        if n < 0:
            raise ValueError("negative draw count")
        ctr = np.uint64(self._state) + np.uint64(GOLDEN) * np.arange(1, n + 1, dtype=np.uint64)
        self._state = (self._state + n * GOLDEN) & MASK64
        return _scramble_vec(ctr)

    def next_f64(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def f64_block(self, n: int) -> np.ndarray:
        return (self.u64_block(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53

    def randrange(self, bound: int) -> int:
        if bound <= 0:
            raise ValueError("bound must be positive")
        floor = (1 << 64) % bound
        while True:
            u = self.next_u64()
            if u >= floor:
                return u % bound

    def shuffle(self, arr) -> None:
        """Fisher-Yates swapping i with randrange(i+1), i from the top.

        Vectorised draw generation: with no rejection (probability < 2^-40
        per draw at the sizes used here) the draws are one counter block;
        any rejection falls back to the scalar loop from a snapshot.
        """
        n = len(arr)
        if n < 2:
            return
        start = self._state
        bounds = np.arange(n, 1, -1, dtype=np.uint64)  # i + 1 for i = n-1 .. 1
        u = self.u64_block(n - 1)
        floors = (np.uint64(MASK64) % bounds + np.uint64(1)) % bounds  # 2^64 mod b
        if np.any(u < floors):
            self._state = start
            for i in range(n - 1, 0, -1):
                j = self.randrange(i + 1)
                arr[i], arr[j] = arr[j], arr[i]
            return
        js = (u % bounds).astype(np.int64)
        for i, j in zip(range(n - 1, 0, -1), js.tolist()):
            arr[i], arr[j] = arr[j], arr[i]

    def partial_shuffle_prefix(self, n: int, k: int) -> np.ndarray:
        if not 0 <= k <= n:
            raise ValueError("need 0 <= k <= n")
        pool: dict[int, int] = {}
        out = np.empty(k, dtype=np.int64)
        for i in range(k):
            j = i + self.randrange(n - i)
            vi, vj = pool.get(i, i), pool.get(j, j)
            pool[i], pool[j] = vj, vi
            out[i] = vj
        return out


def derive_round_seed(run_seed: int, client_id: int, rnd: int) -> int:
    if not 0 <= client_id < (1 << 32):
        raise ValueError("client_id out of u32 range")
    if not 0 <= rnd < (1 << 32):
        raise ValueError("round out of u32 range")
    return mix64(run_seed ^ ((client_id << 32) | rnd))


def derive_round_prg(run_seed: int, client_id: int, rnd: int) -> Prg:
    return Prg(derive_round_seed(run_seed, client_id, rnd))


def derive_stream(run_seed: int, tag: int) -> Prg:
    return Prg(mix64(run_seed ^ tag))
