"""Seeded random streams, bit-compatible with the reference ``Rng``.

Restates rng.cpp (fnv1a64 :7-15, splitmix64_next :17-22, xoshiro256++
Rng::Rng :32-36, stream :38-43, pixel_stream :45-55, next_u64 :57-67,
uniform :69-73, index :79-81) so host-side assets (palettes, light SPDs,
codec and MLP weights) are drawn exactly as the reference would draw them.

Large per-element arrays use a *counter* stream instead (value i of key k is
``splitmix64(k + (i + 1) * gamma)``), which vectorises in numpy and on the
device (``hc_synth_*``) and does not depend on how the work is sharded.
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def fnv1a64(data: bytes, basis: int = 0xCBF29CE484222325) -> int:
    h = basis
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & MASK
    return h


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def splitmix64_next(state: int) -> tuple[int, int]:
    """Returns (output, new_state) — splitmix64_next(uint64_t&) (rng.cpp:17-22)."""
    state = (state + GAMMA) & MASK
    return _mix(state), state


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & MASK


class Rng:
    """xoshiro256++ (rng.cpp:32-96)."""

    def __init__(self, seed: int):
        st = seed & MASK
        s = []
        for _ in range(4):
            v, st = splitmix64_next(st)
            s.append(v)
        self.s = s

    @staticmethod
    def stream(seed: int, purpose: str) -> "Rng":
        return Rng(stream_key(seed, purpose))

    @staticmethod
    def pixel_stream(seed: int, x: int, y: int, sample: int, lane: int) -> "Rng":
        st = seed & MASK
        h, st = splitmix64_next(st)
        st = h ^ ((x & 0xFFFFFFFF) | ((y & 0xFFFFFFFF) << 32))
        h, st = splitmix64_next(st)
        st = h ^ ((sample & 0xFFFFFFFF) | ((lane & 0xFFFFFFFF) << 32))
        v, _ = splitmix64_next(st)
        return Rng(v)

    def next_u64(self) -> int:
        s = self.s
        result = (_rotl((s[0] + s[3]) & MASK, 23) + s[0]) & MASK
        t = (s[1] << 17) & MASK
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def uniform(self, a: float = 0.0, b: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return u if (a == 0.0 and b == 1.0) else a + (b - a) * u

    def index(self, n: int) -> int:
        return self.next_u64() % n


def stream_key(seed: int, purpose: str) -> int:
    """The seed Rng::stream hands to Rng (rng.cpp:38-43); also the key of the
    counter stream for `purpose`."""
    st = (seed ^ fnv1a64(purpose.encode())) & MASK
    v, _ = splitmix64_next(st)
    return v


# ----------------------------------------------------------------- counter streams (numpy)
def ctr_u64(key: int, index: np.ndarray) -> np.ndarray:
    """splitmix64(key + (i + 1) * gamma) for an array of indices (uint64 wraparound)."""
    i = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (i + np.uint64(1)) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def ctr_u24(key: int, index: np.ndarray) -> np.ndarray:
    """U[0,1) float32 with 24 random bits: (v >> 40) * 2^-24 (exact in fp32)."""
    return (ctr_u64(key, index) >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
