"""Key holder for the counter-based generator (mirrors pkg/src/cuppl/rng.py:16-45).

`Rng(seed, stream)` derives the same 64-bit key as the reference (rng.py:26-29) and
`split(i)` the same child key (rng.py:31-37), so a reference `cuppl.rng.Rng` and this class
are interchangeable as the `rng` argument of the inference entry points: the engines only
read `rng.key`. The GPU draws are Philox4x32-10 keyed by that key with counter
(id_lo, id_hi, block, tag) (include/cuppl_gpu.h), replacing the SplitMix counter of
rng.py:39-41; `next_u64` / `uniform` are kept for API compatibility and host-side use.
"""

from __future__ import annotations

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    """SplitMix64 finaliser (rng.py:16-20)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


class Rng:
    __slots__ = ("key", "counter", "seed")

    def __init__(self, seed=0, stream=0):
        self.seed = seed
        self.key = _mix((seed & _MASK) ^ _mix((stream + 1) * _GOLDEN))
        self.counter = 0

    def split(self, i):
        """Independent child stream for index i; deterministic in (seed, i) (rng.py:31-37)."""
        child = Rng.__new__(Rng)
        child.seed = self.seed
        child.key = _mix(self.key ^ _mix((i + 1) * _GOLDEN))
        child.counter = 0
        return child

    def next_u64(self):
        self.counter = (self.counter + _GOLDEN) & _MASK
        return _mix(self.key ^ self.counter)

    def uniform(self):
        """Float in [0, 1) with 53 random bits (rng.py:43-45)."""
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))


def key_of(rng) -> int:
    """The 64-bit Philox key of an Rng (this module's or the reference's)."""
    if isinstance(rng, int):
        return rng & _MASK
    key = getattr(rng, "key", None)
    if key is None:
        raise TypeError("rng must be an Rng (cuppl.rng.Rng-compatible) or an int key")
    return int(key) & _MASK


def seed_of(rng):
    return getattr(rng, "seed", None)
