"""Seeded 64-bit hash family (host-side metadata and scalar forms).

Restates reference ``hashing.py``: mix64 finalizer (:56-75), derived seeds
``seed_i = mix64(base ^ mix64(i+1))`` (:96-100), words
``mix64(seed_i ^ key)`` (:114-118), bit positions ``word % range`` (:121-126,
:141-145) and unit values ``(word+1) * 2**-64`` (:129-138, :148-153).

Only O(1) host work lives here (seed derivation, scalar per-key forms used
by the reference API).  Vector hashing of whole neighbourhoods happens on the
device inside the sketch builders (csrc/pg_build.cu); ``hash_words`` /
``bit_positions`` / ``unit_values`` below run the device kernel
``pg_hash_words``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["DEFAULT_HASH_SEED", "HashFamily", "hash_to_bit", "hash_to_unit",
           "hash_words", "bit_positions", "unit_values", "mix64"]

M64 = (1 << 64) - 1
C1 = 0xFF51AFD7ED558CCD
C2 = 0xC4CEB9FE1A85EC53

#: default base seed (reference hashing.py:48)
DEFAULT_HASH_SEED = 0x9E3779B97F4A7C15


def mix64(x: int) -> int:
    """MurmurHash3-style finalizer on a Python int, mod 2**64."""
    x &= M64
    x = (x ^ (x >> 33)) * C1 & M64
    x = (x ^ (x >> 33)) * C2 & M64
    return x ^ (x >> 33)


@dataclass(frozen=True)
class HashFamily:
    """``count`` deterministic functions derived from one base seed."""

    base_seed: int = DEFAULT_HASH_SEED
    count: int = 1
    algorithm: str = "mix64"
    _seeds: tuple = field(init=False, repr=False, compare=False, default=())

    def __post_init__(self):
        if self.algorithm != "mix64":
            raise ValueError(f"unknown hash algorithm {self.algorithm!r}")
        if self.count < 1:
            raise ValueError("hash family needs at least one function")
        base = self.base_seed & M64
        object.__setattr__(self, "base_seed", base)
        object.__setattr__(self, "_seeds", tuple(
            mix64(base ^ mix64(i + 1)) for i in range(self.count)))

    def seed(self, i: int) -> int:
        self._check_index(i)
        return self._seeds[i]

    def seeds_array(self) -> np.ndarray:
        """All derived seeds as uint64 (what the device builders consume)."""
        return np.asarray(self._seeds, dtype=np.uint64)

    def _check_index(self, i: int) -> None:
        if not 0 <= i < self.count:
            raise IndexError(
                f"hash function index {i} out of range for family of {self.count}")


def hash_to_bit(family: HashFamily, i: int, key: int, range_: int) -> int:
    if range_ < 1:
        raise ValueError("range must be >= 1")
    family._check_index(i)
    return mix64(family._seeds[i] ^ (key & M64)) % range_


def hash_to_unit(family: HashFamily, i: int, key: int) -> float:
    family._check_index(i)
    w = mix64(family._seeds[i] ^ (key & M64))
    return float(w + 1) * 2.0 ** -64


def hash_words(family: HashFamily, i: int, keys) -> np.ndarray:
    """Raw words of many keys, computed on the device (pg_hash_words)."""
    import torch
    from . import _native as N
    family._check_index(i)
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.int64).reshape(-1))
    if len(k) == 0:
        return np.empty(0, dtype=np.uint64)
    kd = torch.from_numpy(k).cuda()
    out = torch.empty(len(k), dtype=torch.int64, device="cuda")
    N.call("pg_hash_words", N.ptr(kd), len(k), family._seeds[i], N.ptr(out),
           N.stream_handle())
    return out.cpu().numpy().view(np.uint64)


def bit_positions(family: HashFamily, i: int, keys, range_: int) -> np.ndarray:
    if range_ < 1:
        raise ValueError("range must be >= 1")
    return (hash_words(family, i, keys) % np.uint64(range_)).astype(np.int64)


def unit_values(family: HashFamily, i: int, keys) -> np.ndarray:
    w = hash_words(family, i, keys)
    out = (w + np.uint64(1)).astype(np.float64)
    out[w == np.uint64(M64)] = float(2 ** 64)
    return out * 2.0 ** -64
