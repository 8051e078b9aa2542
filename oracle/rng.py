"""Counter-based noise, restated in NumPy (TEST INFRASTRUCTURE ONLY).

Reference: ``chainscan/noise.py``.  Every value is a pure function of
(seed, slot-id, t, counter):

* slot ids are FNV-1a 64 of the UTF-8 slot name               (noise.py:41-47)
* the mixer is the splitmix64 finaliser, chained over four words
  seed, a, b, c -- each word offset by the golden constant     (noise.py:50-67)
* uniforms are ((h >> 11) + 0.5) * 2^-53                       (noise.py:70-72)
* value k of a slot at step t uses counter 2k (uniform, chi^2) or the pair
  2k, 2k+1 for Box-Muller normals                              (noise.py:140-156)
* Rademacher probes live in the counter namespace
  a = 0xA5B35705 + iteration, b = t, c = (sample << 32) + d     (noise.py:159-171)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import gammaincinv

from .errors import ConfigurationError

U64 = np.uint64
GOLD = U64(0x9E3779B97F4A7C15)
MIX_A = U64(0xBF58476D1CE4E5B9)
MIX_B = U64(0x94D049BB133111EB)
PROBE_NS = U64(0xA5B35705)
TWO_M53 = 2.0 ** -53


def fnv1a64(text: str) -> np.uint64:
    """FNV-1a over the UTF-8 bytes (noise.py:41-47)."""
    acc = 0xCBF29CE484222325
    for ch in text.encode("utf-8"):
        acc = ((acc ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return U64(acc)


def _avalanche(x):
    """splitmix64 finaliser: xorshift 30 / mul / xorshift 27 / mul / xorshift 31."""
    with np.errstate(over="ignore"):
        x = x ^ (x >> U64(30))
        x = x * MIX_A
        x = x ^ (x >> U64(27))
        x = x * MIX_B
        x = x ^ (x >> U64(31))
    return x


def counter_hash(seed, a, b, c):
    """Four chained avalanche rounds over (seed, a, b, c) (noise.py:60-67)."""
    with np.errstate(over="ignore"):
        h = _avalanche(U64(int(seed) & 0xFFFFFFFFFFFFFFFF) + GOLD)
        for w in (a, b, c):
            h = _avalanche(h ^ (np.asarray(w, dtype=U64) + GOLD))
    return h


def bits_to_unit(bits):
    """Open-interval uniform from the top 53 bits (noise.py:70-72)."""
    return ((bits >> U64(11)).astype(np.float64) + 0.5) * TWO_M53


def _unit_grid(seed, slot_id, ts, counters):
    t_col = np.asarray(ts, dtype=U64).reshape(-1, 1)
    c_row = np.asarray(counters, dtype=U64).reshape(1, -1)
    return bits_to_unit(counter_hash(seed, slot_id, t_col, c_row))


@dataclass(frozen=True)
class SlotSpec:
    """Declared slot: values per step and their law (noise.py:83-104)."""

    count: int
    kind: str
    df: float | None = None

    def __post_init__(self):
        if self.count < 1:
            raise ConfigurationError("slot count must be >= 1")
        if self.kind not in ("standard-normal", "uniform-0-1", "chi-squared"):
            raise ConfigurationError(f"unknown distribution {self.kind!r}")
        if self.kind == "chi-squared":
            if self.df is None or self.df <= 0:
                raise ConfigurationError("chi-squared needs df > 0")
        elif self.df is not None:
            raise ConfigurationError("df is only meaningful for chi-squared")


class NoiseTable:
    """Seed-addressed noise over steps t in [0, T] (noise.py:107-156)."""

    def __init__(self, seed: int, layout: dict, T: int):
        if T < 1:
            raise ConfigurationError("T must be >= 1")
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.layout = dict(layout)
        self.T = int(T)
        self.slot_ids = {k: fnv1a64(k) for k in self.layout}

    def spec(self, slot):
        if slot not in self.layout:
            raise ConfigurationError(f"slot {slot!r} not declared")
        return self.layout[slot]

    def block(self, slot, ts):
        sp = self.spec(slot)
        sid = self.slot_ids[slot]
        k2 = 2 * np.arange(sp.count)
        if sp.kind == "uniform-0-1":
            return _unit_grid(self.seed, sid, ts, k2)
        if sp.kind == "standard-normal":
            u1 = _unit_grid(self.seed, sid, ts, k2)
            u2 = _unit_grid(self.seed, sid, ts, k2 + 1)
            return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        u = _unit_grid(self.seed, sid, ts, k2)
        return 2.0 * gammaincinv(0.5 * sp.df, u)

    def noise_at(self, t, slot, k):
        sp = self.spec(slot)
        if not 0 <= k < sp.count:
            raise IndexError(f"k={k} out of range")
        if not 0 <= t <= self.T:
            raise IndexError(f"t={t} out of range")
        return float(self.block(slot, [t])[0, k])


def rademacher_probe(seed, iteration, ts, sample, dim):
    """+-1 probes from the sign bit of the counter hash (noise.py:159-171)."""
    with np.errstate(over="ignore"):
        a = PROBE_NS + U64(int(iteration))
        c = (U64(int(sample)) << U64(32)) + np.arange(dim, dtype=U64).reshape(1, -1)
    t_col = np.asarray(ts, dtype=U64).reshape(-1, 1)
    top = counter_hash(seed, a, t_col, c) >> U64(63)
    return np.where(top == U64(1), 1.0, -1.0)
