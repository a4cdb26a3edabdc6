"""Counter-based SplitMix64 streams, bit-identical to the reference RngStream
(/root/reference/proj/include/diffsim/rng.hpp:11-55).

A stream is keyed by (seed, stream): key = mix(seed ^ phi * (stream + 1)); the
k-th draw (k = 1, 2, ...) is mix(key ^ mix(k)).  Because draws are addressed
by counter, whole blocks of draws vectorise in numpy; ``RngStream`` keeps the
reference's (key, counter) state so a stream can be resumed draw-for-draw.
"""
from __future__ import annotations

import numpy as np

_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO53 = 2.0 ** -53


def mix(z):
    """SplitMix64 finaliser on a uint64 array (rng.hpp:46-51)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _PHI
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class RngStream:
    """Mirror of diffsim::RngStream (rng.hpp:11-55)."""

    def __init__(self, seed: int, stream: int):
        with np.errstate(over="ignore"):
            s = np.array([seed], dtype=np.uint64)
            k = _PHI * (np.array([stream], dtype=np.uint64) + np.uint64(1))
        self.key = mix(s ^ k)[0]
        self.counter = 0

    def next_u64_block(self, n: int) -> np.ndarray:
        ctr = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
        self.counter += n
        return mix(self.key ^ mix(ctr))

    def doubles(self, n: int) -> np.ndarray:
        return (self.next_u64_block(n) >> np.uint64(11)).astype(np.float64) * _TWO53

    def uniform(self, lo, hi, n: int | None = None):
        """n draws of lo + (hi - lo) u (rng.hpp:27-29); a float when n is None."""
        if n is None:
            return float(lo + (hi - lo) * self.doubles(1)[0])
        return lo + (hi - lo) * self.doubles(n)

    def normal(self) -> float:
        """One Box-Muller cosine draw (rng.hpp:35-43)."""
        return float(self.normals(1)[0])

    def next_double(self) -> float:
        return float(self.doubles(1)[0])

    def normals(self, n: int) -> np.ndarray:
        """n Box-Muller cosine draws; each consumes (u1, u2) and re-draws u1
        while u1 <= 0, exactly as rng.hpp:35-43."""
        out = np.empty(n)
        i = 0
        while i < n:
            m = n - i
            start = self.counter
            d = self.doubles(2 * m).reshape(m, 2)
            bad = np.nonzero(d[:, 0] <= 0.0)[0]
            if bad.size:  # rare: fall back to exact sequential semantics
                self.counter = start
                for _ in range(m):
                    u1 = self.next_double()
                    u2 = self.next_double()
                    while u1 <= 0.0:
                        u1 = self.next_double()
                    out[i] = np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925286766559 * u2)
                    i += 1
                return out
            out[i:] = np.sqrt(-2.0 * np.log(d[:, 0])) * np.cos(6.283185307179586476925286766559 * d[:, 1])
            i = n
        return out
