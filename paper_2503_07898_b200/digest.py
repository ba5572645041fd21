"""Host restatement of the device state digest (csrc/digest.cuh).

    h(i, b) = splitmix64(b ^ splitmix64(i))      b = IEEE bits of canonical element i
    digest  = (sum_i h mod 2^64, xor_i rotl(h, 29))

Used by the tests to check the device digest against a canonical state read
back to the host at small sizes; at full size (512^3) the engines' digests are
compared with each other (partition invariance, strategy equivalence, fused ==
staged) without moving the field to the host.
"""
from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def digest(canonical: np.ndarray, base: int = 0, chunk: int = 1 << 22) -> tuple[int, int]:
    """Digest of a canonical fp64 array (element i at index base + i)."""
    x = np.ascontiguousarray(canonical, np.float64).view(np.uint64).ravel()
    s = 0
    r = np.uint64(0)
    with np.errstate(over="ignore"):
        for o in range(0, x.size, chunk):
            b = x[o:o + chunk]
            idx = np.arange(base + o, base + o + b.size, dtype=np.uint64)
            h = _mix(b ^ _mix(idx))
            s = (s + int(h.sum(dtype=np.uint64))) & int(_M)
            r ^= np.bitwise_xor.reduce((h << np.uint64(29)) | (h >> np.uint64(35)))
    return s, int(r)
