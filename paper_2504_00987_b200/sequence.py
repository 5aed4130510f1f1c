"""Host-side value helpers for packed ±1 sequences (Python mirror of
proj/include/labsolve/sequence.hpp:15-68).

Bit convention (sequence.hpp:11-14): position i lives in word i // 64 at bit
i % 64; bit 0 = spin +1, bit 1 = spin -1; padding bits are always zero.
Hex codec (sequence.cpp:89-128): uppercase, ceil(n/4) digits, the first digit
carries positions 0..3 with position 0 in the digit's most significant bit.
"""
from __future__ import annotations

import numpy as np


def nwords(n: int) -> int:
    return (n + 63) // 64


def tail_mask(n: int) -> int:
    rem = n % 64
    return (1 << 64) - 1 if rem == 0 else (1 << rem) - 1


def decode_hex(hexstr: str, n: int) -> np.ndarray:
    """decode_hex (sequence.cpp:89-114); raises ValueError like the reference's
    std::invalid_argument."""
    if n < 1:
        raise ValueError("decode_hex: length must be positive")
    want = (n + 3) // 4
    if len(hexstr) != want:
        raise ValueError(f"decode_hex: expected {want} digits for length {n}, got {len(hexstr)}")
    w = [0] * nwords(n)
    for d, ch in enumerate(hexstr):
        try:
            v = int(ch, 16)
        except ValueError:
            raise ValueError(f"decode_hex: invalid digit '{ch}'") from None
        for b in range(4):
            pos = d * 4 + b
            bit = (v >> (3 - b)) & 1
            if pos >= n:
                if bit:
                    raise ValueError("decode_hex: nonzero padding bit")
                continue
            if bit:
                w[pos >> 6] |= 1 << (pos & 63)
    return np.array(w, dtype=np.uint64)


def encode_hex(words, n: int) -> str:
    """encode_hex (sequence.cpp:116-128)."""
    w = [int(x) for x in words]
    out = []
    for d in range((n + 3) // 4):
        v = 0
        for b in range(4):
            pos = d * 4 + b
            if pos < n and (w[pos >> 6] >> (pos & 63)) & 1:
                v |= 1 << (3 - b)
        out.append("0123456789ABCDEF"[v])
    return "".join(out)


def spins(words, n: int) -> np.ndarray:
    w = [int(x) for x in words]
    return np.array([-1 if (w[i >> 6] >> (i & 63)) & 1 else 1 for i in range(n)], dtype=np.int64)


def from_spins(s) -> np.ndarray:
    n = len(s)
    w = [0] * nwords(n)
    for i, v in enumerate(s):
        if v < 0:
            w[i >> 6] |= 1 << (i & 63)
    return np.array(w, dtype=np.uint64)


def energy_naive(words, n: int) -> int:
    """energy (sequence.cpp:138-147), O(n^2) from spins."""
    s = spins(words, n)
    return int(sum(int(np.dot(s[:n - k], s[k:])) ** 2 for k in range(1, n)))


def merit_factor(n: int, e: int) -> float:
    """merit_factor (sequence.cpp:149-153)."""
    if e == 0:
        raise ZeroDivisionError("merit factor of zero energy")
    return n * n / (2.0 * e)


def random_words(n: int, count: int, rng: np.random.Generator) -> np.ndarray:
    """Bernoulli(1/2) packed sequences with zeroed padding, shape (count, W)."""
    w = rng.integers(0, 2**64, size=(count, nwords(n)), dtype=np.uint64)
    w[:, -1] &= np.uint64(tail_mask(n))
    return w
