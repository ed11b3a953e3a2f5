"""splitmix64 stream, dispatch permutations and the synthetic content law.

Host-side mirror of the reference's determinism contract
(gpuiosim/simcore.py:64-122): the same splitmix64 output stream, the same
rejection-sampled bounded draw, Fisher-Yates shuffle and child-stream
derivation, so a shuffled dispatch order computed here is the order the
reference would use for the same seed (gpuiosim/simulation.py:28,208-210).

File content is the 64-bit word law W(f, i) = mix64(page_tag(f, i >> 9) ^ i)
over 8-byte word index i, i.e. the reference's per-page tag
(simcore.py:116-122) at 4 KiB granularity, stirred per word so that any
misrouted word (not only a misrouted page) is detected.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
TAG_SALT = 0xA5A5A5A5A5A5A5A5


def mix64(x: int) -> int:
    """One splitmix64 finalizer step on a Python int."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def page_tag(file_id: int, page_index: int) -> int:
    """The reference's content tag of (file, page)."""
    return mix64(((file_id << 40) ^ page_index ^ TAG_SALT) & MASK64)


class SeededRng:
    """splitmix64 generator: next_u64 / below / shuffle / fork."""

    def __init__(self, seed: int):
        self._s = seed & MASK64

    def next_u64(self) -> int:
        self._s = (self._s + GOLDEN) & MASK64
        z = self._s
        z = ((z ^ (z >> 30)) * _M1) & MASK64
        z = ((z ^ (z >> 27)) * _M2) & MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        if n <= 0:
            raise ValueError("below() needs n >= 1")
        bound = (1 << 64) - ((1 << 64) % n)
        while True:
            v = self.next_u64()
            if v < bound:
                return v % n

    def shuffle(self, seq: list) -> None:
        for hi in range(len(seq) - 1, 0, -1):
            j = self.below(hi + 1)
            seq[hi], seq[j] = seq[j], seq[hi]

    def fork(self, tag: int) -> "SeededRng":
        return SeededRng(mix64(self._s ^ mix64(tag)))


def shuffled_order(n: int, rng: SeededRng) -> list[int]:
    order = list(range(n))
    rng.shuffle(order)
    return order


# -- vectorised content law (numpy, uint64 wrap-around arithmetic) -----------

def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def words(file_id: int, first_word: int, count: int) -> np.ndarray:
    """W(f, i) for i in [first_word, first_word + count) as uint64."""
    with np.errstate(over="ignore"):
        i = np.arange(first_word, first_word + count, dtype=np.uint64)
        tag_in = (np.uint64(file_id) << np.uint64(40)) ^ (i >> np.uint64(9)) ^ np.uint64(TAG_SALT)
        return _mix64_np(_mix64_np(tag_in) ^ i)


def content(file_id: int, offset: int, nbytes: int) -> bytes:
    """Bytes [offset, offset + nbytes) of synthetic file `file_id`."""
    if nbytes <= 0:
        return b""
    w0 = offset >> 3
    w1 = (offset + nbytes + 7) >> 3
    raw = words(file_id, w0, w1 - w0).astype("<u8").tobytes()
    lo = offset - (w0 << 3)
    return raw[lo:lo + nbytes]


def checksum(buf: bytes | np.ndarray, word_base: int = 0) -> int:
    """sum_i mix64(word_i ^ (i * golden)) mod 2^64 over little-endian words
    (zero padded); the device checksum kernel computes the same value."""
    b = np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray) else buf.view(np.uint8)
    pad = (-len(b)) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, dtype=np.uint8)])
    w = b.view("<u8").astype(np.uint64)
    with np.errstate(over="ignore"):
        idx = np.arange(word_base, word_base + len(w), dtype=np.uint64)
        return int(_mix64_np(w ^ (idx * np.uint64(GOLDEN))).sum(dtype=np.uint64))
