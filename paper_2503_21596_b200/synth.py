"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds NO arithmetic of the method (no norms, no Gray codes): it
only draws integer matrices.  Both the CUDA path and the CPU oracle receive
the matrices it produces; neither imports the other.

Generator: SplitMix64(seed); entry =
lo + (u64 mod (hi - lo + 1)), filled row-major.  Default distribution:
uniform integers in [-10, 10], dense (BASELINE.json config 1).
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class SplitMix64:
    """Counter-based 64-bit generator (Steele, Lea & Flood 2014)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (modulo bias <= (hi-lo+1)/2^64)."""
        return lo + self.next() % (hi - lo + 1)

    def permutation(self, k: int) -> np.ndarray:
        """Fisher-Yates permutation of range(k)."""
        p = list(range(k))
        for i in range(k - 1, 0, -1):
            j = self.next() % (i + 1)
            p[i], p[j] = p[j], p[i]
        return np.array(p, dtype=np.int64)


def random_matrix(n: int, m: int, seed: int, lo: int = -10, hi: int = 10) -> np.ndarray:
    """Dense n x m int32 matrix, entries uniform in [lo, hi], row-major SplitMix64 draw."""
    g = SplitMix64(seed)
    out = np.empty((n, m), dtype=np.int32)
    for i in range(n):
        for j in range(m):
            out[i, j] = g.randint(lo, hi)
    return out


def direct_sum(blocks) -> np.ndarray:
    """Block-diagonal direct sum of integer matrices."""
    n = sum(b.shape[0] for b in blocks)
    m = sum(b.shape[1] for b in blocks)
    out = np.zeros((n, m), dtype=np.int32)
    r = c = 0
    for b in blocks:
        out[r:r + b.shape[0], c:c + b.shape[1]] = b
        r += b.shape[0]
        c += b.shape[1]
    return out


def scramble(M: np.ndarray, seed: int, row_flips: bool = True, keep_first: bool = False) -> np.ndarray:
    """Random row/column permutations and sign flips (seeded).

    keep_first: leave row 0 and column 0 in place and unflipped (marginal layout).
    row_flips=False: flip columns only (row sign flips are not an L_d symmetry).
    """
    g = SplitMix64(seed)
    n, m = M.shape
    s = 1 if keep_first else 0
    rp = np.concatenate([np.arange(s), s + g.permutation(n - s)])
    cp = np.concatenate([np.arange(s), s + g.permutation(m - s)])
    out = M[rp][:, cp].astype(np.int32).copy()
    for j in range(s, m):
        if g.next() & 1:
            out[:, j] = -out[:, j]
    if row_flips:
        for i in range(s, n):
            if g.next() & 1:
                out[i, :] = -out[i, :]
    return out


def planted_l1(blocks_seeds=(21, 22, 23), block: int = 14, scramble_seed: int = 24):
    """BASELINE config 2 planted twin: direct sum of random block x block matrices, scrambled.

    Returns (matrix, list of blocks); L_1(matrix) = sum of the blocks' L_1 values."""
    blocks = [random_matrix(block, block, s) for s in blocks_seeds]
    return scramble(direct_sum(blocks), scramble_seed), blocks


def planted_marg(corner: int = 3, blocks_seeds=(31, 32, 33), block: int = 13, scramble_seed: int = 34):
    """BASELINE config 3 planted twin: shared-corner marginal direct sum.

    M = [[c, r_A, r_B, ...], [c_A, A, 0, ...], [c_B, 0, B, ...], ...]; each block
    comes with its own marginal row/column.  L_marg(M) = c + sum_X L_marg([[0, r_X], [c_X, X]]).
    Returns (matrix, corner, list of (block+marginal) sub-matrices with zero corner)."""
    subs = []
    for s in blocks_seeds:
        full = random_matrix(block + 1, block + 1, s)
        full[0, 0] = 0
        subs.append(full)
    n = 1 + block * len(subs)
    M = np.zeros((n, n), dtype=np.int32)
    M[0, 0] = corner
    off = 1
    for S in subs:
        M[0, off:off + block] = S[0, 1:]
        M[off:off + block, 0] = S[1:, 0]
        M[off:off + block, off:off + block] = S[1:, 1:]
        off += block
    return scramble(M, scramble_seed, keep_first=True), corner, subs
