"""GPU: batched search -- many same-shape matrices in one walk launch."""
import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu


def batch_of(b, n, m, seed, lo=-6, hi=6):
    return np.stack([synth.random_matrix(n, m, seed + i, lo, hi) for i in range(b)])


@pytest.mark.parametrize("d,marg", [(1, False), (1, True), (2, False)])
@pytest.mark.parametrize("b,n,m", [(1, 12, 14), (37, 11, 13), (200, 9, 9), (64, 16, 10)])
def test_batch_matches_single_and_oracle(lib, d, marg, b, n, m):
    Ms = batch_of(b, n, m, 80_000 + 1000 * d + 100 * marg + n)
    vals, args = lib.compute_batch(Ms, d=d, with_marginals=marg)
    if b > 1:
        assert lib.last_stats()["variant"] in (5, 7)     # one batched launch of the byte or paired walk
    for i in range(b):
        v1, a1 = lib.compute(Ms[i], d=d, with_marginals=marg)
        assert vals[i] == v1 and list(args[i]) == list(a1)
        if i % 10 == 0:
            assert vals[i] == oracle.norm(Ms[i], d=d, with_marginals=marg)[0]
            assert oracle.value(Ms[i], args[i], d=d, marg=marg) == vals[i]


@pytest.mark.parametrize("d,marg,b,n,m,variant", [
    (1, False, 37, 16, 16, 7), (1, True, 33, 14, 16, 7), (2, False, 40, 14, 12, 7), (1, False, 9, 15, 29, 7),
    (3, False, 29, 12, 12, 8), (3, False, 17, 13, 20, 8), (4, False, 11, 10, 10, 8), (3, False, 6, 14, 23, 8),
])
def test_batch_byte_kernels_vs_oracle(lib, d, marg, b, n, m, variant):
    """The batched byte walks (one launch, tables restaged per matrix, per-matrix keys): every
    matrix's value and canonical argmax equal the oracle's; ragged batch sizes and columns."""
    Ms = batch_of(b, n, m, 83_000 + 977 * d + 31 * marg + n + m, -10, 10)
    vals, args = lib.compute_batch(Ms, d=d, with_marginals=marg)
    st = lib.last_stats()
    assert st["variant"] == variant and st["launches"] == 7
    for i in range(b):
        v, a = oracle.norm(Ms[i], d=d, with_marginals=marg)
        assert vals[i] == v and list(args[i]) == list(a), i


def test_batch_worst_case_guard(lib):
    """The batched plan is made for the element-wise worst case of the batch's guards: one matrix
    with wider column sums moves the whole batch to a family that is exact for it too."""
    Ms = batch_of(24, 14, 14, 84_000, -10, 10)
    Ms[7] = Ms[7] * 3
    vals, args = lib.compute_batch(Ms)
    for i in range(24):
        v, a = oracle.l1(Ms[i])
        assert vals[i] == v and list(args[i]) == list(a), i
    L3 = batch_of(12, 11, 12, 84_500, -10, 10)
    L3[5] = L3[5] * 3
    vals, args = lib.compute_batch(L3, d=3)
    for i in range(12):
        v, a = oracle.ld(L3[i], 3)
        assert vals[i] == v and list(args[i]) == list(a), i


def test_batch_fallbacks(lib):
    Ms = batch_of(5, 9, 10, 81_000)
    Ms[2] = Ms[2] * 400                                   # beyond the paired guard: per-matrix path
    vals, args = lib.compute_batch(Ms)
    for i in range(5):
        assert vals[i] == oracle.l1(Ms[i])[0]
    L3 = batch_of(4, 8, 7, 82_000)
    vals, args = lib.compute_batch(L3, d=3)
    for i in range(4):
        v, a = oracle.ld(L3[i], 3)
        assert vals[i] == v and list(args[i]) == list(a)
