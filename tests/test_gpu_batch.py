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
        assert lib.last_stats()["variant"] == 5          # one batched launch of the paired walk
    for i in range(b):
        v1, a1 = lib.compute(Ms[i], d=d, with_marginals=marg)
        assert vals[i] == v1 and list(args[i]) == list(a1)
        if i % 10 == 0:
            assert vals[i] == oracle.norm(Ms[i], d=d, with_marginals=marg)[0]
            assert oracle.value(Ms[i], args[i], d=d, marg=marg) == vals[i]


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
