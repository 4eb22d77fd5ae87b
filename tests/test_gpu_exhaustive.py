"""GPU parity, exhaustive tiny spaces: EVERY matrix with entries in {-1, 0, 1} of
shape 3x3 (3^9 = 19,683), 2x4 and 4x2 (3^8 = 6,561 each) through the batched C-ABI call
(lnorm_compute_batch: one walk launch for the whole batch) in L_1, L_marg, L_2 and L_3, compared
element by element with the CPU oracle: the value, and the argmax

  * n <= m (and every L_d): the oracle's lexicographically smallest optimum (R2);
  * n > m for L_1 / L_marg: the transposed-search rule (R6) emulated
    here from the oracle: y* = the oracle's lexicographically smallest optimum of M^T, x_i =
    sgn((M y*)_i) with sgn(0) = +1, then x_0 = +1 (L_1: negate x if x_0 = -1; L_marg: set x_0).

These spaces are dense in ties, zero rows/columns and degenerate shapes.
"""
import itertools

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

MODES = [(1, False), (1, True), (2, False), (3, False)]


def all_matrices(n, m):
    vals = np.array(list(itertools.product((-1, 0, 1), repeat=n * m)), dtype=np.int32)
    return vals.reshape(-1, n, m)


def r6_argmax(M, marg):
    """DESIGN.md R6 from the oracle: the argmax the library returns when it searches M^T."""
    T = np.ascontiguousarray(M.T)
    _, ystar = oracle.marg(T, threads=1) if marg else oracle.l1(T, threads=1)
    z = M.astype(np.int64) @ ystar.astype(np.int64)
    x = np.where(z >= 0, 1, -1).astype(np.int8)
    if marg:
        x[0] = 1
    elif x[0] == -1:
        x = -x
    return x


def expected(M, d, marg):
    v, arg = oracle.norm(M, d=d, with_marginals=marg, threads=1)
    if d == 1 and M.shape[0] > M.shape[1]:
        arg = r6_argmax(M, marg)
    return v, arg


@pytest.mark.parametrize("shape", [(3, 3), (2, 4), (4, 2)], ids=["3x3", "2x4", "4x2"])
@pytest.mark.parametrize("d,marg", MODES, ids=["L1", "marg", "L2", "L3"])
def test_every_ternary_matrix(lib, shape, d, marg):
    Ms = all_matrices(*shape)
    vals, args = lib.compute_batch(Ms, d=d, with_marginals=marg)
    assert lib.last_stats()["units"] >= len(Ms)         # one batched walk over all matrices
    bad = []
    for i, M in enumerate(Ms):
        ev, earg = expected(M, d, marg)
        if vals[i] != ev or list(args[i]) != list(earg):
            bad.append((M.tolist(), int(vals[i]), ev, list(args[i]), list(earg)))
    assert not bad, (len(bad), bad[:5])


def test_r6_rule_is_the_single_call_rule_too(lib):
    """The transposed rule also holds for single calls (not only the batched path), on random 7x3."""
    from paper_2503_21596_b200 import synth
    for seed in range(20):
        M = synth.random_matrix(7, 3, 31_000 + seed, -5, 5)
        for marg in (False, True):
            v, arg = lib.compute(M, with_marginals=marg)
            ev, earg = expected(M, 1, marg)
            assert v == ev and list(arg) == list(earg), (seed, marg)


@pytest.mark.parametrize("d,marg", MODES + [(4, False)], ids=["L1", "marg", "L2", "L3", "L4"])
def test_spec_1000_random_small_matrices(lib, d, marg):
    """SPEC.md acceptance criterion: 1000 seeded random matrices with n, m <= 6 and entries
    in [-9, 9]; grouped by shape into batched calls; value and argmax against the oracle."""
    from paper_2503_21596_b200 import synth
    g = synth.SplitMix64(423 + 10 * d + marg)
    by_shape = {}
    for i in range(1000):
        n, m = 1 + g.next() % 6, 1 + g.next() % 6
        by_shape.setdefault((n, m), []).append(synth.random_matrix(n, m, 42_300 + i, -9, 9))
    assert sum(len(v) for v in by_shape.values()) == 1000
    for (n, m), mats in sorted(by_shape.items()):
        Ms = np.stack(mats)
        vals, args = lib.compute_batch(Ms, d=d, with_marginals=marg)
        for i, M in enumerate(Ms):
            ev, earg = expected(M, d, marg)
            assert vals[i] == ev and list(args[i]) == list(earg), ((n, m), M.tolist())
