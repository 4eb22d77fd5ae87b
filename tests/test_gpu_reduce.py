"""GPU: the paper's norm-preserving reductions (App. A/B) + map-back.

The value must equal the oracle's norm of the ORIGINAL matrix; the expanded argmax must
attain it (R11: it need not be the lexicographically smallest optimum)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def check_reduced(L, M, d=1, marg=False):
    M = np.ascontiguousarray(M, dtype=np.int32)
    v, arg, shape = L.compute_reduced(M, d=d, with_marginals=marg)
    ov, _ = oracle.norm(M, d=d, with_marginals=marg)
    assert v == ov, (M.tolist(), d, marg, v, ov)
    assert oracle.value(M, arg, d=d, marg=marg) == v
    assert v == L.compute(M, d=d, with_marginals=marg)[0]
    return shape


def test_paper_preprocessing_example(lib):
    g = json.load(open(os.path.join(GOLD, "paper_preprocessing_example.json")))
    A = np.array(g["original"], dtype=np.int32)
    assert check_reduced(lib, A) == (2, 4)              # 4x4 -> 2x4
    assert check_reduced(lib, A, d=2)[0] == 2           # rows merge with c = +2 (rule A3)
    check_reduced(lib, A, d=3)


def test_spec_ld_row_merge(lib):
    g = json.load(open(os.path.join(GOLD, "spec_ld_row_merge.json")))
    assert check_reduced(lib, np.array(g["original"]), d=2) == (2, 2)


def planted(n, m, seed, marg=False):
    g = synth.SplitMix64(seed)
    base = synth.random_matrix(n, m, seed, -5, 5)
    rows = [base[i] for i in range(n)]
    s = 1 if marg else 0
    for _ in range(3):                                  # proportional rows (both signs)
        src = rows[s + g.next() % (n - s)]
        c = [2, -1, 3, -2][g.next() % 4]
        rows.append(c * src)
    rows.append(np.zeros(m, dtype=np.int32))            # a zero row
    M = np.array(rows, dtype=np.int32)
    cols = [M[:, j] for j in range(m)]
    for _ in range(2):                                  # proportional columns
        src = cols[s + g.next() % (m - s)]
        cols.append([-1, 2][g.next() % 2] * src)
    cols.append(np.zeros(M.shape[0], dtype=np.int32))   # a zero column
    cols.append(np.abs(cols[s]))                        # sign-uniform columns (L_d rule)
    cols.append(-np.abs(cols[s + 1]))
    M = np.stack(cols, axis=1).astype(np.int32)
    # shuffle rows/cols >= s so merged lines are not adjacent
    rp = np.concatenate([np.arange(s), s + synth.SplitMix64(seed + 1).permutation(M.shape[0] - s)])
    cp = np.concatenate([np.arange(s), s + synth.SplitMix64(seed + 2).permutation(M.shape[1] - s)])
    return M[rp][:, cp].copy()


@pytest.mark.parametrize("d,marg", [(1, False), (1, True), (2, False), (3, False)])
def test_planted_reductions(lib, d, marg):
    for seed in range(6):
        M = planted(5 + seed % 3, 6, 900 + seed, marg)
        shape = check_reduced(lib, M, d=d, marg=marg)
        assert shape[0] < M.shape[0] and shape[1] < M.shape[1]


def test_marg_zero_first_line_becomes_l1(lib):
    for seed in range(4):
        inner = synth.random_matrix(6, 7, 950 + seed)
        M = np.zeros((7, 8), dtype=np.int32)
        M[1:, 1:] = inner
        assert check_reduced(lib, M, marg=True) == (6, 7)


def test_random_matrices_unchanged_value(lib):
    for seed in range(10):
        M = synth.random_matrix(8 + seed % 4, 9, 980 + seed)
        for d, marg in [(1, False), (1, True), (2, False), (3, False)]:
            check_reduced(lib, M, d=d, marg=marg)


def test_everything_reduced_away(lib):
    Z = np.zeros((5, 6), dtype=np.int32)
    for d, marg in [(1, False), (1, True), (3, False)]:
        v, arg, shape = lib.compute_reduced(Z, d=d, with_marginals=marg)
        assert v == 0 and oracle.value(Z, arg, d=d, marg=marg) == 0
