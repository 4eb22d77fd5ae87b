"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/lnorm_oracle.c) is checked against what the paper and the
mathematics fix -- worked examples printed in PAPER.md, closed forms,
independent brute-force formulations (tests/brute.py), invariances and the
norm chain -- never against itself or the CUDA path.
"""
import json
import os
from itertools import permutations

import numpy as np
import pytest

import brute
import oracle
from paper_2503_21596_b200 import synth

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rnd(n, m, seed, lo=-9, hi=9):
    return synth.random_matrix(n, m, seed, lo, hi)


# --------------------------------------------------------------- paper pins --

def test_paper_incremental_example_values():
    g = gold("paper_incremental_example.json")
    M = np.array(g["matrix"])
    for row in g["strategy_values"]:
        assert oracle.value(M, row["a"]) == row["value"]
    a0 = np.array(g["strategy_values"][0]["a"])
    assert list(a0 @ M) == g["strategy_values"][0]["m"]


def test_spec_l1_example_and_lexmin_argmax():
    g = gold("spec_l1_example.json")
    M = np.array(g["matrix"])
    v, arg = oracle.l1(M)
    assert v == g["L1"] == brute.l1_bilinear(g["matrix"])
    assert list(arg) == g["L1_lexmin_argmax"]
    assert list(arg @ M) == g["L1_argmax_m"]
    # unrestricted enumeration (all 2^n) finds the same lexmin optimum: it has a_0 = +1
    v2, arg2 = oracle.l1(M, fix_first=False)
    assert v2 == v and list(arg2) == list(arg)


def test_paper_preprocessing_example_invariance():
    g = gold("paper_preprocessing_example.json")
    A, B = np.array(g["original"]), np.array(g["reduced"])
    assert oracle.l1(A)[0] == oracle.l1(B)[0] == brute.l1_bilinear(g["reduced"])
    for d in (2, 3):
        assert oracle.ld(A, d)[0] == oracle.ld(B, d)[0]


def test_spec_ld_row_merge():
    g = gold("spec_ld_row_merge.json")
    assert oracle.ld(np.array(g["original"]), 2)[0] == oracle.ld(np.array(g["reduced"]), 2)[0]
    assert oracle.ld(np.array(g["original"]), 2)[0] == brute.ld_dual(g["original"], 2)


def test_bell_textbook_bounds():
    g = gold("bell_cg_forms.json")
    assert oracle.marg(np.array(g["CH_x4"]))[0] == g["CH_local_bound"]
    assert oracle.marg(np.array(g["I3322_x4"]))[0] == g["I3322_local_bound"]
    assert oracle.l1(np.array(g["CHSH"]))[0] == g["CHSH_L1"]
    # CHSH with d = 2: each row its own message reaches sum |M| = 4 (d >= n)
    assert oracle.ld(np.array(g["CHSH"]), 2)[0] == 4


# ------------------------------------------------------------- closed forms --

@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_identity(n):
    I = np.eye(n, dtype=np.int32)
    assert oracle.l1(I)[0] == n
    for d in (2, 3, 4):
        assert oracle.ld(I, d)[0] == n


@pytest.mark.parametrize("n,m", [(1, 1), (2, 3), (4, 4), (5, 2), (6, 7)])
def test_all_ones(n, m):
    J = np.ones((n, m), dtype=np.int32)
    assert oracle.l1(J)[0] == n * m
    for d in (2, 3):
        assert oracle.ld(J, d)[0] == n * m


@pytest.mark.parametrize("seed", range(6))
def test_rank_one(seed):
    g = synth.SplitMix64(1000 + seed)
    n, m = 2 + seed % 4, 1 + (seed * 3) % 5
    u = np.array([g.randint(-5, 5) for _ in range(n)])
    v = np.array([g.randint(-5, 5) for _ in range(m)])
    M = np.outer(u, v).astype(np.int32)
    expect = int(np.abs(u).sum() * np.abs(v).sum())
    assert oracle.l1(M)[0] == expect
    for d in (2, 3):
        assert oracle.ld(M, d)[0] == expect


def test_degenerate_shapes():
    row = np.array([[3, -4, 0, 7]])
    col = row.T.copy()
    assert oracle.l1(row)[0] == 14 and oracle.l1(col)[0] == 14
    assert oracle.ld(row, 2)[0] == 14 and oracle.ld(row, 3)[0] == 14
    assert oracle.ld(col, 2)[0] == 14   # one column, d=2: positives and negatives in separate messages
    assert oracle.ld(col, 2)[0] == brute.ld_dual(col.tolist(), 2)
    Z = np.zeros((4, 5), dtype=np.int32)
    assert oracle.l1(Z)[0] == 0 and oracle.marg(Z)[0] == 0 and oracle.ld(Z, 3)[0] == 0
    assert oracle.marg(np.array([[-5]]))[0] == -5
    assert oracle.marg(np.array([[-5, 1], [0, 0]]))[0] == -4


# ------------------------------------------------- brute-force second opinions --

@pytest.mark.parametrize("seed", range(40))
def test_l1_vs_bilinear(seed):
    n, m = 1 + seed % 4, 1 + (seed // 4) % 4
    M = rnd(n, m, 5000 + seed)
    assert oracle.l1(M)[0] == brute.l1_bilinear(M.tolist())
    assert oracle.l1(M, fix_first=False)[0] == oracle.l1(M)[0]


@pytest.mark.parametrize("seed", range(40))
def test_marg_vs_bilinear(seed):
    n, m = 1 + seed % 4, 1 + (seed // 4) % 4
    M = rnd(n, m, 6000 + seed)
    assert oracle.marg(M)[0] == brute.marg_bilinear(M.tolist())


@pytest.mark.parametrize("seed", range(24))
def test_ld_vs_eq5_and_dual(seed):
    d = 2 + seed % 2
    n, m = 1 + seed % 3, 1 + (seed // 3) % 2
    M = rnd(n, m, 7000 + seed)
    v = oracle.ld(M, d)[0]
    assert v == brute.ld_dual(M.tolist(), d)
    assert v == brute.ld_eq5(M.tolist(), d)
    assert oracle.ld(M, d, fix_first=False)[0] == v


@pytest.mark.parametrize("seed", range(12))
def test_ld_dual_larger(seed):
    d = 2 + seed % 3
    M = rnd(4 + seed % 3, 2, 7500 + seed)
    assert oracle.ld(M, d)[0] == brute.ld_dual(M.tolist(), d)


# ------------------------------------------------------------ argmax rules --

@pytest.mark.parametrize("seed", range(30))
def test_argmax_attains_and_is_lexmin(seed):
    n, m = 2 + seed % 4, 2 + seed % 3
    M = rnd(n, m, 8000 + seed, -2, 2)   # small range -> many ties
    from itertools import product
    v, arg = oracle.l1(M)
    assert oracle.value(M, arg) == v and arg[0] == 1
    # lexmin over all strategies with +1 before -1, row 0 first
    allopt = [s for s in product((1, -1), repeat=n) if oracle.value(M, s) == v]
    key = lambda s: tuple(0 if x == 1 else 1 for x in s)
    assert tuple(arg) == min(allopt, key=key)
    vm, am = oracle.marg(M)
    assert am[0] == 1 and oracle.value(M, am, marg=True) == vm
    for d in (2, 3):
        vd, ad = oracle.ld(M, d)
        assert oracle.value(M, ad, d=d) == vd
        allopt = [s for s in product(range(d), repeat=n) if oracle.value(M, s, d=d) == vd]
        assert tuple(ad) == min(allopt)
        # lexmin over ALL labellings is a restricted-growth string (first-occurrence order)
        seen = -1
        for lab in ad:
            assert lab <= seen + 1
            seen = max(seen, lab)


# ------------------------------------------------------------- invariances --

@pytest.mark.parametrize("seed", range(10))
def test_l1_invariances(seed):
    M = rnd(4, 5, 9000 + seed)
    v = oracle.l1(M)[0]
    assert oracle.l1(M.T.copy())[0] == v                       # transpose
    assert oracle.l1(synth.scramble(M, seed))[0] == v          # row/col perms + sign flips


@pytest.mark.parametrize("seed", range(10))
def test_ld_invariances(seed):
    M = rnd(5, 4, 9100 + seed)
    for d in (2, 3):
        v = oracle.ld(M, d)[0]
        assert oracle.ld(synth.scramble(M, seed, row_flips=False), d)[0] == v


def test_ld_row_flip_is_not_a_symmetry():
    # DESIGN.md reading R8: row sign flips do not preserve L_d (d >= 2)
    M = np.array([[-1, -1], [-1, -1], [-1, 1]])
    F = M.copy(); F[0] *= -1
    assert oracle.ld(M, 2)[0] == 6 == brute.ld_dual(M.tolist(), 2)
    assert oracle.ld(F, 2)[0] == 4 == brute.ld_dual(F.tolist(), 2)


@pytest.mark.parametrize("seed", range(10))
def test_marg_invariances(seed):
    M = rnd(4, 5, 9200 + seed)
    v = oracle.marg(M)[0]
    assert oracle.marg(M.T.copy())[0] == v                     # bilinear form is symmetric in the parties
    assert oracle.marg(synth.scramble(M, seed, keep_first=True))[0] == v


# --------------------------------------------------------------- norm chain --

@pytest.mark.parametrize("seed", range(20))
def test_norm_chain(seed):
    n, m = 2 + seed % 5, 1 + seed % 4
    M = rnd(n, m, 9300 + seed)
    total = int(np.abs(M.astype(np.int64)).sum())
    l1 = oracle.l1(M)[0]
    lds = [oracle.ld(M, d)[0] for d in range(2, n + 2)]
    assert l1 <= lds[0]
    assert all(a <= b for a, b in zip(lds, lds[1:]))
    assert lds[n - 2] == total and lds[-1] == total             # d >= n: each row its own message
    assert oracle.marg(M)[0] <= l1


def test_marg_zero_first_line_is_l1():
    # first row and column all zero -> L_1 of the remainder
    for seed in range(8):
        inner = rnd(3, 4, 9400 + seed)
        M = np.zeros((4, 5), dtype=np.int32); M[1:, 1:] = inner
        assert oracle.marg(M)[0] == oracle.l1(inner)[0]


def test_marg_marginals_only_closed_form():
    M = np.array([[3, -2, 5], [4, 0, 0], [-7, 0, 0]])
    assert oracle.marg(M)[0] == 3 + 4 + 7 + 2 + 5 == 21


# ------------------------------------------------------------ direct sums --

def test_direct_sum_additivity():
    A, B = rnd(3, 3, 9500), rnd(3, 4, 9501)
    S = synth.direct_sum([A, B])
    assert oracle.l1(S)[0] == oracle.l1(A)[0] + oracle.l1(B)[0]
    for d in (2, 3):
        assert oracle.ld(S, d)[0] == oracle.ld(A, d)[0] + oracle.ld(B, d)[0]


def test_planted_marg_identity_small():
    M, c, subs = synth.planted_marg(corner=2, blocks_seeds=(1, 2), block=3, scramble_seed=3)
    assert oracle.marg(M)[0] == c + sum(oracle.marg(S)[0] for S in subs)


# --------------------------------------------------- prefix max / samples --

@pytest.mark.parametrize("d", [1, 2, 3])
def test_prefix_max_partitions_the_search(d):
    from itertools import product
    M = rnd(5, 4, 9600 + d)
    full = oracle.l1(M)[0] if d == 1 else oracle.ld(M, d)[0]
    base = 2 if d == 1 else d
    best = max(oracle.prefix_max(M, (0,) + p, d)[0] for p in product(range(base), repeat=2))
    assert best == full
    s = (0, 1, 1, 0, 1) if d == 1 else (0, 1, 0, 1, 1)
    expect = oracle.value(M, [1 - 2 * x for x in s]) if d == 1 else oracle.value(M, s, d=d)
    assert oracle.prefix_max(M, s, d)[0] == expect


def test_sample_full_range_equals_norm():
    M = rnd(6, 5, 9700)
    assert oracle.sample(M, 0, 2 ** 5) == oracle.l1(M)[0]
    assert oracle.sample(M, 0, 3 ** 5, d=3) == oracle.ld(M, 3)[0]
    assert oracle.sample(M, 0, 2 ** 5, with_marginals=True) == oracle.marg(M)[0]


@pytest.mark.parametrize("threads", [1, 2, 3, 7])
def test_thread_count_independence(threads):
    M = rnd(9, 6, 9800, -2, 2)
    assert oracle.l1(M, threads=threads)[0] == oracle.l1(M, threads=1)[0]
    assert list(oracle.l1(M, threads=threads)[1]) == list(oracle.l1(M, threads=1)[1])
    assert list(oracle.ld(M, 3, threads=threads)[1]) == list(oracle.ld(M, 3, threads=1)[1])


@pytest.mark.parametrize("d,marg,n,m", [(1, False, 6, 4), (1, True, 6, 4), (2, False, 6, 3), (3, False, 5, 3),
                                        (4, False, 5, 2)])
def test_prefix_max_brute_force_pin(d, marg, n, m):
    """oracle.prefix_max with 1 < nfixed < n against an independent brute force (tests/brute.py:
    lexicographic itertools enumeration of the completions, bilinear / Eq. (5) values): the
    maximum over the completions of the fixed rows AND its lexicographically smallest maximiser.
    A prefix that is ignored, mis-ordered or read with the wrong digit convention fails here: the
    cases include prefixes whose constrained maximum is strictly below the norm."""
    base = 2 if d == 1 else d
    below = 0
    for seed in range(6):
        M = rnd(n, m, 9900 + 10 * seed + d + 5 * marg, -4, 4)
        full = oracle.norm(M, d=d, with_marginals=marg)[0]
        g = synth.SplitMix64(991 + seed)
        for nfixed in range(2, n):
            fixed = [0] + [g.next() % base for _ in range(nfixed - 1)]
            v, arg = oracle.prefix_max(M, fixed, d=d, with_marginals=marg)
            bv, barg = brute.prefix_max_brute(M.tolist(), fixed, d=d, marg=marg)
            assert v == bv, (seed, fixed)
            assert list(arg) == barg, (seed, fixed, list(arg), barg)
            assert v <= full
            below += v < full
    assert below > 0
