"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Values must be bit-exact (integer arithmetic).  The argmax must equal the
oracle's lexicographically smallest optimum where the library promises it
(n <= m for L_1/L_marg, always for L_d); otherwise (transposed search,
DESIGN.md R6) it must attain the value.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODES = [(1, False), (1, True), (2, False), (3, False), (4, False)]


def mode_id(d, marg):
    return "marg" if marg else ("L1" if d == 1 else f"L{d}")


def check(L, M, d=1, marg=False, exact_argmax=None):
    M = np.ascontiguousarray(M, dtype=np.int32)
    v, arg = L.compute(M, d=d, with_marginals=marg)
    ov, oarg = oracle.norm(M, d=d, with_marginals=marg)
    assert v == ov, (mode_id(d, marg), M.tolist(), v, ov)
    # the returned strategy attains the value (from-scratch oracle evaluation)
    assert oracle.value(M, arg, d=d, marg=marg) == v
    if exact_argmax is None:
        exact_argmax = d >= 2 or M.shape[0] <= M.shape[1]
    if exact_argmax:
        assert list(arg) == list(oarg), (mode_id(d, marg), M.tolist(), list(arg), list(oarg))
    if d == 1:
        assert arg[0] == 1
    else:
        mx = -1
        for a in arg:                      # restricted-growth form
            assert a <= mx + 1
            mx = max(mx, a)
    return v, arg


# ------------------------------------------------------------- paper pins --

def test_paper_worked_example_trace(lib):
    """values 19, 17, 17 along the first Gray steps (negation-symmetric start)."""
    g = json.load(open(os.path.join(GOLD, "paper_incremental_example.json")))
    M = np.array(g["matrix"], dtype=np.int32)
    vals, digs = lib.walk_trace(M, [0], d=1)
    assert list(vals[:3]) == [r["value"] for r in g["strategy_values"]]
    # every step is the from-scratch value of the strategy it claims, and steps are Hamming-1
    for w in range(len(vals)):
        a = [1 - 2 * x for x in digs[w]]
        assert vals[w] == oracle.value(M, a)
        if w:
            assert int(np.sum(digs[w] != digs[w - 1])) == 1
    # the strategies visited are exactly the paper's (up to the global sign a <-> -a)
    paper = [r["a"] for r in g["strategy_values"]]
    for w in range(3):
        assert [-(1 - 2 * x) for x in digs[w]] == paper[w]


@pytest.mark.parametrize("d,marg", MODES, ids=[mode_id(*m) for m in MODES])
def test_walk_trace_matches_from_scratch(lib, d, marg):
    M = synth.random_matrix(6, 5, 42 + d)
    base = 2 if d == 1 else d
    pre = [0, 1 % base]
    vals, digs = lib.walk_trace(M, pre, d=d, with_marginals=marg)
    assert len(vals) == base ** 4
    seen = set()
    for w in range(len(vals)):
        s = digs[w]
        assert list(s[:2]) == pre
        seen.add(tuple(s))
        strat = [1 - 2 * x for x in s] if d == 1 else s
        assert vals[w] == oracle.value(M, strat, d=d, marg=marg)
    assert len(seen) == len(vals)          # the Gray walk covers the suffix space exactly once


def test_paper_examples(lib):
    g = json.load(open(os.path.join(GOLD, "spec_l1_example.json")))
    v, arg = check(lib, np.array(g["matrix"]))
    assert v == g["L1"] and list(arg) == g["L1_lexmin_argmax"]
    p = json.load(open(os.path.join(GOLD, "paper_preprocessing_example.json")))
    for d in (1, 2, 3):
        assert check(lib, np.array(p["original"]), d=d)[0] == check(lib, np.array(p["reduced"]), d=d)[0]
    b = json.load(open(os.path.join(GOLD, "bell_cg_forms.json")))
    assert check(lib, np.array(b["CH_x4"]), marg=True)[0] == 0
    assert check(lib, np.array(b["I3322_x4"]), marg=True)[0] == 0
    assert check(lib, np.array(b["CHSH"]))[0] == 2


# ------------------------------------------------------------ exhaustive --

@pytest.mark.parametrize("d,marg", MODES, ids=[mode_id(*m) for m in MODES])
def test_random_sweep_small(lib, d, marg):
    for seed in range(60):
        n = 1 + seed % 9
        m = 1 + (seed * 7) % 10
        M = synth.random_matrix(n, m, 10_000 + seed + 100 * d + 1000 * marg, -3 if seed % 2 else -10, 3 if seed % 2 else 10)
        check(lib, M, d=d, marg=marg)


HOT_SHAPES = [
    (1, False, 12, 37), (1, False, 14, 64), (1, False, 13, 5), (1, False, 16, 16),
    (1, True, 11, 13), (1, True, 12, 41), (2, False, 11, 9), (2, False, 13, 30),
    (3, False, 9, 7), (3, False, 10, 32), (3, False, 8, 13), (4, False, 7, 5), (4, False, 8, 29),
    (5, False, 6, 4), (1, False, 9, 70), (2, False, 8, 100),
    (1, True, 10, 97), (1, False, 11, 190), (1, False, 12, 128),      # wide rows (config 5a m = 4n)
    (1, True, 12, 150), (1, False, 13, 133),                           # > 128 columns: lane pairs
    (3, False, 12, 40), (3, False, 13, 44), (4, False, 10, 36),        # d-ary byte walk beyond 32 columns
    (3, False, 11, 33), (3, False, 9, 48),
]


@pytest.mark.parametrize("d,marg,n,m", HOT_SHAPES)
def test_hot_kernel_shapes(lib, d, marg, n, m):
    """Shapes that run the templated hot kernels (several column tiles, ragged tails)."""
    for seed in range(3):
        M = synth.random_matrix(n, m, 20_000 + 31 * n + m + seed)
        check(lib, M, d=d, marg=marg)
        st = lib.last_stats()
        assert st["launches"] >= 4 and st["steps"] >= 1


@pytest.mark.parametrize("marg", [False, True])
def test_wide_even_word_instances(lib, marg):
    """Every even word count above 32 (136-184 columns) has its own lane-pair byte instance
    (no padding to a multiple of 8 words): each one against the oracle, incl. the ragged
    last word (c not a multiple of 4)."""
    for c in (135, 143, 151, 167, 175, 183, 136, 144):
        M = synth.random_matrix(13, c, 40_000 + c + 7 * marg)
        P = lib.plan(M, with_marginals=marg)
        assert P["variant_name"] == "bin_u8" and P["lanes_per_unit"] == 2, (c, P)
        assert P["words"] == (c + 3) // 4 + ((c + 3) // 4) % 2, (c, P)      # the even word count itself
        check(lib, M, marg=marg)


def test_ties_identity_and_ones(lib):
    for n in (1, 2, 5, 9, 12):
        for d, marg in MODES:
            check(lib, np.eye(n, dtype=np.int32), d=d, marg=marg)
            check(lib, np.ones((n, n + 1), dtype=np.int32), d=d, marg=marg)
            check(lib, np.zeros((n, 3), dtype=np.int32), d=d, marg=marg)


def test_transposed_orientation(lib):
    for seed in range(10):
        M = synth.random_matrix(9, 4, 30_000 + seed)
        v, _ = check(lib, M, exact_argmax=False)
        assert lib.last_stats()["transposed"] == 1
        assert v == lib.compute(M.T.copy())[0]
        vm, _ = check(lib, M, marg=True, exact_argmax=False)
        assert vm == lib.compute(M.T.copy(), with_marginals=True)[0]


# ----------------------------------------------------------- configs ----

def test_config1_l1_20x20_full(lib):
    """BASELINE config 1: L_1 of a random 20x20 matrix, entries in [-10, 10], seed 1."""
    M = synth.random_matrix(20, 20, 1)
    check(lib, M)


def test_config4_l2_24x24_full(lib):
    M = synth.random_matrix(24, 24, 4)
    check(lib, M, d=2)


def test_l3_l4_medium_full(lib):
    check(lib, synth.random_matrix(13, 24, 4), d=3)
    check(lib, synth.random_matrix(10, 16, 5), d=4)
    # more than 32 columns: the byte walk (the int32 d-ary walk stops at 32 columns)
    M = synth.random_matrix(14, 40, 6)
    check(lib, M, d=3)
    assert lib.last_stats()["variant"] == 8
    check(lib, synth.random_matrix(11, 44, 7), d=4)
    assert lib.last_stats()["variant"] == 8


def test_marg_medium_full(lib):
    check(lib, synth.random_matrix(20, 22, 3), marg=True)


def test_planted_42x42_l1(lib):
    """BASELINE config 2 planted twin: direct sum of three 14x14 blocks, scrambled (value known exactly)."""
    M, blocks = synth.planted_l1()
    expect = sum(oracle.l1(B)[0] for B in blocks)
    v, arg = lib.compute(M)
    assert v == expect
    assert oracle.value(M, arg) == v and arg[0] == 1


@pytest.mark.parametrize("marg", [False, True], ids=["L1_42x42", "marg_40x40"])
def test_bench_workload_families_and_metamorphic(lib, marg, monkeypatch):
    """The bench workloads in full (BASELINE configs 2 and 3, 2^41 / 2^39 strategies): the byte
    kernel and the independent strategy-paired 16-bit kernel return the same value and the same
    canonical argmax; the argmax attains the value (oracle, from scratch); L_1(M) = L_1(M^T) and
    L_marg(M) = L_marg(M^T)."""
    n = 40 if marg else 42
    M = synth.random_matrix(n, n, 3 if marg else 2)
    assert lib.plan(M, with_marginals=marg)["variant_name"] == "bin_u8"
    v, arg = lib.compute(M, with_marginals=marg)
    assert oracle.value(M, arg, marg=marg) == v
    monkeypatch.setenv("LNORM_KERNEL", "pair16")
    assert lib.plan(M, with_marginals=marg)["variant_name"] == "bin_pair16"
    v2, arg2 = lib.compute(M, with_marginals=marg)
    assert v2 == v and list(arg2) == list(arg)
    monkeypatch.setenv("LNORM_KERNEL", "auto")
    vt, _ = lib.compute(np.ascontiguousarray(M.T), with_marginals=marg)
    assert vt == v


@pytest.mark.parametrize("d,n,seed", [(3, 24, 4), (3, 26, 226), (4, 18, 218)])
def test_ld_workload_families_agree(lib, d, n, seed, monkeypatch):
    """BASELINE config 4 / 5b sizes in full: the byte d-ary walk (three rows paired) and the
    independent last-row-paired 16-bit walk agree on value and canonical (RGS) argmax; the
    argmax attains the value (oracle, from scratch)."""
    M = synth.random_matrix(n, n, seed)
    assert lib.plan(M, d=d)["variant_name"] == "ld_u8"
    v, arg = lib.compute(M, d=d)
    assert oracle.value(M, arg, d=d) == v
    monkeypatch.setenv("LNORM_KERNEL", "pair16")
    assert lib.plan(M, d=d)["variant_name"] == "ld_pair16"
    v2, arg2 = lib.compute(M, d=d)
    assert v2 == v and list(arg2) == list(arg)


@pytest.mark.parametrize("shift", [1, 3, 8])
def test_coarse_reduction_keys_exact(lib, shift, monkeypatch):
    """Splits with more than 2^31 units (50+ rows) reduce on unit >> shift and recover the
    whole winning group; forced here on small inputs (LNORM_KEY_SHIFT): same value and the
    same lexicographically smallest argmax as the oracle, including tie-heavy inputs and the
    multi-rank slices."""
    monkeypatch.setenv("LNORM_KEY_SHIFT", str(shift))
    cases = [(synth.random_matrix(14, 16, 65_000 + shift), 1, False),
             (synth.random_matrix(13, 15, 65_100 + shift), 1, True),
             (synth.random_matrix(12, 14, 65_200 + shift), 2, False),
             (np.eye(12, dtype=np.int32), 1, False), (np.ones((11, 13), dtype=np.int32), 2, False),
             (synth.random_matrix(14, 16, 65_300 + shift, -1, 1), 1, False)]
    for M, d, marg in cases:
        assert lib.plan(M, d=d, with_marginals=marg)["variant_name"] == "bin_u8"
        check(lib, M, d=d, marg=marg)
        ref = oracle.norm(M, d=d, with_marginals=marg)
        for sl in (3, 8):
            got = lib.compute_sliced(M, sl, d=d, with_marginals=marg)
            assert got[0] == ref[0] and list(got[1]) == list(ref[1])


def test_maximum_sizes(lib):
    """The ABI limits: 1024 columns (and 1024 rows, searched transposed), 63 enumerated rows
    (sampled through the hook with the byte kernel's lane groups), one past each limit rejected."""
    check(lib, synth.random_matrix(5, 1024, 66_000), d=1)
    check(lib, synth.random_matrix(5, 1024, 66_001), d=3)
    T = synth.random_matrix(1024, 5, 66_002)                      # searched as its 5 x 1024 transpose
    v, arg = lib.compute(T)
    assert v == oracle.l1(np.ascontiguousarray(T.T))[0] and oracle.value(T, arg) == v
    with pytest.raises(Exception):
        lib.compute(synth.random_matrix(5, 1025, 66_003))
    with pytest.raises(Exception):
        lib.compute(synth.random_matrix(64, 64, 66_004))
    # a full 63-row search is 2^62 strategies (and 63 x 20 would be searched transposed): the
    # hook walks the 63 rows of per-prefix sub-searches instead (no orientation)
    M = synth.random_matrix(63, 20, 66_005, -2, 2)
    P = np.zeros((8, 55), dtype=np.int8)
    g = synth.SplitMix64(66_006)
    for i in range(8):
        P[i, 1:53] = [g.next() % 2 for _ in range(52)]
        P[i, :53] = P[i - i % 4, :53]
        P[i, 53], P[i, 54] = (i % 4) >> 1, (i % 4) & 1
    got = lib.prefix_maxima(M, P)
    for i in range(8):
        assert got[i] == oracle.prefix_max(M, P[i])[0]


def test_coarse_keys_full_size_planted(lib, monkeypatch):
    """Coarse keys at the bench size: the planted 42x42 twin with groups of 256 units per key
    gives the exact value (sum of the blocks) and the same canonical argmax as exact keys."""
    M, blocks = synth.planted_l1()
    expect = sum(oracle.l1(B)[0] for B in blocks)
    v0, a0 = lib.compute(M)
    monkeypatch.setenv("LNORM_KEY_SHIFT", "8")
    v8, a8 = lib.compute(M)
    assert v0 == v8 == expect and list(a8) == list(a0) and oracle.value(M, a8) == v8


def test_planted_40x40_marg(lib):
    """BASELINE config 3 planted twin: shared-corner marginal direct sum."""
    M, c, subs = synth.planted_marg()
    expect = c + sum(oracle.marg(S)[0] for S in subs)
    v, arg = lib.compute(M, with_marginals=True)
    assert v == expect
    assert oracle.value(M, arg, marg=True) == v


@pytest.mark.parametrize("d,marg", [(1, False), (1, True), (2, False)], ids=["L1", "marg", "L2"])
def test_sampled_prefixes_ungrouped(lib, d, marg):
    """Prefixes that do not form aligned lane groups (arbitrary order and count) take the
    per-unit kernels and still match the oracle."""
    M = synth.random_matrix(30, 33, 880 + d + marg)
    g = synth.SplitMix64(881)
    P = np.zeros((7, 16), dtype=np.int8)
    for i in range(7):
        for x in range(1, 16):
            P[i, x] = g.next() % 2
    got = lib.prefix_maxima(M, P, d=d, with_marginals=marg)
    for i in range(7):
        assert got[i] == oracle.prefix_max(M, P[i], d=d, with_marginals=marg)[0]


@pytest.mark.parametrize("allh", ["1", "0"], ids=["allH", "allE"])
@pytest.mark.parametrize("d", [3, 4])
@pytest.mark.parametrize("s", [2, 3, 4, 5, 6])
def test_ldu8_paired_rows_every_suffix_length(lib, d, s, allh, monkeypatch):
    """The byte d-ary walk pairs the last 1, 2 or 3 rows depending on the suffix length
    (s = 2, 3, >= 4; L_3: the all-H kernel pairs 3 rows at s = 4 and 4 rows from s = 5,
    LNORM_LDU8W=0 keeps the all-E kernel): per-prefix maxima for every case against the oracle,
    and the value of the full search (whose planner picks its own split)."""
    monkeypatch.setenv("LNORM_LDU8W", allh)
    n, m = 11, 13
    M = synth.random_matrix(n, m, 64_000 + 10 * d + s)
    nfixed = n - s
    g = synth.SplitMix64(640 + s)
    P = np.zeros((40, nfixed), dtype=np.int8)
    for i in range(40):
        for x in range(1, nfixed):
            P[i, x] = g.next() % d
    got = lib.prefix_maxima(M, P, d=d)
    assert lib.last_stats()["variant"] == 8
    for i in range(40):
        assert got[i] == oracle.prefix_max(M, P[i], d=d)[0], (i, list(P[i]))
    check(lib, M, d=d)


@pytest.mark.parametrize("d,cap", [(3, 3), (3, 4), (3, 5), (4, 3), (4, 4)])
def test_allh_instances_every_width(lib, d, cap, monkeypatch):
    """The all-H byte d-ary walk (walk_ldu8w) at every paired-row count it compiles (L_3: 3-5,
    L_4: 3-4, capped with LNORM_LDU8W_PR) over column counts that hit both translation-unit
    halves, ragged last words, the five-row instances with kappas in shared memory (all but
    24 columns) and registers (24): per-prefix maxima of random RGS-free prefixes against the
    oracle, through the prefix hook with an 8-row suffix."""
    monkeypatch.setenv("LNORM_LDU8W_PR", str(cap))
    n = 13 if d == 3 else 11
    for c in (5, 13, 24, 27, 33, 47):
        M = synth.random_matrix(n, c, 65_000 + 100 * d + 10 * cap + c, -5, 5)
        nfixed = n - 8
        g = synth.SplitMix64(650 + c + d)
        P = np.zeros((24, nfixed), dtype=np.int8)
        for i in range(24):
            for x in range(1, nfixed):
                P[i, x] = g.next() % d
        got = lib.prefix_maxima(M, P, d=d)
        st = lib.last_stats()
        assert st["variant"] == 8 and st["paired_rows"] == cap, (c, st["paired_rows"])
        for i in range(24):
            assert got[i] == oracle.prefix_max(M, P[i], d=d)[0], (c, i, list(P[i]))


def test_bench_configs_plan_the_byte_kernel(lib):
    """The 42x42 L_1 and 40x40 L_marg bench workloads run the byte-packed kernel."""
    assert lib.plan(synth.random_matrix(42, 42, 2))["variant_name"] == "bin_u8"
    assert lib.plan(synth.random_matrix(40, 40, 3), with_marginals=True)["variant_name"] == "bin_u8"


# ------------------------------------------------------------- errors ----

def test_errors(lib):
    from paper_2503_21596_b200 import LNormError
    with pytest.raises(LNormError) as e:
        lib.compute(np.full((3, 3), 2 ** 29, dtype=np.int32))
    assert e.value.name == "EOVERFLOW"
    with pytest.raises(LNormError) as e:
        lib.compute(np.eye(3, dtype=np.int32), d=2, with_marginals=True)
    assert e.value.name == "EINVAL"
    with pytest.raises(LNormError) as e:
        lib.compute(np.ones((64, 64), dtype=np.int32))
    assert e.value.name == "ETOOLARGE"


def test_device_resident_and_rank_paths(lib):
    import torch
    M = synth.random_matrix(18, 21, 99)
    ref = lib.compute(M)
    t = torch.from_numpy(M).cuda()
    v, arg = lib.compute_device(t)
    assert v == ref[0] and list(arg) == list(ref[1])
    c = lib.Comm(None, 0, 1, torch.cuda.current_device())
    v2, arg2 = c.compute(M)
    c.close()
    assert v2 == ref[0] and list(arg2) == list(ref[1])
    v3, arg3 = lib.compute_multi(M, devices=[0])
    assert v3 == ref[0] and list(arg3) == list(ref[1])


# ------------------------------------------------------ kernel families ----

@pytest.mark.parametrize("family", ["int32", "packed", "pair16", "generic", "u8", "auto"])
@pytest.mark.parametrize("d,marg", MODES, ids=[mode_id(*m) for m in MODES])
def test_every_kernel_family_matches_oracle(lib, family, d, marg, monkeypatch):
    """The byte-packed, paired-16, packed-16, int32 and generic kernels all reproduce the oracle bit for bit."""
    monkeypatch.setenv("LNORM_KERNEL", family)
    for seed, (n, m) in enumerate([(11, 21), (12, 8), (9, 33), (10, 16)]):
        M = synth.random_matrix(n, m, 40_000 + seed + 10 * d)
        check(lib, M, d=d, marg=marg)
    if family == "generic":
        assert lib.last_stats()["variant"] == 2


def test_large_entries_use_int32_path_exactly(lib):
    """Entries too large for the packed s16 guard: the int32 kernels run and stay exact."""
    for seed in range(3):
        M = synth.random_matrix(14, 17, 50_000 + seed, -3000, 3000)
        assert lib.plan(M)["packed_ok"] == 0
        check(lib, M)
        check(lib, M, marg=True)
        check(lib, synth.random_matrix(10, 12, 50_100 + seed, -3000, 3000), d=3)


def _with_abs_sums(col_sums, n, seed):
    """n x len(col_sums) matrix with random signs whose column |.|-sums are exactly col_sums."""
    g = synth.SplitMix64(seed)
    M = np.zeros((n, len(col_sums)), dtype=np.int64)
    for y, tot in enumerate(col_sums):
        base, extra = divmod(tot, n)
        for x in range(n):
            v = base + (1 if x < extra else 0)
            M[x, y] = v if g.next() & 1 else -v
    return M.astype(np.int32)


@pytest.mark.parametrize("S_pair", [16383, 16384])
def test_pair_guard_boundary_exact(lib, S_pair, monkeypatch):
    """sum |M| at the strategy-paired path's guard (<= 16383) and one past it: both exact."""
    monkeypatch.setenv("LNORM_KERNEL", "pair16")
    n, m = 10, 12
    cols = [S_pair // m + (1 if y < S_pair % m else 0) for y in range(m)]
    M = _with_abs_sums(cols, n, 60_000 + S_pair)
    assert int(np.abs(M.astype(np.int64)).sum()) == S_pair
    P = lib.plan(M)
    assert P["variant_name"] == ("bin_pair16" if S_pair <= 16383 else "bin_packed16")
    check(lib, M)
    # all-positive matrix: the optimum sits exactly at the bound (value = S)
    A = np.abs(M)
    v, _ = check(lib, A)
    assert v == S_pair


@pytest.mark.parametrize("par", [32767, 32768])
def test_packed_guard_boundary_exact(lib, par):
    """Per-parity column |.|-sums at the packed column-pair guard (<= 32767) and one past it."""
    n = 6                                                             # n < m: no transposition
    M = _with_abs_sums([par - 7, par - 10, 5, 7, 1, 1, 1, 1], n, 61_000 + par)   # parity sums: par, par - 1
    P = lib.plan(M)
    assert P["packed_ok"] == (1 if par <= 32767 else 0)
    check(lib, M)
    v, _ = check(lib, np.abs(M))
    assert v == int(np.abs(M.astype(np.int64)).sum())


def _u8_boundary_matrix(W, d, seed, s=7, n=9, m=12):
    """n x m matrix whose last s rows give column 0 the window |.|-sum W (column 3 too,
    all positive), every other column less, and row n-s-1 non-zero in column 0 so that a
    longer window breaks the byte guard.  The u8 kernel's window is its 5-row suffix (4
    unrolled digits + the paired last row) plus the 2 prefix rows of its lane group
    (walk_u8_impl.cuh)."""
    g = synth.SplitMix64(seed)
    M = np.array(synth.random_matrix(n, m, seed, -6, 6), dtype=np.int64)
    for y, sign in ((0, None), (3, 1)):
        base, extra = divmod(W, s)
        for i in range(s):
            v = base + (1 if i < extra else 0)
            M[n - s + i, y] = v if (sign == 1 or g.next() & 1) else -v
    M[n - s - 1, 0] = 5
    return M.astype(np.int32)


@pytest.mark.parametrize("d,marg,W", [(1, False, 127), (1, False, 128), (1, True, 127), (1, True, 128),
                                      (2, False, 255), (2, False, 256)])
def test_u8_guard_boundary_exact(lib, d, marg, W):
    """Byte-packed walk: a suffix window exactly at the byte guard (2W <= 255 for L_1/L_marg,
    W <= 255 for L_2) runs the u8 kernel and is exact; one past it falls back, also exact."""
    M = _u8_boundary_matrix(W, d, 62_000 + W + 10 * d + (5 if marg else 0))
    P = lib.plan(M, d=d, with_marginals=marg)
    fits = (W <= 127) if d == 1 else (W <= 255)
    assert (P["variant_name"] == "bin_u8") == fits, P
    if fits:
        assert P["suffix_digits"] == 5 and P["prefix_digits"] == 3
    check(lib, M, d=d, marg=marg)
    check(lib, np.abs(M), d=d, marg=marg)
    check(lib, -np.abs(M), d=d, marg=marg)


@pytest.mark.parametrize("d", [3, 4])
@pytest.mark.parametrize("W", [255, 256])
def test_ldu8_guard_boundary_exact(lib, d, W):
    """Byte-packed d-ary walk: a column |.|-sum exactly at the byte guard (255) runs the
    ld_u8 kernel and is exact (subset sums span the whole byte); 256 falls back, exact too."""
    n, m = 9, 12
    M = _with_abs_sums([W, W - 40, 7, 90, 31, 5, 60, 12, W - 1, 3, 44, 18], n, 63_000 + W + d)
    P = lib.plan(M, d=d)
    assert (P["variant_name"] == "ld_u8") == (W <= 255), P
    check(lib, M, d=d)
    check(lib, np.abs(M), d=d)
    check(lib, -np.abs(M), d=d)


# ------------------------------------------------- multi-GPU decomposition --

@pytest.mark.parametrize("d,marg", MODES, ids=[mode_id(*m) for m in MODES])
def test_sliced_ranks_bit_identical(lib, d, marg):
    """results for 1/2/3/4/8 ranks (Algorithm-1 slices, max-reduced key) are bit-identical."""
    for seed, (n, m) in enumerate([(14, 20), (12, 12), (16, 9), (10, 31)]):
        M = synth.random_matrix(n, m, 70_000 + seed + 7 * d, -4, 4)
        ref = lib.compute(M, d=d, with_marginals=marg)
        for slices in (2, 3, 4, 8):
            got = lib.compute_sliced(M, slices, d=d, with_marginals=marg)
            assert got[0] == ref[0] and list(got[1]) == list(ref[1]), (slices, seed)
        check(lib, M, d=d, marg=marg)


def test_sliced_ranks_42x42_planted(lib):
    """The 42x42 planted twin split over 8 virtual ranks: same exact value as the direct sum of blocks."""
    M, blocks = synth.planted_l1()
    expect = sum(oracle.l1(B)[0] for B in blocks)
    v, arg = lib.compute_sliced(M, 8)
    assert v == expect and oracle.value(M, arg) == v


@pytest.mark.parametrize("marg", [False, True], ids=["L1", "marg"])
@pytest.mark.parametrize("c", [33, 34, 37, 38, 41, 42, 45, 46])
def test_u8_merged_last_word(lib, c, marg):
    """Byte walk with c mod 4 in {1, 2} (a partly padded last word; with LN_U8_MERGE=1 the merged
    last-word instances of walk_u8_impl.cuh): the full search and EVERY unit's maximum (all four
    units of each lane group) equal the oracle's."""
    n = 14
    M = synth.random_matrix(n, c, 1300 + c + 50 * marg)
    check(lib, M, d=1, marg=marg)
    assert lib.last_stats()["variant"] == 7
    k = 8
    units = np.arange(1 << k, dtype=np.uint64)
    got = lib.unit_maxima(M, k, units, with_marginals=marg)
    for u, gv in zip(units.tolist(), got):
        pre = [0] + [(u >> (k - x)) & 1 for x in range(1, k + 1)]
        assert gv == oracle.prefix_max(M, pre, with_marginals=marg)[0], (u, c, marg)


def _rgs(length, d):
    """Restricted-growth labellings of the given length in lexicographic order (independent of the library)."""
    out = []

    def rec(pre, mx):
        if len(pre) == length:
            out.append(list(pre))
            return
        for a in range(min(mx + 2, d)):
            rec(pre + [a], max(mx, a))
    rec([0], 0)
    return out


@pytest.mark.parametrize("d,n", [(3, 14), (4, 12)], ids=["L3", "L4"])
@pytest.mark.parametrize("c", [4, 20, 24, 26, 32])
def test_packed_two_unit_walk_every_unit(lib, d, n, c):
    """The packed two-unit all-H walk (walk_ldu8w_impl.cuh, walk_ldu8w_pk_kernel: L_3 with five
    paired rows, L_4 with four, up to 32 columns): both units of every lane -- the low and the high
    16-bit half of every packed sum -- give the oracle's maximum for EVERY unit of the search."""
    M = synth.random_matrix(n, c, 1700 + 10 * d + c)
    k = 5
    lst = _rgs(k + 1, d)
    units = np.arange(len(lst), dtype=np.uint64)
    got = lib.unit_maxima(M, k, units, d=d)
    st = lib.last_stats()
    assert st["variant"] == 8 and st["paired_rows"] == (5 if d == 3 else 4)
    assert st["packed_units"] == 2
    for i, gv in enumerate(got):
        assert gv == oracle.prefix_max(M, lst[i], d=d)[0], (i, lst[i])


@pytest.mark.parametrize("d,n", [(3, 20), (4, 18)], ids=["L3_20x20", "L4_18x18"])
def test_packed_walk_sliced_and_checkpointed(lib, tmp_path, d, n):
    """The packed two-unit walk under Algorithm-1 slices (2/3/8 virtual ranks: slices start and end
    inside a 64-unit chunk) and under checkpoint chunks of an odd unit count: bit-identical value and
    argmax to the one-shot search, whose argmax attains the value (from-scratch oracle evaluation);
    the one-shot search itself is checked against the oracle per sampled prefix in test_gpu_fullsize."""
    M = synth.random_matrix(n, n, 4_200 + n + d)
    v, arg = lib.compute(M, d=d)
    assert lib.last_stats()["packed_units"] == 2
    assert oracle.value(M, arg, d=d) == v
    for slices in (2, 3, 8):
        got = lib.compute_sliced(M, slices, d=d)
        assert got[0] == v and list(got[1]) == list(arg), slices
    units = lib.plan(M, d=d)["units"]
    path = str(tmp_path / "ck.bin")
    chunk = units // 5 + 33
    while True:
        done, cv, carg, _ = lib.compute_checkpointed(M, path, d=d, chunk_units=chunk, max_chunks=1)
        if done:
            break
        assert cv <= v
    assert cv == v and list(carg) == list(arg)
