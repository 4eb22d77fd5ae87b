"""C-ABI library: loads, exports every declared symbol, host-side helpers (-m "not gpu").

The Gray-code helpers are the same __host__ __device__ code the kernels run
(paper_2503_21596_b200/csrc/gray.cuh); they are pinned here to the paper's
Tables 1 and 3 and to its appendix lemmas.
"""
import json
import os
import re

import numpy as np
import pytest

import paper_2503_21596_b200 as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_functions():
    txt = open(os.path.join(ROOT, "include", "lnorm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lnorm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = L.load()
    funcs = header_functions()
    assert len(funcs) >= 14
    for f in funcs:
        assert hasattr(lib, f), f
    assert sorted(funcs) == sorted(L.SYMBOLS)
    assert L.load().lnorm_version() >> 16 == 2


def test_status_strings():
    for s in range(9):
        assert L.status_string(s)


def gray_word(d, h, j):
    return [L.gray_digit(d, i, j) for i in range(h)]


def test_table1_brgc():
    g = json.load(open(os.path.join(GOLD, "gray_tables.json")))
    rows = g["brgc4_rows_i3_to_i0"]
    for j in range(16):
        for i in range(4):
            assert L.gray_digit(2, i, j) == rows[3 - i][j]
    # bottom row of Table 1: digit and direction of the change (word 0 compares with word 15)
    for j in range(1, 16):
        dig, frm, to = L.gray_change(2, j)
        mark = g["brgc4_change"][j]
        assert dig == int(mark[0]) and (to == 1) == (mark[1] == "+") and frm == 1 - to


def test_table3_trgc():
    g = json.load(open(os.path.join(GOLD, "gray_tables.json")))
    rows = g["trgc3_rows_i2_to_i0"]
    for j in range(27):
        for i in range(3):
            assert L.gray_digit(3, i, j) == rows[2 - i][j]
    for j in range(1, 27):
        assert L.gray_change(3, j)[0] == g["trgc3_change_from_word1"][j - 1]


def reflect_construct(d, h):
    """Recursive reflected construction (Table 4, d-ary analogue): words as digit tuples."""
    if h == 0:
        return [()]
    prev = reflect_construct(d, h - 1)
    out = []
    for a in range(d):
        seq = prev if a % 2 == 0 else prev[::-1]
        out += [w + (a,) for w in seq]   # new most-significant digit
    return out


@pytest.mark.parametrize("d,h", [(2, 1), (2, 4), (2, 9), (3, 3), (3, 6), (4, 4), (5, 3)])
def test_closed_form_equals_reflection_and_hamming(d, h):
    words = reflect_construct(d, h)
    assert len(set(words)) == d ** h
    for j, w in enumerate(words):
        assert tuple(gray_word(d, h, j)) == w
        if j:
            diff = [i for i in range(h) if w[i] != words[j - 1][i]]
            assert len(diff) == 1
            dig, frm, to = L.gray_change(d, j)
            assert diff == [dig] and frm == words[j - 1][dig] and to == w[dig] and abs(to - frm) == 1


@pytest.mark.parametrize("d,h,l", [(2, 6, 2), (2, 8, 3), (3, 5, 2), (4, 4, 1)])
def test_appendix_e_group_alignment(d, h, l):
    # for k > 0 the change digit of word g*d^(h-l)+k does not depend on g
    for k in range(1, d ** (h - l)):
        digs = {L.gray_change(d, g * d ** (h - l) + k)[0] for g in range(d ** l)}
        assert len(digs) == 1


def test_eq16_equals_eq17_and_ctz():
    for d in (2, 3, 5):
        for j in range(1, 2000):
            i16 = max(i for i in range(40) if j % d ** i == 0)
            assert L.gray_change(d, j)[0] == i16
    for j in range(1, 4096):
        assert L.gray_change(2, j)[0] == (j & -j).bit_length() - 1


def test_change_probe_count_bound():
    # expected number of probes of Eq. (9) is sum i/2^i -> 2 (<= 2 d^h total)
    for d in (2, 3, 4):
        h = 8 if d == 2 else 5
        probes = 0
        for j in range(1, d ** h):
            probes += L.gray_change(d, j)[0] + 1
        assert probes <= 2 * d ** h


def test_algorithm1_partition():
    # examples: SPEC.md:292-294 (hand trace of Algorithm 1)
    assert [L.partition(8, 3, t) for t in range(3)] == [(0, 2), (3, 5), (6, 7)]
    assert [L.partition(8, 4, t) for t in range(4)] == [(0, 1), (2, 3), (4, 5), (6, 7)]
    assert [L.partition(2, 4, t) for t in range(4)] == [(0, 0), (1, 1), (2, 1), (2, 1)]
    for C in range(1, 200):
        for T in (1, 2, 3, 7, 16, 40):
            rngs = [L.partition(C, T, t) for t in range(T)]
            covered = [j for lo, hi in rngs for j in range(lo, hi + 1)]
            assert covered == list(range(C))
            sizes = [hi - lo + 1 for lo, hi in rngs]
            assert max(sizes) - min(sizes) <= 1


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(L.LNormError) as e:
        L.compute(np.eye(3, dtype=np.int32))
    assert e.value.name == "ENODEV"


# ------------------------------------------------------------ host planner --

def rgs_count(length, d):
    """Restricted-growth strings of the given length with at most d labels (brute force)."""
    from itertools import product
    cnt = 0
    for s in product(range(d), repeat=length):
        mx, ok = -1, True
        for a in s:
            if a > mx + 1:
                ok = False
                break
            mx = max(mx, a)
        cnt += ok
    return cnt


@pytest.mark.parametrize("n,m,d,marg", [(42, 42, 1, False), (20, 20, 1, False), (40, 40, 1, True),
                                        (24, 24, 2, False), (24, 24, 3, False), (12, 9, 4, False),
                                        (30, 9, 1, False), (9, 30, 1, True), (5, 70, 1, False), (3, 3, 3, False)])
def test_plan_covers_the_search_space(n, m, d, marg):
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(n, m, 5)
    P = L.plan(M, d=d, with_marginals=marg)
    r = min(n, m) if d == 1 else n
    assert P["rows"] == r and P["transposed"] == (d == 1 and n > m)
    assert P["prefix_digits"] + P["suffix_digits"] == r - 1
    dw = P["d_walked"]
    if dw == 2:
        assert P["units"] == 2 ** P["prefix_digits"]
        assert P["steps"] == 2 ** (r - 1)                  # 2^(n-1) strategies
    else:
        assert dw == min(d, n)
        assert P["units"] == rgs_count(P["prefix_digits"] + 1, dw) if P["prefix_digits"] < 9 else P["units"] > 0
        assert P["steps"] == P["units"] * dw ** P["suffix_digits"]
        # RGS prefixes x full suffixes cover all canonical labellings: at least S(n,<=d) of them
        assert P["steps"] >= (dw ** (n - 1) + 1) / 2 if dw == 3 else True


def test_plan_packed_guard_and_fallback():
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(30, 30, 1)
    assert L.plan(M)["variant_name"] == "bin_u8"                   # suffix window fits a byte
    assert L.plan((M * 2).astype(np.int32))["variant_name"] == "bin_u8"
    assert L.plan((M * 3).astype(np.int32))["variant_name"] == "bin_pair16"    # sum |M| <= 16383, windows too wide
    mid = (M * 8).astype(np.int32)                   # sum |M| > 32767, per-parity column sums still fit
    assert L.plan(mid)["packed_ok"] == 1 and L.plan(mid)["variant_name"] == "bin_packed16"
    big = (M * 300).astype(np.int32)                 # column abs sums exceed the s16 guard
    P = L.plan(big)
    assert P["packed_ok"] == 0 and P["variant_name"] == "bin_int32"
    assert L.plan(synth.random_matrix(24, 24, 4), d=3)["variant_name"] == "ld_u8"       # column |.|-sums <= 255
    assert L.plan(synth.random_matrix(24, 24, 4) * 3, d=3)["variant_name"] == "ld_pair16"
    # 40 columns: the byte d-ary walk is not limited by the int32 walk's 32-column constant bank
    assert L.plan(synth.random_matrix(24, 40, 4), d=3)["variant_name"] == "ld_u8"
    assert L.plan(np.eye(3, dtype=np.int32))["variant_name"] == "generic"     # suffix shorter than the unroll


def test_plan_lane_pairs_for_wide_rows():
    """Beyond 128 columns the byte walk splits a unit over a lane pair; the extra window row
    shortens the suffix, and splits beyond 2^31 units use coarse reduction keys (48x192: k = 32)."""
    from paper_2503_21596_b200 import synth
    assert L.plan(synth.random_matrix(42, 168, 142))["lanes_per_unit"] == 2
    P = L.plan(synth.random_matrix(48, 192, 148))
    assert P["variant_name"] == "bin_u8" and P["lanes_per_unit"] == 2 and P["prefix_digits"] == 32
    assert L.plan(synth.random_matrix(42, 42, 2))["lanes_per_unit"] == 1


def test_plan_byte_walk_word_counts():
    """Packed words per unit of the byte instance: exact up to 16 words, multiples of 4 up to 32,
    every even count above (lane pairs: 136 columns run 34 words, not 36 or 40)."""
    from paper_2503_21596_b200 import synth
    for c, words in ((42, 11), (61, 16), (66, 20), (72, 20), (128, 32), (132, 34), (136, 34), (144, 36),
                     (152, 38), (168, 42), (176, 44), (184, 46), (192, 48)):
        P = L.plan(synth.random_matrix(14, c, 900 + c))
        assert P["variant_name"] == "bin_u8" and P["words"] == words, (c, P)
    assert L.plan(synth.random_matrix(14, 14, 3), d=3)["words"] == 0          # other families: 0


def test_plan_large_rows_use_byte_walk_and_reach_63_rows():
    """50-56 rows keep the byte walk (more than 2^31 units: coarse keys, up to 2^39 units);
    up to 63 rows plan with at most 31 suffix digits per unit."""
    from paper_2503_21596_b200 import synth
    for n in (50, 56):
        P = L.plan(synth.random_matrix(n, n, 7))
        assert P["variant_name"] == "bin_u8" and 31 < P["prefix_digits"] <= 39
    for n in (56, 60, 63):
        P = L.plan(synth.random_matrix(n, n, 7))
        assert P["suffix_digits"] <= 31 and P["steps"] == 2.0 ** (n - 1)
        assert P["prefix_digits"] <= (39 if P["variant_name"] == "bin_u8" else 31)


@pytest.mark.parametrize("hi", [10, 40])
def test_plan_invariants_over_shapes(hi):
    """Every plan covers exactly the canonical strategy space (2^(r-1) words for +-1 / L_2):
    units x 2^s = steps, s <= 31, units below the key range, byte plans only where the window
    guard holds, for every row count up to 63 and several column counts."""
    from paper_2503_21596_b200 import synth
    for n in list(range(2, 64, 3)) + [63]:
        for m in (n, 7, 64, 130, 192):
            M = synth.random_matrix(n, m, 3 * n + m + hi, -hi, hi)
            for d, marg in ((1, False), (1, True), (2, False)):
                try:
                    P = L.plan(M, d=d, with_marginals=marg)
                except L.LNormError:
                    continue                                      # ETOOLARGE / EOVERFLOW limits
                r = P["rows"]
                assert P["units"] * 2.0 ** P["suffix_digits"] == P["steps"] == 2.0 ** (r - 1)
                assert P["suffix_digits"] <= 31 and P["prefix_digits"] + P["suffix_digits"] == r - 1
                assert P["prefix_digits"] <= (39 if P["variant_name"] == "bin_u8" else 31)
                if P["variant_name"] == "bin_u8":     # the byte window holds at least the suffix rows
                    A = np.abs(np.asarray(M if not P["transposed"] else M.T, dtype=np.int64))
                    W = A[r - P["suffix_digits"]:].sum(axis=0).max()
                    assert (2 * W <= 255) if d == 1 else (W <= 255)


def test_plan_is_identical_for_every_rank_and_grows_with_world():
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(42, 42, 2)
    p1, p8 = L.plan(M, world=1), L.plan(M, world=8)
    assert p8["units"] >= p1["units"] and p8["steps"] == p1["steps"] == 2.0 ** 41


def test_plan_errors():
    with pytest.raises(L.LNormError) as e:
        L.plan(np.full((3, 3), 2 ** 29, dtype=np.int32))
    assert e.value.name == "EOVERFLOW"
    with pytest.raises(L.LNormError) as e:
        L.plan(np.ones((64, 64), dtype=np.int32))
    assert e.value.name == "ETOOLARGE"
    with pytest.raises(L.LNormError) as e:
        L.plan(np.eye(3, dtype=np.int32), d=2, with_marginals=True)
    assert e.value.name == "EINVAL"


def test_dary_block_start_matches_eq17():
    """The unrolled d-ary walks' block-start shortcut equals Eqs. (13)-(17) at word t*d."""
    import ctypes
    for d in (3, 4):
        for t in range(1, 3 ** 7):
            dig, frm, to = L.gray_change(d, t * d)
            # same quantities from the closed form of Eqs. (13)-(15)
            assert frm == L.gray_digit(d, dig, t * d - 1) and to == L.gray_digit(d, dig, t * d)
            tt, ip = t, 0
            while tt % d == 0:
                tt //= d
                ip += 1
            S = list(range(d)) + list(range(d - 1, -1, -1))
            assert (dig, frm, to) == (1 + ip, S[(tt - 1) % (2 * d)], S[tt % (2 * d)])


def test_binding_rejects_lossy_matrix_casts():
    """The binding never wraps or truncates entries into int32: non-integer dtypes and
    out-of-range integers raise before any library call."""
    from paper_2503_21596_b200 import LNormError
    with pytest.raises(TypeError):
        L.compute(np.ones((3, 3)) * 1.7)
    with pytest.raises(TypeError):
        L.compute(np.ones((3, 3), dtype=bool))
    with pytest.raises(LNormError) as e:
        L.compute(np.array([[2 ** 33 + 3, 1], [1, 1]], dtype=np.int64))
    assert e.value.name == "EOVERFLOW"
    with pytest.raises(LNormError):
        L.compute_batch(np.full((2, 2, 2), -(2 ** 31) - 1, dtype=np.int64))
    with pytest.raises(ValueError):
        L.compute(np.ones(4, dtype=np.int32))
    # int64 input within range is accepted by the binding (then needs a device on this host)
    A = L._mat(np.array([[5, -7], [2 ** 31 - 1, -(2 ** 31)]], dtype=np.int64))
    assert A.dtype == np.int32 and A[1, 0] == 2 ** 31 - 1 and A[1, 1] == -(2 ** 31)


def test_rank_entry_checks_communicator_arguments_before_the_device():
    """lnorm_compute_rank: world > 1 without a communicator, or a rank outside [0, world), is
    EINVAL (checked before any device work, so also on this GPU-less host)."""
    from paper_2503_21596_b200 import LNormError
    M = np.eye(3, dtype=np.int32)
    for rank, world in ((0, 2), (2, 2), (-1, 1), (0, 0)):
        with pytest.raises(LNormError) as e:
            L.compute_rank(M, None, rank, world)
        assert e.value.name == "EINVAL", (rank, world)
