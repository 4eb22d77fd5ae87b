"""The roofline floor model bench.py reports against, pinned by
counting the instructions of each kernel family's algorithm by hand -- CPU only."""
import itertools

import pytest

import bench


def brute_conv_maxes(d, pr):
    """Three-input max instructions of the subset convolution, counted from its definition:
    every intermediate level reduces the 2^|U| candidates of each subset U (ceil((2^|U|-1)/2)),
    d - 2 such levels, then the last step reduces 2^pr candidates plus the running best."""
    level = 0
    for U in range(1 << pr):
        cands = 1 << bin(U).count("1")
        level += (cands - 1 + 1) // 2
    return (d - 2) * level + ((1 << pr) + 1 - 1 + 1) // 2


@pytest.mark.parametrize("d,pr", [(3, 3), (3, 4), (3, 5), (4, 3), (4, 4)])
def test_conv_max_ops_matches_subset_count(d, pr):
    assert bench.conv_max_ops(d, pr) == brute_conv_maxes(d, pr)


def test_byte_binary_floor():
    # 42 columns: 42/4 VABSDIFF4 per strategy + one VIMNMX3 per two strategies (not the padded 11 words)
    assert bench.alu_floor(7, 1, 42, 17, 2)[0] == pytest.approx(42 / 4 + 0.5)
    # L_2: two groups, two bias sets
    assert bench.alu_floor(7, 2, 24, 4, 2)[0] == pytest.approx(2 * 24 / 4 + 0.5)


def test_byte_dary_floor_and_packed_halving():
    # L_3, five paired rows, 24 columns: 2 * 32 * 6 VABSDIFF4 + 137 maxes for 3^5 strategies
    per, pipe, lanes = bench.alu_floor(8, 3, 24, 9, 3, 5)
    assert pipe == "alu" and lanes == 64.0
    assert per == pytest.approx((2 * 32 * 6 + 137) / 243)
    # packed two-unit instance: the u16x2 maxima serve two units -> half the maxes per strategy
    assert bench.alu_floor(8, 3, 24, 9, 3, 5, 2)[0] == pytest.approx((2 * 32 * 6 + 137 / 2) / 243)
    # L_4, four paired rows, 22 columns (6 words of 4 columns; the floor counts c / 4 = 5.5)
    assert bench.alu_floor(8, 4, 22, 9, 4, 4, 2)[0] == pytest.approx((2 * 16 * 5.5 + 88 / 2) / 256)


def test_every_labelling_is_counted_once():
    # the convolution's candidates (sum over U of 2^|U| at each level) equal the labellings it covers:
    # d = 3: 3^pr partitions (T0, T1, T2) of the paired rows
    for pr in range(1, 6):
        pairs = sum(1 << bin(U).count("1") for U in range(1 << pr))
        assert pairs == 3 ** pr
        assert sum(1 for _ in itertools.product(range(3), repeat=pr)) == 3 ** pr
