"""GPU: SURVEY §8(f4) experiment -- the tcgen05 kind::i8 formulation of the L_1 search
(csrc/imma_l1.cu) against the ORACLE: exact L_1 over the full strategy space, the maximum over
a slice of tiles (each strategy's value from oracle.value, Eq. 1), and its input guards."""
import numpy as np
import pytest

import oracle
import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu


def tile_strategies(n, t):
    """The 512 strategies of tile t, numbered as lnorm.h documents: rows 1, 2 = the bits of
    i in [0, 4), rows 3..n-8 = bits of the Gray word g(t) = t ^ (t >> 1), rows n-7..n-1 = bits
    of l in [0, 128) (set bit = -1)."""
    g = t ^ (t >> 1)
    mid = [-1 if (g >> (x - 3)) & 1 else 1 for x in range(3, n - 7)]
    out = []
    for i in range(4):
        hi = [1, -1 if i & 1 else 1, -1 if i & 2 else 1] + mid
        for l in range(128):
            out.append(hi + [-1 if (l >> k) & 1 else 1 for k in range(7)])
    return out


@pytest.mark.parametrize("n,m", [(10, 8), (11, 13), (12, 16), (14, 42), (16, 64), (17, 37), (18, 24), (20, 20)])
def test_imma_full_space_equals_oracle(lib, n, m):
    M = synth.random_matrix(n, m, 95_000 + 64 * n + m)
    v, arg, cnt, ms = L.imma_l1(M)
    assert cnt == 2 ** (n - 1)
    assert v == oracle.l1(M)[0]
    assert oracle.value(M, arg) == v and arg[0] == 1


def test_imma_tile_slice_equals_oracle_max(lib):
    """The bench matrix (42x42, seed 2): three tiles in the middle of the 2^32-tile space."""
    M = synth.random_matrix(42, 42, 2)
    t0 = 0x9E3779B
    v, arg, cnt, ms = L.imma_l1(M, t0, 3)
    assert cnt == 3 * 512
    ref = max(oracle.value(M, np.array(s, dtype=np.int8)) for t in range(t0, t0 + 3) for s in tile_strategies(42, t))
    assert v == ref and oracle.value(M, arg) == v


def test_imma_guards(lib):
    M = synth.random_matrix(12, 12, 5)
    for bad, status in [(synth.random_matrix(9, 12, 5), "EINVAL"), (synth.random_matrix(12, 65, 5), "EINVAL"),
                        (synth.random_matrix(44, 8, 5), "ETOOLARGE")]:
        with pytest.raises(L.LNormError) as e:
            L.imma_l1(bad)
        assert e.value.name == status
    big = M.copy()
    big[-1, 0] = 128                                  # int8 operand row
    with pytest.raises(L.LNormError) as e:
        L.imma_l1(big)
    assert e.value.name == "EOVERFLOW"
    with pytest.raises(L.LNormError) as e:
        L.imma_l1(M, 1, 0x10)                          # beyond the 2^(n-10) tiles
    assert e.value.name == "EINVAL"
