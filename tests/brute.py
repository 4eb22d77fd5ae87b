"""Independent brute-force second opinions for tiny matrices (pure Python loops).

These are NOT the oracle's formulas retyped: each uses a different (but
equivalent, per the paper) formulation of the same maximum, so agreement with
``oracle`` pins the oracle against a plausible mistake in its own loop.

- L_1   = max_{x in {+-1}^n, y in {+-1}^m} x^T M y     (bilinear form; |s| = max_b b*s)
- L_marg= max_{x_0 = y_0 = +1} x^T M y                 (Eq. 2 with the first column's sign forced)
- L_d   = Eq. (5): max over messages a_x and outputs b_y^a of sum_x sum_y M_xy b^{a_x}_y
- L_d   = dual form max_{b^0..b^{d-1}} sum_x max_a (M b^a)_x
"""
from itertools import product


def l1_bilinear(M):
    n, m = len(M), len(M[0])
    best = None
    for x in product((1, -1), repeat=n):
        for y in product((1, -1), repeat=m):
            v = sum(x[i] * M[i][j] * y[j] for i in range(n) for j in range(m))
            best = v if best is None or v > best else best
    return best


def marg_bilinear(M):
    n, m = len(M), len(M[0])
    best = None
    for xr in product((1, -1), repeat=n - 1):
        x = (1,) + xr
        for yr in product((1, -1), repeat=m - 1):
            y = (1,) + yr
            v = sum(x[i] * M[i][j] * y[j] for i in range(n) for j in range(m))
            best = v if best is None or v > best else best
    return best


def ld_eq5(M, d):
    """Eq. (5): joint maximum over the message map a and Bob's outputs b^a_y."""
    n, m = len(M), len(M[0])
    best = None
    for a in product(range(d), repeat=n):
        for bflat in product((1, -1), repeat=d * m):
            b = [bflat[k * m:(k + 1) * m] for k in range(d)]
            v = sum(M[x][y] * b[a[x]][y] for x in range(n) for y in range(m))
            best = v if best is None or v > best else best
    return best


def ld_dual(M, d):
    """Dual form: for fixed outputs each row picks its best message."""
    n, m = len(M), len(M[0])
    best = None
    for bflat in product((1, -1), repeat=d * m):
        b = [bflat[k * m:(k + 1) * m] for k in range(d)]
        v = 0
        for x in range(n):
            v += max(sum(M[x][y] * b[k][y] for y in range(m)) for k in range(d))
        best = v if best is None or v > best else best
    return best
