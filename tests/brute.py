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


def strategy_value_bilinear(M, x, marg=False):
    """Value of one +-1 strategy x as max over Bob's y of x^T M y (y_0 = +1 for L_marg)."""
    n, m = len(M), len(M[0])
    best = None
    ys = product((1, -1), repeat=m - 1) if marg else product((1, -1), repeat=m)
    for yr in ys:
        y = ((1,) + yr) if marg else yr
        v = sum(x[i] * M[i][j] * y[j] for i in range(n) for j in range(m))
        best = v if best is None or v > best else best
    return best


def labelling_value_eq5(M, a, d):
    """Value of one labelling a by Eq. (5) with a fixed: max over outputs b^g_y, column by column."""
    n, m = len(M), len(M[0])
    v = 0
    for g in range(d):
        for y in range(m):
            v += max(sum(M[x][y] * b for x in range(n) if a[x] == g) for b in (1, -1))
    return v


def prefix_max_brute(M, fixed, d=1, marg=False):
    """Max over completions of a fixed prefix of rows 0..len(fixed)-1, and the lexicographically
    smallest maximising completion (digits: 0/1 <-> +1/-1 for d = 1, labels for d >= 2).
    Completions are enumerated with itertools in lexicographic order; the value of each comes
    from the bilinear form (d = 1) or Eq. (5) (d >= 2), not from the oracle's column sums."""
    n = len(M)
    base = 2 if d == 1 else d
    best, arg = None, None
    for rest in product(range(base), repeat=n - len(fixed)):
        dig = tuple(fixed) + rest
        if d == 1:
            v = strategy_value_bilinear(M, [1 - 2 * t for t in dig], marg)
        else:
            v = labelling_value_eq5(M, dig, d)
        if best is None or v > best:
            best, arg = v, dig
    return best, list(arg)
