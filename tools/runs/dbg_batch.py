import sys, numpy as np
sys.path.insert(0, '.')
import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import synth
def batch_of(b, n, m, seed, lo=-6, hi=6):
    return np.stack([synth.random_matrix(n, m, seed + i, lo, hi) for i in range(b)])
for (d, b, n, m) in [(3, 6, 14, 23), (3, 6, 14, 20), (3, 6, 13, 23), (3, 12, 14, 23), (3, 6, 12, 23)]:
    Ms = batch_of(b, n, m, 83_000 + 977 * d + n + m, -10, 10)
    try:
        v, a = L.compute_batch(Ms, d=d)
        print("ok", d, b, n, m, L.last_stats())
    except Exception as e:
        print("ERR", d, b, n, m, e)
