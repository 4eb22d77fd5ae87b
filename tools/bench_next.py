"""Measurements for SURVEY 8(f)'s "next" rows on one GPU (one JSON line each).

f3  batched many-small-matrix API: `lnorm_compute_batch` on B random n x n matrices against
    B separate `lnorm_compute` calls (the launch-bound regime it exists for), matrices/s.
f1  the paper's norm-preserving reductions: `lnorm_compute_reduced` on a matrix with planted
    proportional / zero lines against the plain search of the same matrix.

Every value is checked against the plain search of the same matrix before it is reported
(the oracle parity of both paths is covered by tests/test_gpu_batch.py and
tests/test_gpu_reduce.py).

python tools/bench_next.py [--out profiles/r01/next_rows.jsonl]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402


def timed(fn, reps=3):
    fn()                                   # warm-up (plans, tables, contexts)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        best = min(best, time.perf_counter() - t0)
    return best, out


def f3(batch, n, d, marg):
    Ms = np.stack([synth.random_matrix(n, n, 90_000 + i) for i in range(batch)])
    tb, (vb, ab) = timed(lambda: L.compute_batch(Ms, d=d, with_marginals=marg))
    st = L.last_stats()
    ts, single = timed(lambda: [L.compute(M, d=d, with_marginals=marg) for M in Ms[:min(batch, 256)]], reps=1)
    ts *= batch / min(batch, 256)
    assert all(int(vb[i]) == single[i][0] for i in range(len(single)))
    return {"variant": L.VARIANTS.get(st["variant"], st["variant"]), "walk_ms": st["walk_ms"], "total_ms": st["total_ms"],
            "strategies_per_s_walk": st["steps"] / (st["walk_ms"] * 1e-3) if st["walk_ms"] > 0 else None,
            "row": "f3 batched API", "mode": "L_marg" if marg else f"L_{'1' if d == 1 else d}",
            "matrices": batch, "shape": [n, n], "batched_s": tb, "per_call_s": ts,
            "matrices_per_s_batched": batch / tb, "matrices_per_s_per_call": batch / ts, "speedup": ts / tb}


def f1(n, m, d, seed):
    # planted structure: every third row is a multiple of the previous one, plus two zero
    # columns -> the reductions remove about a third of the rows (2x per removed row)
    g = synth.SplitMix64(seed)
    M = np.array(synth.random_matrix(n, m, seed), dtype=np.int64)
    for x in range(2, n, 3):
        M[x] = M[x - 1] * (1 + g.next() % 2) * (1 if g.next() & 1 else -1)
    M[:, 3] = 0
    M[:, 7] = 0
    M = M.astype(np.int32)
    tr, (vr, ar, shape) = timed(lambda: L.compute_reduced(M, d=d), reps=1)
    tp, (vp, ap) = timed(lambda: L.compute(M, d=d), reps=1)
    assert vr == vp
    return {"row": "f1 reductions", "mode": f"L_{d}", "shape": [n, m], "reduced_shape": list(shape),
            "reduced_s": tr, "plain_s": tp, "speedup": tp / tr, "value": int(vr)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch-only", action="store_true")
    a = ap.parse_args()
    rows = [f3(4096, 16, 1, False), f3(4096, 16, 1, True), f3(1024, 20, 1, False), f3(1024, 24, 1, False),
            f3(1024, 14, 2, False), f3(256, 24, 2, False), f3(256, 16, 3, False), f3(64, 18, 3, False), f3(64, 14, 4, False)]
    if not a.batch_only:
        rows += [f1(36, 40, 1, 7), f1(22, 24, 3, 8)]
    for r in rows:
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
