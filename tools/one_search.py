"""One search through lnorm_compute (for ncu captures of a given shape):
python tools/one_search.py N M [--d D] [--marg] [--seed S] [--lo LO --hi HI] [--reps R]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int)
ap.add_argument("m", type=int)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--marg", action="store_true")
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--lo", type=int, default=-10)
ap.add_argument("--hi", type=int, default=10)
ap.add_argument("--reps", type=int, default=1, help="searches; the minimum walk time is printed")
a = ap.parse_args()
M = synth.random_matrix(a.n, a.m, a.seed, a.lo, a.hi)
ts = []
for _ in range(a.reps):
    v, arg = L.compute(M, d=a.d, with_marginals=a.marg)
    st = L.last_stats()
    ts.append(st["walk_ms"])
print(v, L.VARIANTS[st["variant"]], st["prefix_digits"], st["suffix_digits"], f"{min(ts):.3f} ms")
