"""Run one search twice (warm-up + profiled) for ncu captures of the walk kernel.

python tools/profile_walk.py --n 38 --m 42 [--d 1] [--marg]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=38)
ap.add_argument("--m", type=int, default=42)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--marg", action="store_true")
ap.add_argument("--seed", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
M = synth.random_matrix(a.n, a.m, a.seed)
for _ in range(a.reps):
    v, arg = L.compute(M, d=a.d, with_marginals=a.marg)
print(v, L.last_stats())
