"""SURVEY §8(f4) measurement: the tcgen05 kind::i8 formulation (lnorm_imma_l1) against the byte walk
(lnorm_compute) on the bench matrix (42x42 L_1, seed 2), strategies per second on one B200.

python tools/bench_imma.py [--tiles-log2 21] [--reps 3] [--no-walk]   -> one JSON line
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tiles-log2", type=int, default=21)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-walk", action="store_true")
a = ap.parse_args()

M = synth.random_matrix(42, 42, 2)
tiles = 1 << a.tiles_log2
t0 = 0x5555555 & ((1 << 32) - tiles)          # a slice in the middle of the 2^32-tile space
L.imma_l1(M, t0, 1024)                          # warm-up (module load, attribute set)
runs = []
for _ in range(a.reps):
    v, arg, cnt, ms = L.imma_l1(M, t0, tiles)
    runs.append(ms)
ms = min(runs)
out = {"what": "f4 tcgen05 kind::i8 formulation vs the byte walk, 42x42 L_1 seed 2",
       "imma": {"tiles": tiles, "strategies": cnt, "kernel_ms": runs, "strategies_per_s": cnt / (ms * 1e-3),
                "slice_max": v}}
if not a.no_walk:
    v2, _ = L.compute(M)
    st = L.last_stats()
    out["byte_walk"] = {"value": v2, "walk_ms": st["walk_ms"], "strategies": st["steps"],
                        "strategies_per_s": st["steps"] / (st["walk_ms"] * 1e-3), "variant": st["variant"]}
    out["ratio_walk_over_imma"] = out["byte_walk"]["strategies_per_s"] / out["imma"]["strategies_per_s"]
    out["imma_projected_full_search_s"] = 2 ** 41 / out["imma"]["strategies_per_s"]
print(json.dumps(out), flush=True)
