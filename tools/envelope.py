"""Entry-range envelope of the headline number: exact L_1 of a 42x42 matrix with entries uniform in
[-hi, hi] (SplitMix64 seed 2) for growing hi -- which kernel family the planner picks and how long
the search takes on one B200 (the byte walk needs every unit's column window to fit a byte, so wider
entries shorten the suffix, then fall back to the packed 16-bit walk).

python tools/envelope.py  -> one JSON line per hi
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402

for hi in (10, 15, 20, 25, 30):
    M = synth.random_matrix(42, 42, 2, -hi, hi)
    L.compute(M)                                   # warm-up
    v, _ = L.compute(M)
    st = L.last_stats()
    print(json.dumps({"entries": [-hi, hi], "value": v, "variant": L.VARIANTS[st["variant"]],
                      "prefix_digits": st["prefix_digits"], "suffix_digits": st["suffix_digits"],
                      "walk_ms": st["walk_ms"], "total_ms": st["total_ms"],
                      "strategies_per_s": st["steps"] / (st["walk_ms"] * 1e-3)}), flush=True)
