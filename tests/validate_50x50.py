"""At-scale validation of the coarse-key byte walk (test infrastructure: uses the oracle).

Full 50x50 L_1 (2^49 strategies; seed 150 plans 2^36 units, reduced in key groups of 32)
through the byte kernel and through the independent strategy-paired 16-bit kernel: same value
and canonical argmax, and the argmax attains the value (oracle, from scratch).

python tests/validate_50x50.py [--out profiles/r01/validate_50x50.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--n", type=int, default=50)
ap.add_argument("--seed", type=int, default=150)
a = ap.parse_args()
M = synth.random_matrix(a.n, a.n, a.seed)
out = {"n": a.n, "seed": a.seed, "plan": L.plan(M)}
for fam in ("auto", "pair16"):
    os.environ["LNORM_KERNEL"] = fam
    t0 = time.perf_counter()
    v, arg = L.compute(M)
    st = L.last_stats()
    out[fam] = {"value": v, "argmax": [int(x) for x in arg], "wall_s": time.perf_counter() - t0,
                "walk_ms": st["walk_ms"], "variant": L.VARIANTS[st["variant"]], "k": st["prefix_digits"],
                "strategies_per_s": st["steps"] / (st["walk_ms"] / 1e3)}
    print(json.dumps({fam: {k: v_ for k, v_ in out[fam].items() if k != "argmax"}}), flush=True)
out["same_value_and_argmax"] = out["auto"]["value"] == out["pair16"]["value"] and out["auto"]["argmax"] == out["pair16"]["argmax"]
out["argmax_attains"] = oracle.value(M, out["auto"]["argmax"]) == out["auto"]["value"]
print(json.dumps({"same_value_and_argmax": out["same_value_and_argmax"], "argmax_attains": out["argmax_attains"]}))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
