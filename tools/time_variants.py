"""Time experiment builds (paper_2503_21596_b200/_exp/liblnorm_*.so) on one search shape.

python tools/time_variants.py [--n 38 --m 42 --d 1 --marg --reps 3]
Each build runs in its own process (LNORM_LIB); prints one JSON line per build.
"""
import argparse
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=38)
ap.add_argument("--m", type=int, default=42)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--marg", action="store_true")
ap.add_argument("--seed", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--child", default=None)
a = ap.parse_args()

if a.child:
    sys.path.insert(0, ROOT)
    import paper_2503_21596_b200 as L
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(a.n, a.m, a.seed)
    ts = []
    for _ in range(a.reps + 1):
        v, arg = L.compute(M, d=a.d, with_marginals=a.marg)
        ts.append(L.last_stats()["walk_ms"])
    st = L.last_stats()
    print(json.dumps({"build": a.child, "value": int(v), "walk_ms_min": min(ts[1:]), "walk_ms": ts[1:],
                      "variant": st["variant"], "k": st["prefix_digits"], "s": st["suffix_digits"],
                      "grid": st["grid_blocks"]}), flush=True)
    sys.exit(0)

builds = [("product", os.path.join(ROOT, "paper_2503_21596_b200", "liblnorm.so"))]
builds += [(os.path.basename(p)[len("liblnorm_"):-3], p)
           for p in sorted(glob.glob(os.path.join(ROOT, "paper_2503_21596_b200", "_exp", "liblnorm_*.so")))]
for name, so in builds:
    env = dict(os.environ, LNORM_LIB=so)
    cmd = [sys.executable, __file__, "--child", name, "--n", str(a.n), "--m", str(a.m), "--d", str(a.d),
           "--seed", str(a.seed), "--reps", str(a.reps)] + (["--marg"] if a.marg else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or json.dumps({"build": name, "error": r.stderr[-400:]}), flush=True)
