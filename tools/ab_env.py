"""A/B timing of one search under several environment settings (each in its own process).

python tools/ab_env.py --n 24 --m 24 --d 3 --seed 4 --env "" --env "LNORM_LDU8W=0" --env "LNORM_LDU8W_PR=3"
Prints one JSON line per setting: value, min/all walk_ms, kernel variant, split.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--m", type=int, default=24)
ap.add_argument("--d", type=int, default=3)
ap.add_argument("--marg", action="store_true")
ap.add_argument("--seed", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--env", action="append", default=[])
ap.add_argument("--child", action="store_true")
a = ap.parse_args()

if a.child:
    sys.path.insert(0, ROOT)
    import paper_2503_21596_b200 as L
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(a.n, a.m, a.seed)
    ts, tt = [], []
    for _ in range(a.reps + 1):
        v, arg = L.compute(M, d=a.d, with_marginals=a.marg)
        st = L.last_stats()
        ts.append(st["walk_ms"])
        tt.append(st["total_ms"])
    print(json.dumps({"value": int(v), "walk_ms_min": min(ts[1:]), "walk_ms": ts[1:], "total_ms_min": min(tt[1:]),
                      "variant": st["variant"], "k": st["prefix_digits"], "s": st["suffix_digits"],
                      "grid": st["grid_blocks"], "argmax": [int(x) for x in arg]}), flush=True)
    sys.exit(0)

for e in a.env or [""]:
    env = dict(os.environ)
    for kv in e.split():
        k, v = kv.split("=", 1)
        env[k] = v
    cmd = [sys.executable, __file__, "--child", "--n", str(a.n), "--m", str(a.m), "--d", str(a.d),
           "--seed", str(a.seed), "--reps", str(a.reps)] + (["--marg"] if a.marg else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout.strip().splitlines()
    rec = json.loads(out[-1]) if out else {"error": r.stderr[-500:]}
    rec.update({"env": e, "shape": [a.n, a.m], "d": a.d, "marg": a.marg})
    print(json.dumps(rec), flush=True)
