"""Scaling sweep (BASELINE.json config 5): L_1 for n = 32..48 (m = n and m = 4n) and L_3 for
n = 16..26, reporting Gray steps/s and column updates/s against the integer roofline.

Configurations whose full search fits the time budget run through lnorm_compute; larger ones
are timed on a fixed seeded sample of prefixes through the same kernels (lnorm_prefix_maxima:
2^s-strategy units exactly like the full search's), labelled "sampled".

python tools/sweep.py [--budget-s 20] [--out profiles/r01/sweep.jsonl]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402  (the roofline floor model)
import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import synth


def roofline(steps_per_s, variant, d, c, s, d_walked, pr, packed=0, nsm=148, mhz=1965.0):
    """Fraction of the kernel family's binding-pipe floor (bench.alu_floor):
    floor instructions per strategy x strategies/s over lanes/clk/SM x SMs x f_max."""
    per, pipe, lanes = bench.alu_floor(variant, d, c, s, d_walked, pr or None, packed)
    if per is None:
        return None, None
    return per * steps_per_s / (lanes * nsm * mhz * 1e6), pipe


def run(n, m, d, seed, budget_s):
    import torch
    M = synth.random_matrix(n, m, seed)
    plan = L.plan(M, d=d)
    r = plan["rows"]
    updates_per_step = plan["cols"] * (2 if d >= 3 else 1)
    est_rate = 5e11 if d == 1 else 4e11                      # strategies/s, rough, to size the run
    full = 2 * plan["steps"] / est_rate <= budget_s      # warm-up + timed run
    if full:
        L.compute(M, d=d)                      # warm-up: lazy kernel loading, plans, tables
        t0 = time.perf_counter()
        v, _ = L.compute(M, d=d)
        wall = time.perf_counter() - t0
        st = L.last_stats()
        steps, secs = st["steps"], st["walk_ms"] / 1e3
        kind, variant = "full", st["variant"]
    else:
        base = 2 if d == 1 else d
        # a seeded sample of 2^21 prefixes (enough to fill every resident warp many
        # times) with the full search's split: each walks the planned suffix of s digits
        nfixed = n - plan["suffix_digits"]
        per = float(base) ** (n - nfixed)
        count = 1 << 21
        rng = np.random.default_rng(seed + 17)
        P = np.zeros((count, nfixed), dtype=np.int8)
        P[:, 1:] = rng.integers(0, base, size=(count, nfixed - 1), dtype=np.int8)
        if base == 2:   # aligned lane groups of 4 (the byte kernel's units, walk_u8_impl.cuh)
            P[:, :nfixed - 2] = P[::4, :nfixed - 2].repeat(4, axis=0)
            j = np.arange(count) % 4
            P[:, nfixed - 2], P[:, nfixed - 1] = j >> 1, j & 1
        L.prefix_maxima(M, P[:4096], d=d)                 # warm-up
        L.prefix_maxima(M, P, d=d)
        secs = L.last_stats()["walk_ms"] / 1e3            # the walk launch (CUDA events), as for "full"
        steps = count * per
        wall, v = secs, None
        kind, variant = f"sampled ({count} prefixes of {nfixed} rows)", L.last_stats()["variant"]
    rate = steps / secs
    cu = rate * updates_per_step
    st = L.last_stats()
    frac, pipe = roofline(rate, variant, d, plan["cols"], plan["suffix_digits"], st["d"] if d > 1 else 2,
                          st["paired_rows"], st.get("packed_units", 0))
    return {"config": f"L_{d} {n}x{m}", "n": n, "m": m, "d": d, "seed": seed, "kind": kind, "value": v,
            "kernel_variant": L.VARIANTS.get(variant, variant), "strategies": plan["steps"],
            "steps_per_s": rate, "column_updates_per_s": cu,
            "roofline_frac": frac, "roofline_pipe": pipe, "lanes_per_unit": plan["lanes_per_unit"],
            "projected_full_search_s": plan["steps"] / rate, "measured_s": secs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget-s", type=float, default=20.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--wide-only", action="store_true", help="only the m = 4n L_1 rows")
    ap.add_argument("--l3-only", action="store_true", help="only the L_3 rows (config 5b)")
    a = ap.parse_args()
    rows = []
    for n in ([] if a.l3_only else range(32, 49, 2)):
        for m in ((4 * n,) if a.wide_only else (n, 4 * n)):
            rows.append(run(n, m, 1, 100 + n, a.budget_s))
            print(json.dumps(rows[-1]), flush=True)
    for n in ([] if a.wide_only else range(16, 27, 2)):
        rows.append(run(n, n, 3, 200 + n, a.budget_s))
        print(json.dumps(rows[-1]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
