"""Per-call latency of small searches (SURVEY 8(f) f3 / VERDICT r1 item 7): wall time of one
lnorm_compute call against its GPU-event time (first H2D .. last D2H) and the walk kernel.

python tools/latency_probe.py [--calls 300]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_21596_b200 as L  # noqa: E402
from paper_2503_21596_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=300)
a = ap.parse_args()
for (n, m, d, marg, seed) in [(20, 20, 1, False, 1), (24, 24, 2, False, 4), (16, 16, 3, False, 216), (12, 12, 1, False, 5),
                              (18, 18, 4, False, 218)]:
    M = synth.random_matrix(n, m, seed)
    for _ in range(20):
        L.compute(M, d=d, with_marginals=marg)
    wall, gpu, walk = [], [], []
    for _ in range(a.calls):
        t0 = time.perf_counter()
        L.compute(M, d=d, with_marginals=marg)
        wall.append((time.perf_counter() - t0) * 1e3)
        st = L.last_stats()
        gpu.append(st["total_ms"])
        walk.append(st["walk_ms"])
    print(json.dumps({"shape": [n, m], "d": d, "calls": a.calls, "wall_ms_median": statistics.median(wall),
                      "gpu_events_ms_median": statistics.median(gpu), "walk_ms_median": statistics.median(walk),
                      "launches": st["launches"], "variant": st["variant"]}), flush=True)
