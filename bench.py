#!/usr/bin/env python
"""Benchmark: exact L_1 of a synthetic 42x42 integer matrix (BASELINE.json configs[1]).

One "step" = one complete search through the C ABI (validate, orient, plan,
Gray walk over all 2^41 strategies, reduce, all-reduce for N > 1, argmax
recovery).  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

value  : Gray-code steps (strategies) per second of the whole job, matrix resident in HBM
e2e    : the same metric through lnorm_compute / lnorm_compute_rank with a pinned host matrix
         (H2D of M and D2H of value+argmax inside every timed step)
roofline: ALU-pipe roofline of the walk kernel: the kernel family's binding-pipe
         instruction floor per strategy x strategies / walk time, against 64 lane-instr/clk/SM x SMs x f_max
cpu_baseline: the naive oracle (oracle/) on the box's host cores, bounded sample (rank 0, N = 1)
--impl reference: the oracle as the reference arm (host cores, bounded sample per step)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, m, d, marg, seed, description)
    "l1_42x42": (42, 42, 1, False, 2, "L_1 of a synthetic 42x42 integer matrix, entries uniform in [-10,10], SplitMix64 seed 2 (Brierley et al. size)"),
    "l1_20x20": (20, 20, 1, False, 1, "L_1 of a random 20x20 integer matrix, entries in [-10,10], seed 1"),
    "marg_40x40": (40, 40, 1, True, 3, "L_marg of a 40x40 marginal-augmented correlator matrix, entries in [-10,10], seed 3"),
    "l2_24x24": (24, 24, 2, False, 4, "L_2 of a random 24x24 witness matrix, entries in [-10,10], seed 4"),
    "l3_24x24": (24, 24, 3, False, 4, "L_3 of a random 24x24 witness matrix, entries in [-10,10], seed 4"),
    # config-5 sweep points used for profiles (not the headline)
    "l3_26x26": (26, 26, 3, False, 226, "L_3 of a random 26x26 matrix, entries in [-10,10], seed 226 (config 5b top)"),
    "l4_18x18": (18, 18, 4, False, 218, "L_4 of a random 18x18 matrix, entries in [-10,10], seed 218 (P:371)"),
    "l4_22x22": (22, 22, 4, False, 222, "L_4 of a random 22x22 matrix, entries in [-10,10], seed 222 (a search long enough for the kernel's own rate)"),
    "l1_36x144": (36, 144, 1, False, 136, "L_1 of a random 36x144 matrix, entries in [-10,10], seed 136 (config 5a, m = 4n)"),
    "l1_40x160": (40, 160, 1, False, 140, "L_1 of a random 40x160 matrix, entries in [-10,10], seed 140 (config 5a, m = 4n)"),
}


def conv_max_ops(d, pr):
    """ALU max instructions per walked word of the all-H kernel's subset convolution
    (walk_ldu8w_impl.cuh: w_max_tree over every subset's candidates, D - 2 levels, last step)."""
    from math import comb
    level = sum(comb(pr, k) * ((2 ** k - 1 + 1) // 2) for k in range(pr + 1))   # sum_U ceil((2^|U|-1)/2)
    return (d - 2) * level + (2 ** pr + 1) // 2


def alu_floor(variant, d, c, s, d_walked, pr=None, packed=0):
    """Binding-pipe instruction floor per strategy of the kernel family's own algorithm
    (DESIGN.md "Roofline"): (instructions per strategy, pipe, lane-instructions/clk/SM of that pipe).

    7 byte walk (L_1/L_marg/L_2): per walked word, per unit, G*c/4 VABSDIFF4 per bias set (two
      sets: the paired last row's two signs) + one VIMNMX3 per two strategies
      -> G*c/4 + 1/2 per strategy on the ALU pipe (G = 2 for L_2's two groups).
    8 byte d-ary walk (L_3/L_4), PR paired rows (lnorm_stats.paired_rows): a move recomputes the
      2^PR bias sums of the two changed groups: 2*2^PR*c/4 VABSDIFF4.  PR >= 3 is the all-H kernel
      (walk_ldu8w_impl.cuh), whose best labelling is a max-plus subset convolution: per level a
      max tree over the 2^|U| candidates of every subset U (ceil((2^|U|-1)/2) three-input maxes),
      D - 2 levels, then ceil(2^PR/2) for the last step with the running best (conv_max_ops);
      PR <= 2 is the all-E kernel: the max of the T = d^PR labellings (ceil((T-1)/2)) + 1.
      Shared by the d^PR strategies of the word, on the ALU pipe.  Packed two-unit instances
      (lnorm_stats.packed_units = 2: both units' values as u16 halves) take each max once for
      the two units: half the max instructions per strategy.
    16-bit / int32 families: issue-bound (both integer pipes), instructions per strategy."""
    if variant == 7:
        G = 2 if d == 2 else 1
        return G * c / 4.0 + 0.5, "alu", 64.0
    if variant == 8:
        if not pr:
            pr = 3 if s >= 4 else (2 if s == 3 else 1)
        T = d_walked ** pr
        maxes = conv_max_ops(d_walked, pr) if pr >= 3 else T // 2 + 1   # all-H vs all-E epilogue
        if packed == 2:
            maxes = maxes / 2.0                                              # u16x2 maxima serve two units
        per_word = 2 * (2 ** pr) * c / 4.0 + maxes
        return per_word / T, "alu", 64.0
    if variant in (3, 5):
        return float(c), "issue", 128.0
    if variant == 6:
        return 4.0 * c / d_walked, "issue", 128.0
    if variant == 4:
        return 2.0 * c, "issue", 128.0
    if variant == 0:
        return 2.0 * c, "issue", 128.0
    if variant == 1:
        return 4.0 * c, "issue", 128.0
    return None, None, None

def metric_name(n, m, d, marg):
    norm = "L_marg" if marg else ("L_1" if d == 1 else f"L_{d}")
    return f"Gray-code steps/s (strategies evaluated per second), exact {norm} of the {n}x{m} matrix"

SMI_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thr = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].lower().startswith("active")})
        pw = [float(s[3]) for s in self.samples if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "power_w_max": max(pw) if pw else None}


def cpu_baseline(M, d, marg, target_s=12.0):
    """The oracle as it stands, on all host cores, on a bounded sample of the same workload."""
    import oracle
    n = M.shape[0]
    total = (2 if d == 1 else d) ** (n - 1)
    cores = oracle.max_threads()
    cnt = min(total, 1 << 16)
    t0 = time.perf_counter()
    oracle.sample(M, 0, cnt, d=d, with_marginals=marg)
    dt = time.perf_counter() - t0
    cnt2 = int(min(total, max(cnt, cnt * target_s / max(dt, 1e-6))))
    t0 = time.perf_counter()
    oracle.sample(M, 0, cnt2, d=d, with_marginals=marg)
    dt2 = time.perf_counter() - t0
    return {"value": cnt2 / dt2, "unit": "steps/s", "cores": cores, "kind": "oracle",
            "sample": f"first {cnt2} of {total} row-0-fixed strategies of the same matrix, "
                      f"from-scratch int64 evaluation, {dt2:.1f} s"}


VARIANT_NAMES = {0: "bin_int32", 1: "ld_int32", 2: "generic", 3: "bin_packed16", 4: "ld_packed16", 5: "bin_pair16",
                 6: "ld_pair16", 7: "bin_u8", 8: "ld_u8"}
ALU_FLOOR_NOTE = {
    7: "per strategy: G*c/4 VABSDIFF4 (four |.|-accumulates each) + 1/2 VIMNMX3, ALU pipe (c columns, G = 1; L_2: 2)",
    8: ("per walked word: 2*2^PR*c/4 VABSDIFF4 + the subset convolution's three-input maxes (PR >= 3; all-E: "
        "ceil((d^PR-1)/2) + 1) for d^PR strategies, ALU pipe; packed two-unit instances: half the maxes"),
}


def load_walk_profile(config):
    """ncu numbers of the walk kernel for this config (profiles/r02/walk_profiles.json, captured with
    `ncu --set full` on this bench's own launch; tools/ncu_bench.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "walk_profiles.json")) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def flush_l2(buf):
    buf.add_(1)   # 256 MiB write > 126 MB L2


def load_peak_clock():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        return 1965.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="l1_42x42", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n, m, d, marg, seed, desc = CONFIGS[args.config]
    from paper_2503_21596_b200 import synth
    M = synth.random_matrix(n, m, seed)
    total_steps = float((2 if d == 1 else d) ** (n - 1)) if d <= 2 else None

    if args.impl == "reference":
        if rank != 0:
            return
        import oracle
        # one step = a bounded sample of the same workload on the host cores
        base = 2 if d == 1 else d
        total = base ** (n - 1)
        cores = oracle.max_threads()
        probe = min(total, 1 << 15)
        t0 = time.perf_counter(); oracle.sample(M, 0, probe, d=d, with_marginals=marg); dt = time.perf_counter() - t0
        per_step = int(min(total, max(probe, probe * 8.0 / max(dt, 1e-6))))
        for _ in range(args.warmup):
            oracle.sample(M, 0, min(per_step, probe), d=d, with_marginals=marg)
        times = []
        for i in range(args.steps):
            lo = (i * per_step) % max(1, total - per_step)
            t0 = time.perf_counter(); oracle.sample(M, lo, lo + per_step, d=d, with_marginals=marg)
            times.append(time.perf_counter() - t0)
        T = sum(times)
        val = per_step * args.steps / T
        line = {"metric": metric_name(n, m, d, marg), "impl": "reference",
                "value": val, "unit": "steps/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "config": {"workload": desc, "n": n, "m": m, "d": d, "with_marginals": marg,
                           "sample_per_step": per_step},
                "cpu_baseline": {"value": val, "unit": "steps/s", "cores": cores, "kind": "oracle",
                                 "sample": f"{per_step} strategies per step of {total}"},
                "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2503_21596_b200 as L
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # launched by torchrun (also with --nproc-per-node 1): one rank per GPU, torch's own NCCL
    # communicator is handed to the library (caller-owned comm, lnorm_compute_rank), which
    # all-reduces the 8-byte key (+ error flag) on our stream
    distributed = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    dist = None
    comm = None
    if distributed:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        t0 = torch.ones(1, device=dev)
        dist.all_reduce(t0)
        comm = L.torch_nccl_comm(device=dev)
    stream = torch.cuda.Stream(device=dev)

    Md = torch.from_numpy(M).to(dev)
    pinned = torch.from_numpy(M).pin_memory()
    Mh = pinned.numpy()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)

    def run_device():
        if distributed:
            return L.compute_rank_device(Md, comm, rank, world, d=d, with_marginals=marg, stream=stream)
        return L.compute_device(Md, d=d, with_marginals=marg, stream=stream)

    def run_host():
        if distributed:
            return L.compute_rank(Mh, comm, rank, world, d=d, with_marginals=marg, stream=stream)
        return L.compute(Mh, d=d, with_marginals=marg)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            res = run_device()
        barrier()

        stats_walk = []
        times = []
        launches = 0
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                flush_l2(flush)
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                res = run_device()
                e1.record(stream)
                barrier()
                times.append(e0.elapsed_time(e1))
                st = L.last_stats()
                stats_walk.append(st["walk_ms"])
                launches += st["launches"]
            # e2e: host buffers through the public API, H2D + D2H inside the timed region
            e2e_times = []
            for _ in range(args.steps):
                flush_l2(flush)
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                res_h = run_host()
                e1.record(stream)
                barrier()
                e2e_times.append(e0.elapsed_time(e1))
    st = L.last_stats()
    value, argmax = res
    assert res_h[0] == value and list(res_h[1]) == list(argmax), "host and device paths disagree"

    mine = torch.tensor([sum(times), sum(e2e_times), sum(stats_walk), float(st["steps"])], dtype=torch.float64, device=dev)
    if dist is not None:
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = torch.stack(allr).cpu().tolist()
    else:
        per_rank = [mine.cpu().tolist()]
    T = max(r[0] for r in per_rank)
    TE = max(r[1] for r in per_rank)
    TW = per_rank[0][2]
    if total_steps is None:
        total_steps = sum(r[3] for r in per_rank)
    ms_per_step = T / args.steps
    val = total_steps / (ms_per_step / 1e3)
    e2e = total_steps / (TE / args.steps / 1e3)

    if rank == 0:
        c = clk.summary()
        cols = st["cols"]
        col_updates = total_steps * (cols if st["d"] <= 2 else 2 * cols)
        walk_ms = TW / args.steps
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_mhz = load_peak_clock()
        variant = st["variant"]
        per_strat, pipe, lanes = alu_floor(variant, d, cols, st["suffix_digits"], st["d"] if d > 1 else 2,
                                           st.get("paired_rows"), st.get("packed_units", 0))
        dtype = {7: "u8x4", 8: "u8x4", 3: "int16x2", 4: "int16x2", 5: "int16x2", 6: "int16x2"}.get(variant, "int32")
        rank_steps = per_rank[0][3]
        roof = {"bound": "alu", "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None}
        if per_strat is not None:
            floor_instr = rank_steps * per_strat                         # binding-pipe lane-instructions per launch
            achieved = floor_instr / (walk_ms / 1e3) / 1e12
            peak = lanes * nsm * peak_mhz * 1e6 / 1e12
            roof.update({
                "achieved": achieved, "peak": peak,
                "unit": f"T lane-instr/s on the {'ALU pipe' if pipe == 'alu' else 'issue slots (ALU + FMA-heavy integer pipes)'}",
                "frac": achieved / peak,
                "frac_at_measured_clock": (achieved / (peak * c["sm_mhz"] / peak_mhz)) if c.get("sm_mhz") else None,
                "kernel": f"walk variant {variant} ({VARIANT_NAMES.get(variant, '?')}), 1 launch per search per GPU",
                "walk_ms_per_launch": walk_ms,
                "floor_instr_per_strategy": per_strat,
                "floor_model": ALU_FLOOR_NOTE.get(variant, ""),
                "peak_basis": (f"{lanes:.0f} lane-instr/clk/SM ({'ALU pipe: VABSDIFF4 measured 64/clk/SM, profiles/r01/peaks_u8.jsonl' if pipe == 'alu' else 'issue limit, 4 SMSPs x 32 lanes'})"
                               f" x {nsm} SMs x {peak_mhz:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"),
            })
        prof = load_walk_profile(args.config)
        if prof:
            roof["traffic"] = prof.get("dram_bytes_per_launch")
            roof["ncu"] = {k: prof.get(k) for k in ("alu_pipe_pct", "issue_active_pct", "fma_pipe_pct",
                                                      "smem_bank_conflicts", "dram_bytes_per_launch", "source")}
        line = {
            "metric": metric_name(n, m, d, marg),
            "value": val, "unit": "steps/s", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic",
            "config": {"workload": desc, "name": args.config, "n": n, "m": m, "d": d, "with_marginals": marg,
                       "strategies_per_step": total_steps,
                       "parallelism": (f"units split over {world} GPU rank(s) (Algorithm 1) + 1 ncclAllReduce(max) through "
                                       f"torch's NCCL communicator" if distributed else "1 GPU, no collective"),
                       "l2": "256 MiB buffer written between timed steps (flush); matrix 7 KB"},
            "result": {"value": value, "argmax": [int(x) for x in argmax]},
            "wall_s_per_search": ms_per_step / 1e3,
            "column_updates_per_s": col_updates / (ms_per_step / 1e3),
            "e2e": {"value": e2e, "unit": "steps/s", "h2d_bytes_per_step": int(M.nbytes),
                    "d2h_bytes_per_step": 8 + n, "ms_per_step": TE / args.steps},
            "gpu_launches": int(launches),
            "per_rank": [{"rank": i, "ms_per_step": r[0] / args.steps, "walk_ms": r[2] / args.steps,
                          "e2e_ms_per_step": r[1] / args.steps, "strategies": r[3]} for i, r in enumerate(per_rank)],
            "roofline": roof,
            "clocks": c,
            "stats": st,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(M, d, marg)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
