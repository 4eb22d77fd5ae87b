"""Fold `ncu --set full` captures of bench.py's own walk launch into profiles/r02/walk_profiles.json
(read by bench.py for roofline.traffic and the ncu cross-check of roofline.frac).

On the GPU box (one capture per config, the first walk launch of the bench's warm-up):
    ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8)_kernel" -c 1 \
        -o gpurun_out/ncu_r2_<config> python bench.py --config <config> --steps 1 --warmup 0 --no-cpu-baseline
Here:
    python tools/ncu_bench.py <config> gpurun_out/ncu_r2_<config>.ncu-rep [...pairs]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_BENCH_OUT") or os.path.join(ROOT, "profiles", "r02", "walk_profiles.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TIME_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def raw_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def num(d, k):
    u, v = d.get(k, ("", ""))
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1)
    except ValueError:
        return None


def summarise(rep):
    d = raw_metrics(rep)
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    return {
        "kernel": d.get("Kernel Name", ("", ""))[1],
        "duration_ms": num(d, "gpu__time_duration.sum") * TIME_MS.get(d.get("gpu__time_duration.sum", ("",))[0], 1.0),
        "alu_pipe_pct": num(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num(d, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "note_dram": "includes write-back of the bench's L2-flush buffer evicted during the launch",
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "registers": num(d, "launch__registers_per_thread"),
        "grid": num(d, "launch__grid_size"),
        "smem_bank_conflicts": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "local_spill_requests": num(d, "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum"),
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "sm_clock_hz": num(d, "sm__cycles_elapsed.avg.per_second"),
        "source": os.path.basename(rep),
    }


if __name__ == "__main__":
    args = sys.argv[1:]
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for cfg, rep in zip(args[::2], args[1::2]):
        db[cfg] = summarise(rep)
        print(cfg, json.dumps(db[cfg]))
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
