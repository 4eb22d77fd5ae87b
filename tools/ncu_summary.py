"""Summarise an ncu --set full capture of a walk kernel: pipes, issue, stalls, DRAM
traffic and the dynamic instruction mix (SASS opcodes), as JSON.

python tools/ncu_summary.py gpurun_out/walk.ncu-rep > profiles/r01/walk_summary.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]
out = {k: d.get(k) for k in keys}
st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v or 0)
      for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
out["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hdr = srows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
for r in srows[2:]:
    s = r[ix["Source"]].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    mix[op] += int(r[ix["Instructions Executed"]] or 0)
tot = sum(mix.values())
out["instruction_mix_pct"] = {op: round(100.0 * n / tot, 2) for op, n in mix.most_common(10)}
out["warp_instructions_executed"] = tot
print(json.dumps(out, indent=1))
