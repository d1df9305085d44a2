"""Side-by-side key metrics of ncu --set full captures (one kernel each).

python tools/ncu_compare.py a.ncu-rep b.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
STALL = "smsp__average_warp_latency_issue_stalled_"


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


reps = [load(p) for p in sys.argv[1:]]
for k in KEYS:
    print(f"{k[:60]:60s}", *[f"{(d.get(k) or '')[:40]:>28s}" for d, _ in reps])
stall_keys = sorted({k for d, _ in reps for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")})
for k in stall_keys:
    vals = [d.get(k, "") for d, _ in reps]
    try:
        if max(float(v or 0) for v in vals) < 0.05:
            continue
    except ValueError:
        pass
    print(f"{k.replace('smsp__average_warps_issue_stalled_', 'stall ')[:60]:60s}", *[f"{v:>28s}" for v in vals])
