"""Summarise an ncu launch list + full capture into profiles/*.json.

python tools/profile_summary.py <launches.csv> <capture.ncu-rep> <tag> [kernel-key] [attempts-per-launch]
                                [output.json] [bench flags]
"""
import collections
import csv
import io
import json
import subprocess
import sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
key = sys.argv[4] if len(sys.argv) > 4 else "k_win"
attempts = int(sys.argv[5]) if len(sys.argv) > 5 else 8 * 64 * 1024 * 1024
out_path = sys.argv[6] if len(sys.argv) > 6 else "profiles/ncu_summary.json"
bench_flags = sys.argv[7] if len(sys.argv) > 7 else ""
rows = list(csv.reader(open(launches)))
hdr = None
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        tot[name][0] += 1
        tot[name][1] += float(d["Metric Value"])
allt = sum(v for c, v in tot.values())
lsum = {"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 10 --warmup 3 --no-cpu "
                   + bench_flags,
        "unit": "ns",
        "note": f"cold-cache serialised launches; each timed bench step is one {key} launch. k_int_peak = INT32 "
                "peak microbenchmark, FillFunctor<uchar> = L2 flush between steps, linear/observe kernels = e2e leg",
        "kernels": {k: {"launches": c, "total_ns": round(v, 1), "mean_ns": round(v / c, 1), "share": round(v / allt, 4)}
                    for k, (c, v) in sorted(tot.items(), key=lambda x: -x[1][1])}}
json.dump(lsum, open(f"profiles/launches_{tag}_summary.json", "w"), indent=1)

out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, u, v = r[0], r[1], r[2]
get = lambda k: float(v[h.index(k)])
dur_us = get("gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[
    u[h.index("gpu__time_duration.sum")]]
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
_sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= _sc[u[h.index("dram__bytes_read.sum")]]
wr *= _sc[u[h.index("dram__bytes_write.sum")]]
scale = 1
insts = get("smsp__inst_executed.sum")
cap = {
    "kernel": v[h.index("Kernel Name")], "duration_us_cold": dur_us,
    "dram_bytes_read": rd * scale, "dram_bytes_write": wr * scale,
    "dram_bytes_per_launch": (rd + wr) * scale, "algorithmic_bytes_per_launch": int(0.375 * attempts),
    "attempts_per_launch": attempts,
    "alu_pipe_pct_of_active": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct_of_elapsed": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    "fma_pipe_pct_of_active": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct_of_max": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": get("launch__registers_per_thread"), "grid": get("launch__grid_size"), "block": get("launch__block_size"),
    "inst_executed_warp": insts, "inst_per_attempt": round(insts * 32 / attempts, 2),
}
summary = {"round": 2, "tag": tag, "capture": rep,
           "command": f"python bench.py --steps 10 --warmup 3 --no-cpu {bench_flags} (cfg2 64 x 1024^2); ncu --set full "
                      f"--clock-control none -k regex:{key} -s 5 -c 1",
           key: cap, "launch_list": f"profiles/launches_{tag}_summary.json"}
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps(summary, indent=1))
