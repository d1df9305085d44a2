"""Instructions executed and stall samples per CUDA source line of an ncu
capture (built with -lineinfo, captured with --import-source on).

python tools/ncu_lines.py capture.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, recs, fname = None, [], "?"
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] == "File Name":
        fname = r[-1].split("/")[-1]
        continue
    if not hdr or len(r) != len(hdr) or not r[0].isdigit():
        continue
    ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    try:
        recs.append((int(r[ii] or 0), int(r[si] or 0), fname, int(r[0]), r[1].strip()[:100]))
    except ValueError:
        pass
ti = sum(x[0] for x in recs) or 1
ts = sum(x[1] for x in recs) or 1
print(f"total inst {ti}, samples {ts}")
for i, s, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * i / ti:6.2f}% inst {100 * s / ts:6.2f}% smp  {f}:{ln}  {src}")
