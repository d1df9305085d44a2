"""Per-function SASS opcode histogram: python tools/sasscount.py <binary> [filter]"""
import re, subprocess, sys, collections
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None; cnt = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m: cur = m.group(1); continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur: cnt[cur][m.group(2)] += 1
for f in sorted(cnt):
    if flt in f:
        c = cnt[f]
        print(f, sum(c.values()), " ".join(f"{k}:{v}" for k, v in c.most_common(14)))
