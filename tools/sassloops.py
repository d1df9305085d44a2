"""Loop bodies (backward branches) of one kernel with opcode histograms:
python tools/sassloops.py <binary> <function-filter> [min_len]"""
import re, subprocess, sys, collections
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
flt, minlen = sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40
funcs, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); funcs[cur] = []; continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur: funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
ALU = ("LOP3", "SHF", "IADD3", "LEA", "ISETP", "SEL", "PRMT", "FLO", "POPC", "BMSK", "SGXT", "IABS", "IMNMX", "VIADD", "PLOP3", "LOP", "MOV")
for f, ins in funcs.items():
    if flt not in f: continue
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, txt) in enumerate(ins):
        m = re.search(r"\bBRA\S*\s+(?:\S+\s+)?`?\(?\.?L?_?x?_?(0x[0-9a-f]+)", txt)
        if not m: continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr: continue
        body = ins[addr[tgt]:i + 1]
        if len(body) < minlen: continue
        c = collections.Counter()
        for _, t in body:
            op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
            c[op] += 1
        alu = sum(v for k, v in c.items() if k.split(".")[0] in ALU)
        fma = sum(v for k, v in c.items() if k.startswith("IMAD") or k.startswith("IADD.") or k.startswith("FFMA"))
        print(f"{f[:90]}\n  loop {tgt:#x}-{a:#x}: {len(body)} instr, ALU-ish {alu}, IMAD {fma}")
        print("  " + " ".join(f"{k}:{v}" for k, v in c.most_common(24)))
