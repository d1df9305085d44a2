"""Dump one kernel's SASS (instruction lines only) by name substring and report
spill instructions near its Philox multiply chain (development tool):
python tools/sassfun.py <libmsb200.so> <substring> <out.sass>"""
import re, subprocess, sys
txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for part in re.split(r"\n\s+Function : ", txt):
    name = part.split("\n", 1)[0]
    if sys.argv[2] in name:
        L = [re.sub(r"\s+", " ", re.sub(r"/\*[0-9a-fx ]*\*/", "", l)).strip()
             for l in part.split("\n") if re.search(r"/\*[0-9a-f]{4}\*/", l)]
        open(sys.argv[3], "w").write("\n".join(L))
        wide = [i for i, l in enumerate(L) if "IMAD.WIDE.U32" in l and ("-0x2daee0ad" in l or "-0x326172a9" in l)]
        spill = [i for i, l in enumerate(L) if re.search(r"\b(STL|LDL)", l)]
        near = [i for i in spill if wide and wide[0] - 50 < i < wide[-1] + 50]
        print(name[-60:], "instrs", len(L), "philox products", len(wide),
              "range", (wide[0], wide[-1]) if wide else None, "spills near", near)
        break
