import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=None; d=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h):
        k=r[h.index('Kernel Name')]
        if 'export' in k or 'from_linear' in k:
            d[k.split('(')[0][-28:]].append(float(r[h.index('Metric Value')].replace(',','')))
for k,v in d.items():
    v=sorted(v); print(f"   {k:30s} n={len(v)} med={v[len(v)//2]/1e3:.2f}us")
