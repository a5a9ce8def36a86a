import csv, collections, sys
hdr=None; rows=[]
for r in csv.reader(open(sys.argv[1])):
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): rows.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for d in rows:
    k=d['Kernel Name'].split('(')[0][:60]
    agg[k][d['Metric Name']].append((float(d['Metric Value']), d['Metric Unit']))
tot=0
for k,mm in agg.items():
    out=[]
    for mn,vals in mm.items():
        out.append(f"{mn.split('__')[1][:18]}={sum(v for v,_ in vals)/len(vals)/1e3:.2f}k{vals[0][1]}")
        if 'time' in mn: tot+=sum(v for v,_ in vals)
    print(f"{k:60s} n={len(next(iter(mm.values())))}", ' '.join(out))
print('total us', tot/1e3)
