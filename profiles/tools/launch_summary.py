import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg={}; tot=0; seq=[]
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',','')); u=r[ui]
    v = v/1e3 if u=='nsecond' else (v*1e3 if u=='msecond' else v)
    k=r[ki][:60]; agg.setdefault(k,[0,0]); agg[k][0]+=v; agg[k][1]+=1; tot+=v; seq.append((k,v))
if len(sys.argv)>2:
    for k,v in seq: print(f"{v/1e6:9.3f} ms {k}")
else:
    for k,(v,n) in sorted(agg.items(), key=lambda x:-x[1][0])[:12]: print(f"{v/1e6:9.3f} ms {n:3d}x {100*v/tot:5.1f}% {k}")
print('total', tot)
