import csv, sys, re
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
stall_cols=[h for h in hdr if h.startswith('stall_') and '(Not Issued)' not in h]
tot=sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data)
print("total samples", tot)
# group into regions by instruction index windows; print top instructions
items=[]
for n,r in enumerate(data):
    s=int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    items.append((s,n,r[ix['Source']].strip(),{c:int(r[ix[c]] or 0) for c in stall_cols}))
top=sorted(items,reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 40]
for s,n,src,st in top:
    best=sorted(st.items(),key=lambda x:-x[1])[:3]
    print(f"{n:5d} {s:6d} {100*s/tot:5.1f}% {src[:60]:60s} {best}")
