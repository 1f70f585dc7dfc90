import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=collections.defaultdict(float); cnt=collections.Counter()
for r in data:
    name=r[ki].split('(')[0][:70]
    try: v=float(r[vi].replace(',',''))
    except: continue
    tot[name]+=v; cnt[name]+=1
T=sum(tot.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:n]:
    print(f"{v/1e3:10.1f} us  {100*v/T:5.1f}%  n={cnt[k]:4d}  avg={v/cnt[k]/1e3:8.1f}us  {k}")
