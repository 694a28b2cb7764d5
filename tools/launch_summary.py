import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
tot=collections.defaultdict(float); cnt=collections.Counter()
scale={'ns':1e-3,'nsecond':1e-3,'us':1,'usecond':1,'ms':1e3,'msecond':1e3}
for r in data:
    if len(r)<=vi: continue
    name=r[ki].split('(')[0][:60]
    us=float(r[vi].replace(',',''))*scale[r[ui]]
    tot[name]+=us; cnt[name]+=1
T=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{k:60s} n={cnt[k]:5d} total={v:10.1f}us avg={v/cnt[k]:8.1f}us share={v/T:.3f}")
