"""Per-tile phase times of k_assign_heavy_tiles from a KM_HEAVY_PROF=1 build's printf log:
   python tools/heavy_phases.py <log>  (the longest tiles of one launch, phase medians)."""
import re,sys,statistics
L=[l for l in open(sys.argv[1]) if l.startswith('htile')]
recs=[dict((k,int(v)) for k,v in re.findall(r'(\w+)=(\d+)',l)) for l in L]
recs.sort(key=lambda r:r['start'])
launches=[]; cur=[]
for r in recs:
    if cur and r['start']-cur[-1]['start']>200000: launches.append(cur); cur=[]
    cur.append(r)
launches.append(cur)
Lr=max(launches[-3:],key=len)
t0=min(r['start'] for r in Lr)
for r in Lr: r['tot']=r['stage']+r['refine']+r['walk']+r['sums']+r['row']; r['end']=r['start']-t0+r['tot']
print("kernel span ns", max(r['end'] for r in Lr), "items", len(Lr))
for r in sorted(Lr,key=lambda r:-r['end'])[:6]: print({k:r[k] for k in ('blk','h','T','chunk','gc','nt','stage','refine','walk','sums','row','tot')}, 'start', r['start']-t0)
for k in ('stage','refine','walk','sums','row','tot'): print(k, 'median', statistics.median(r[k] for r in Lr), 'max', max(r[k] for r in Lr))
