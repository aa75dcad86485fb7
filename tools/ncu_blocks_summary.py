import csv,sys,subprocess
rep=sys.argv[1]
extra=sys.argv[3:] if len(sys.argv)>3 else []
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass']+extra,capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=rows[1]; c={k:j for j,k in enumerate(hdr)}
data=[r for r in rows[2:] if len(r)==len(hdr)]
def f(x):
    try: return float(x)
    except: return 0.0
I=c['Instructions Executed']; S=c['Warp Stall Sampling (All Samples)']
ti=sum(f(r[I]) for r in data); ts=sum(f(r[S]) for r in data)
print('total inst %.4g  samples %d'%(ti,ts))
bbs=[];cur=None
for i,r in enumerate(data):
    n=f(r[I]); src=r[c['Source']].strip()
    if cur and cur[1]==n: cur[2]+=1; cur[3].append(src); cur[4]+=f(r[S])
    else:
        if cur: bbs.append(cur)
        cur=[i,n,1,[src],f(r[S])]
bbs.append(cur)
thr=float(sys.argv[2]) if len(sys.argv)>2 else 0.004
for b in bbs:
    tot=b[1]*b[2]
    if tot/ti>thr or b[4]/ts>thr:
        ops=[s.split()[1] if s.startswith('@') else s.split()[0] for s in b[3]]
        mem=[o for o in ops if o.split('.')[0] in ('LDS','STS','ATOMS','LD','LDG','ST','STG','SHFL','UBLKCP','SYNCS','CREDUX','REDUX','BAR','NANOSLEEP','YIELD')]
        print(f"{b[0]:5d} x{int(b[1]):>10d} n={b[2]:3d} inst {100*tot/ti:5.2f}% stall {100*b[4]/ts:5.2f}%  {' '.join(mem)[:70]}")
