import sys, csv
sys.path.insert(0,'tools')
import sass_lines as S
from collections import defaultdict
name=sys.argv[1]; fn=sys.argv[2] if len(sys.argv)>2 else '_ZN3gut12blend_kernelILi0EEEvNS_6DevCamENS_9BlendBufsE'
src=sys.argv[3] if len(sys.argv)>3 else 'k5_blend.cu'
rows=list(csv.reader(open(f'/tmp/{name}_sass.csv')))
hi=next(i for i,r in enumerate(rows) if r and r[0]=="Address"); h=rows[hi]
ia,iex,ist=h.index("Address"),h.index("Instructions Executed"),h.index("Warp Stall Sampling (All Samples)")
data=[r for r in rows[hi+1:] if len(r)==len(h)]
base=int(data[0][ia],16)
lm=S.line_map(f'/tmp/{name}_lines.sass',fn,src)
acc=defaultdict(lambda:[0,0,0])
for r in data:
    off=int(r[ia],16)-base; ln,f=lm.get(off,(None,""))
    ex=int(r[iex] or 0); st=int(r[ist] or 0)
    acc[ln][0]+=ex; acc[ln][1]+=st; acc[ln][2]+=1
tot=sum(v[0] for v in acc.values())
srcl=open('paper_2412_12507_b200/csrc/'+src).read().split('\n')
lo,hi_=int(sys.argv[4]),int(sys.argv[5])
s=0
for ln in sorted(k for k in acc if k is not None and lo<=k<=hi_):
    v=acc[ln]; s+=v[0]
    print(f"{ln:5d} {v[0]/1e6:7.2f}M n{v[2]:3d} st{v[1]:5d} | {srcl[ln-1].strip()[:90]}")
print("sum %.1fM of %.1fM"%(s/1e6,tot/1e6))
