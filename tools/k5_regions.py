"""K5 instruction / stall-sample breakdown by code region.
usage: k5_regions.py <ncu source-page sass csv> <nvdisasm --print-line-info sass> [k5_blend.cu]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_lines as S, csv
from collections import defaultdict
csvp, sassp = sys.argv[1], sys.argv[2]
rows=list(csv.reader(open(csvp)))
hi=next(i for i,r in enumerate(rows) if r and r[0]=="Address"); h=rows[hi]
ia,iex,ist=h.index("Address"),h.index("Instructions Executed"),h.index("Warp Stall Sampling (All Samples)")
data=[r for r in rows[hi+1:] if len(r)==len(h)]
base=int(data[0][ia],16)
lm=S.line_map(sassp,'_ZN3gut12blend_kernelILi0EEEvNS_6DevCamENS_9BlendBufsE','k5_blend.cu')
src=open(sys.argv[3] if len(sys.argv)>3 else os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', 'paper_2412_12507_b200', 'csrc', 'k5_blend.cu')).read().split('\n')
def L(p): return next(i+1 for i,l in enumerate(src) if p in l)
bounds=[("warp_pass head",L("__device__ __forceinline__ void warp_pass"),L("      // ---- stage entry kk")),
("staging",L("      // ---- stage entry kk"),L("      // ---- conservative cull against")),
("cull1",L("      // ---- conservative cull against"),L("      if (maybe) {")),
("table+cull2",L("      if (maybe) {"),L("    uint32_t m = __ballot_sync(FULL, maybe);")),
("fine",L("    uint32_t m = __ballot_sync(FULL, maybe);"),L("  cp_async_wait<0>();  // a warp leaving")),
("fetch",L("__device__ bool fetch_work"),L("// Persistent CTAs")),
("kernel",L("// Persistent CTAs"),L("    // ---- predecessor peek")),
("peek+pass",L("    // ---- predecessor peek"),L("        // decoupled look-back")),
("lookback",L("        // decoupled look-back"),L("    // ---- exact result")),
("redo/stats",L("    // ---- exact result"),L("    // ---- outputs: single")),
("outputs",L("    // ---- outputs: single"),len(src)+1)]
acc=defaultdict(lambda:[0,0]); tot=[0,0]
for r in data:
    off=int(r[ia],16)-base; ln,_=lm.get(off,(None,""))
    ex=int(r[iex] or 0); st=int(r[ist] or 0)
    g="other(helpers)" if ln is not None else "other(none)"
    if ln is not None:
        for name,lo,hi_ in bounds:
            if lo<=ln<hi_: g=name
    acc[g][0]+=ex; acc[g][1]+=st; tot[0]+=ex; tot[1]+=st
print("total inst %.1fM samples %d"%(tot[0]/1e6, tot[1]))
for g,(ex,st) in sorted(acc.items(), key=lambda kv:-kv[1][1]):
    print(f"{g:28s} {ex/1e6:8.1f}M {100*ex/tot[0]:5.1f}%  stall-samples {100*st/tot[1]:5.1f}%")
