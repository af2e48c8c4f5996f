import sys, numpy as np, torch, ctypes as ct, math
sys.path.insert(0, '.')
from fractions import Fraction as F
import paper_2202_08361_b200 as J
def fma(a,b,c): return float(F(a)*F(b)+F(c))
OMEGA=np.finfo(np.float64).max; MU=5e-324
rows=[(-MU, OMEGA/8, 2.0**1020), (1.48219694e-323, OMEGA/8, -1.0)]
A=[];B=[]
for a11,a22,re in rows:
    ab=abs(re); o=ab*2; a=a11-a22
    t2=math.copysign(min(max(o/abs(a),0.0), math.sqrt(OMEGA)), a)
    t=t2/(1.0+math.sqrt(fma(t2,t2,1.0)))
    s2=fma(t,t,1.0)
    n1=fma(t,fma(a22,t,o),a11)
    print(repr(t2), repr(t), repr(s2), n1.hex(), (n1/s2).hex())
    A += [o, t2, n1]; B += [abs(a), 1.0+math.sqrt(fma(t2,t2,1.0)), s2]
a=np.array(A); b=np.array(B)
L=J.lib(); L.jsvd_debug_primitive.argtypes=[ct.c_int32, ct.c_int64]+[ct.c_void_p]*4
ga,gb=torch.from_numpy(a).cuda(),torch.from_numpy(b).cuda(); q=torch.empty_like(ga)
for mode in (0,1):
    L.jsvd_debug_primitive(mode, a.size, ga.data_ptr(), gb.data_ptr(), q.data_ptr(), None); torch.cuda.synchronize()
    g=q.cpu().numpy()
    for x,y,z in zip(a,b,g): print(mode, x.hex(), y.hex(), z.hex(), (x/y).hex(), z==x/y)
import oracle as O
for a11,a22,re in rows:
    x=[torch.tensor([v],dtype=torch.float64).cuda() for v in (a11,a22,re)]
    for fl in (0,1,2,3):
        g=J.evd2_batched(*x, flags=fl); torch.cuda.synchronize()
        o=O.evd2_one(False,a11,a22,re,0.0,fl)
        print(fl, {k:(g[k].item().hex(), o[k].hex()) for k in ('lam1','lam2','cos','sin_re') if g[k].item()!=o[k] or str(g[k].item())!=str(o[k])})
