import sys, numpy as np, itertools
from fractions import Fraction as F
sys.path.insert(0,'.')
import oracle, paper_2205_02646_b200 as tq
ref=oracle.Reference(); orc=oracle.Oracle()
W,B,P,rows=8,2,4,32
img=tq.synthetic_image(rows, rows+2*B, 500+W+B); pat=tq.generate_pattern(11,P,B); fr=tq.simulate_measurement(img,pat)
orow,ocol=int(sys.argv[1]),int(sys.argv[2])
y=orc.gather(fr,orow,ocol,W)
t=ref.precompute(pat.opaque,P,orow,ocol,W)
K=W*W; L=t["L"]; b=t["b"]; c=t["c"]; d=t["d"]; q=ref.frequency_weights(W)
def fma(a,b_,c_): return float(F(a)*F(b_)+F(c_))
bre=b.real.reshape(K,L); bim=b.imag.reshape(K,L); cc=c.reshape(K,K)
rp,rg,_=ref.block_trace(pat.opaque,P,orow,ocol,W,y,iterations=60)
def run(init_fma, upd, n=30):
    Rr=np.zeros(K); Ri=np.zeros(K)
    for k in range(K):
        re=0.0; im=0.0
        for m in range(L):
            nu = 8*(L//8) + (4 if L%8>=4 else 0)
            if init_fma or m >= nu: re=fma(bre[k,m],y[m],re); im=fma(bim[k,m],y[m],im)
            else: re=re+bre[k,m]*y[m]; im=im+bim[k,m]*y[m]
        Rr[k]=re; Ri[k]=im
    gds=[]; picks=[]
    for it in range(n):
        best=-1; bs=0.0
        for k in range(K):
            dk=d[k]
            if dk<=0: continue
            s=(q[k]*fma(Rr[k],Rr[k],Ri[k]*Ri[k]))/dk
            if best<0 or s>bs: best=k; bs=s
        u=best; du=d[u]; gr=0.5*(Rr[u]/du); gi=0.5*(Ri[u]/du)
        gds.append(complex(gr,gi)); picks.append(u)
        for s in range(K):
            cr=cc[u,s].real; ci=cc[u,s].imag
            a_, b2 = upd(gr,gi,cr,ci)
            Rr[s]=Rr[s]-a_; Ri[s]=Ri[s]-b2
    return picks,gds
upds={
 "A fma(gr,cr,-gi*ci) fma(gr,ci,gi*cr)": lambda gr,gi,cr,ci:(fma(gr,cr,-(gi*ci)), fma(gr,ci,gi*cr)),
 "B fma(-gi,ci,gr*cr) fma(gi,cr,gr*ci)": lambda gr,gi,cr,ci:(fma(-gi,ci,gr*cr), fma(gi,cr,gr*ci)),
 "C fma(gr,cr,-gi*ci) fma(gi,cr,gr*ci)": lambda gr,gi,cr,ci:(fma(gr,cr,-(gi*ci)), fma(gi,cr,gr*ci)),
 "D fma(-gi,ci,gr*cr) fma(gr,ci,gi*cr)": lambda gr,gi,cr,ci:(fma(-gi,ci,gr*cr), fma(gr,ci,gi*cr)),
 "E nofma": lambda gr,gi,cr,ci:(gr*cr-gi*ci, gr*ci+gi*cr),
}
for init_fma in ():
    for name,u in upds.items():
        p,g=run(init_fma,u,8)
        ok=[g[i]==rg[i] for i in range(8)]
        print(init_fma, name, "match first 8:", ok.count(True), "first mismatch", ok.index(False) if False in ok else None)
print("---- 30 iterations, init without fma")
for name,u in upds.items():
    p,g=run(False,u,60)
    ok=[g[i]==rg[i] for i in range(len(rg))]
    print(name, "match:", ok.count(True), "first mismatch", ok.index(False) if False in ok else None, "picks equal", list(p)==list(rp))
print("---- synthesis")
_,_,rwin=ref.block_trace(pat.opaque,P,orow,ocol,W,y,iterations=60)
import math
unit=[]
for k in range(W):
    if k==0: unit.append((1.0,0.0))
    elif k==W//2: unit.append((-1.0,0.0))
    elif k<W//2: a=2*math.pi*k/W; unit.append((math.cos(a),math.sin(a)))
    else: unit.append(None)
for k in range(W//2+1,W): unit[k]=(unit[W-k][0],-unit[W-k][1])
coef={}; order=[]
for u,g in zip(rp,rg):
    u=int(u)
    if u not in coef: coef[u]=0j; order.append(u)
    coef[u]=complex(coef[u].real+g.real, coef[u].imag+g.imag)
variants={"S1":lambda cre,cim,pr,pi:fma(cre,pr,-(cim*pi)),"S2":lambda cre,cim,pr,pi:fma(-cim,pi,cre*pr),"S3":lambda cre,cim,pr,pi:cre*pr-cim*pi}
for name,f in variants.items():
    win=np.zeros((W,W))
    for fl in order:
        s_,r_=divmod(fl,W); cre,cim=coef[fl].real,coef[fl].imag
        for eta in range(W):
            for gam in range(W):
                pr,pi=unit[(eta*s_+gam*r_)%W]
                win[eta,gam]=win[eta,gam]+f(cre,cim,pr,pi)
    print(name, "bitwise:", np.array_equal(win, rwin), np.abs(win-rwin).max())
print("---- detail")
p,g=run(False,upds["A fma(gr,cr,-gi*ci) fma(gr,ci,gi*cr)"],12)
print("picks ref", [int(x) for x in rp[:12]]); print("picks emu", p)
for i in range(8,11): print(i, g[i], rg[i])
print("L", L, "D<=0 count", int((d<=0).sum()), "d of picks", [d[int(x)] for x in rp[:12]])
