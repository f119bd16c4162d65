"""numpy model of the rounding behaviour of the RK4 stage-combine forms on a
C2-like 1D problem (tanh background with 1e-3 noise, h = 400 / (2^22 - 1), dt = 0.8 k_max):
complex64 arithmetic emulated with float32 arrays and an emulated FMA (product and sum in
float64, one rounding to float32), against a float64 run of the same RK4.  CPU only; it shares
no code with the library or the oracle (it is an experiment, not a test).
  v0  write-light form: Psi' = Psi + ((T_A-Psi) + 2 (T_B-Psi) + (T_C-Psi))/3 + k/6 K4
  v7  carried Q = fl(acc - w Psi), Psi' = fl(Q + w T_C) + k/6 K4, w = fl(1/3)   (drifts linearly)
  v9  carried Q = 3 acc - Psi, Psi' = cr((Q + T_C)/3) + k/6 K4                   (sum rounded)
  v10 as built: exact sum s + e, q = fl(s w), r = s - 3 q, Psi' = fl(q + w (r + e + k/2 K4))
Prints the relative L2 error of each form every 100 steps.
  python scripts/carried_sum_rounding.py [nsteps]"""
import numpy as np, sys
f32=np.float32
def fma(a,b,c): return (a.astype(np.float64)*np.float64(b) + c.astype(np.float64)).astype(f32) if np.isscalar(b) or b.ndim==0 else (a.astype(np.float64)*b.astype(np.float64)+c.astype(np.float64)).astype(f32)
n=1<<16
h=400.0/((1<<22)-1)
x=(np.arange(n)-n/2)*h
rng=np.random.default_rng(1)
psi0=(np.tanh(x)*(1+1e-3*(2*rng.random(n)-1))).astype(np.complex128)
# shift so |psi| ~ O(1): use tanh(x+1) region
psi0=(np.tanh(x+1.0)*(1+1e-3*(2*rng.random(n)-1))).astype(np.complex128)
a,s=1.0,-1.0
def F64(p):
    L=np.zeros_like(p)
    L[2:-2]=(-p[:-4]+16*p[1:-3]-30*p[2:-2]+16*p[3:-1]-p[4:])/(12*h*h)
    return 1j*(a*L+s*np.abs(p)**2*p)   # ends: crude (zero L)
kmax=np.sqrt(8)*h*h/(a*(64/12+ np.max(np.abs(psi0))**2*h*h))
dt=0.8*kmax
def rk4_64(p):
    k1=F64(p);k2=F64(p+dt/2*k1);k3=F64(p+dt/2*k2);k4=F64(p+dt*k3)
    return p+dt/6*(k1+2*k2+2*k3+k4)
# fp32 emulation on separate re/im arrays
w16=f32(16/(12*h*h)); w1=f32(1/(12*h*h))
def tF32(re,im):
    # t = a L + N c, F = i t ; lap5 with centre inside differences
    def lap(u):
        L=np.zeros_like(u)
        c2=(f32(2)*u[2:-2]).astype(f32)
        d1=((u[1:-3]+u[3:-1]).astype(f32)-c2).astype(f32)
        d2=((u[:-4]+u[4:]).astype(f32)-c2).astype(f32)
        t=(w16*d1).astype(f32)
        L[2:-2]=fma(d2,-w1,t)
        return L
    Lr,Li=lap(re),lap(im)
    n2=fma(re,re,(im*im).astype(f32))
    N=(f32(s)*n2).astype(f32)
    tr=fma(Lr,f32(a),(N*re).astype(f32)); ti=fma(Li,f32(a),(N*im).astype(f32))
    return tr,ti
def iaxpy(ar,ai,sc,tr,ti): # a + s*(i t)
    return fma(ti,f32(-sc),ar), fma(tr,f32(sc),ai)
def axpy(ar,ai,sc,br,bi): return fma(br,f32(sc),ar), fma(bi,f32(sc),ai)
W=f32(1.0/3.0)
def step(re,im,variant):
    t=tF32(re,im); TA=iaxpy(re,im,dt/2,*t)
    t=tF32(*TA); TB=iaxpy(re,im,dt/2,*t)
    if variant in (7,71,72,73):
        d=((TA[0]-re).astype(f32),(TA[1]-im).astype(f32))
        u=axpy(re,im,W,*d); A2=iaxpy(u[0],u[1],dt/3,*t); Q=axpy(A2[0],A2[1],-W,re,im)
        if variant==71: # Q without its own rounding
            Q=(A2[0].astype(np.float64)-np.float64(W)*re, A2[1].astype(np.float64)-np.float64(W)*im)
        if variant==72: # A2 exact in f64 then Q rounded once
            A2e=(re.astype(np.float64)+np.float64(W)*d[0]-dt/3*t[1].astype(np.float64), im.astype(np.float64)+np.float64(W)*d[1]+dt/3*t[0].astype(np.float64))
            Q=((A2e[0]-np.float64(W)*re).astype(f32),(A2e[1]-np.float64(W)*im).astype(f32))
        if variant==73: # everything of the carry exact (f64)
            A2e=(re.astype(np.float64)+np.float64(W)*d[0]-dt/3*t[1].astype(np.float64), im.astype(np.float64)+np.float64(W)*d[1]+dt/3*t[0].astype(np.float64))
            Q=(A2e[0]-np.float64(W)*re,A2e[1]-np.float64(W)*im)
    if variant in (9,10):
        d=((TA[0]-re).astype(f32),(TA[1]-im).astype(f32))
        tt=(fma(re,f32(2),d[0]),fma(im,f32(2),d[1]))
        Q3=iaxpy(tt[0],tt[1],dt,*t)
    t=tF32(*TB); TC=iaxpy(re,im,dt,*t)
    t=tF32(*TC)
    if variant==0:
        dA=((TA[0]-re).astype(f32),(TA[1]-im).astype(f32)); dB=((TB[0]-re).astype(f32),(TB[1]-im).astype(f32)); dC=((TC[0]-re).astype(f32),(TC[1]-im).astype(f32))
        ds=axpy(dA[0],dA[1],f32(2),*dB); ds=((ds[0]+dC[0]).astype(f32),(ds[1]+dC[1]).astype(f32))
        u=axpy(re,im,W,*ds); return iaxpy(u[0],u[1],dt/6,*t)
    if variant==10:
        out=[]
        for Qc,Tc,sc,tc in ((Q3[0],TC[0],-dt/2,t[1]),(Q3[1],TC[1],dt/2,t[0])):
            sv=(Qc+Tc).astype(f32); e=(Tc-(sv-Qc).astype(f32)).astype(f32)
            q=(sv*W).astype(f32); r=fma(q,f32(-3),sv); r=(r+e).astype(f32); r=fma(tc,f32(sc),r)
            out.append(fma(r,W,q))
        return out[0],out[1]
    if variant==9:
        def div3(sv):
            q=(sv*W).astype(f32); r=fma(q,f32(-3),sv); return fma(r,W,q)
        sr=(Q3[0]+TC[0]).astype(f32); si=(Q3[1]+TC[1]).astype(f32)
        return iaxpy(div3(sr),div3(si),dt/6,*t)
    if variant in (7,71,72,73):
        if Q[0].dtype==np.float64:
            u=((Q[0]+np.float64(W)*TC[0]).astype(f32),(Q[1]+np.float64(W)*TC[1]).astype(f32))
        else: u=axpy(Q[0],Q[1],W,*TC)
        return iaxpy(u[0],u[1],dt/6,*t)
nsteps=int(sys.argv[1]) if len(sys.argv)>1 else 500
p64=psi0.astype(np.complex64).astype(np.complex128)
r0=psi0.real.astype(f32),psi0.imag.astype(f32)
r7=r0; R={v:r0 for v in (9,10)}
for i in range(nsteps):
    p64=rk4_64(p64); r0=step(*r0,0); r7=step(*r7,7)
    for v in R: R[v]=step(*R[v],v)
    if (i+1)%100==0:
        sl=slice(8,-8)
        def err(r):
            d=(r[0].astype(np.float64)+1j*r[1].astype(np.float64))-p64
            return np.linalg.norm(d[sl])/np.linalg.norm(p64[sl]), np.abs(d[sl]).max()/np.abs(p64[sl]).max()
        print(i+1,'v0 %.2e'%err(r0)[0],'v7 %.2e'%err(r7)[0],' '.join('v%d %.2e'%(v,err(R[v])[0]) for v in R))
