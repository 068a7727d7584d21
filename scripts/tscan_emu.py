"""CPU emulation of k_tscan.cu's arithmetic for one spatial mode (chunked scan, closure, carries) in fp64,
with a rounded rho versus the rho-minus-one form, against a 200-bit mpmath reference: forward error and
residual per mode.  Not part of the product or the oracle; python scripts/tscan_emu.py."""
import numpy as np
from mpmath import mp, mpf
def emu(v, mu, alpha, L=16, NW=8, m1=True):
    N=len(v); J=N//L
    h=0.5*mu; cc=1.0/(1.0-h); d=2.0*h*cc; rho=(1.0+h)*cc
    s=np.zeros(N)
    for j in range(J):
        acc=0.0
        for i in range(L):
            t=j*L+i
            if m1: acc = np.float64(d*acc + (acc+v[t])) if i else v[t]
            else: acc = rho*acc+v[t] if i else v[t]
            s[t]=acc
    # serial carry (sufficient to test rounding model roughly)
    if m1:
        dP=d
        q=1
        while q<L: dP=dP*(dP+2.0); q*=2
        G=0.0; pres=[]
        for j in range(J):
            pres.append(G); G=dP*G+(G+s[j*L+L-1])
        dN=dP; q=1
        while q<J: dN=dN*(dN+2.0); q*=2
        zl=alpha*G/((1.0-alpha)-alpha*dN)
        z=np.zeros(N)
        pw=0.0  # P^j -1
        for j in range(J):
            cin=pw*zl+(zl+pres[j])
            qv=cc*cin
            for i in range(L):
                qv=d*qv+qv
                z[j*L+i]=cc*s[j*L+i]+qv
            pw=pw*dP+(pw+dP)
    else:
        P=rho**L
        G=0.0; pres=[]
        for j in range(J):
            pres.append(G); G=P*G+s[j*L+L-1]
        zl=alpha*G/(1.0-alpha*rho**N)
        z=np.zeros(N)
        for j in range(J):
            cin=P**j*zl+pres[j]
            qv=cc*cin
            for i in range(L):
                qv=qv*rho
                z[j*L+i]=cc*s[j*L+i]+qv
    return z
def exact(v, mu, alpha):
    mp.prec=200
    N=len(v); h=mpf(mu)/2; rho=(1+h)/(1-h); c=1/(1-h)
    s=[]; acc=mpf(0)
    for t in range(N):
        acc=rho*acc+c*mpf(float(v[t])); s.append(acc)
    zl=s[-1]/(1-mpf(alpha)*rho**N)
    return [s[t]+rho**(t+1)*mpf(alpha)*zl for t in range(N)]
rng=np.random.default_rng(0)
for N in (1024,2048):
  for alpha in (1.0,0.01):
    for mu in (-4e-5,-1e-3,-0.1,-3.0,-50.0):
        v=rng.standard_normal(N)
        ze=exact(v,mu,alpha)
        zen=np.array([float(x) for x in ze])
        out=[]
        for m1 in (False,True):
            z=emu(v,mu,alpha,m1=m1)
            fe=np.linalg.norm(z-zen)/np.linalg.norm(zen)
            # backward: residual
            h=0.5*mu
            zm=np.roll(z,1); zm[0]=alpha*z[-1]
            res=(1-h)*z-(1+h)*zm-v
            out.append((fe, np.linalg.norm(res)/np.linalg.norm(v)))
        print(N,alpha,mu,"rounded-rho fwd/back %.1e %.1e | minus-one fwd/back %.1e %.1e"%(out[0]+out[1]))
