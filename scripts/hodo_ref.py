import numpy as np, math
def binom(n,k): return math.comb(n,k)
def hodo(n, H):
    w = H[:,2]; P = H[:,:2]/w[:,None]
    D = np.zeros((2*n,2)); E = np.zeros(2*n+1)
    for i in range(n):
        for j in range(n+1):
            c = binom(n-1,i)*binom(n,j)/binom(2*n-1,i+j)
            D[i+j] += c*w[j]*(w[i+1]*(P[i+1]-P[j]) - w[i]*(P[i]-P[j]))
    for i in range(n+1):
        for j in range(n+1):
            E[i+j] += binom(n,i)*binom(n,j)/binom(2*n,i+j)*w[i]*w[j]
    return n*np.max(np.hypot(D[:,0],D[:,1]))/E.min()
def floater(n,H):
    w=H[:,2]; P=H[:,:2]/w[:,None]
    dmax=max(np.hypot(*(P[j]-P[j-1])) for j in range(1,n+1))
    if w.max()==w.min(): return n*dmax
    diam=max(np.hypot(*(P[j]-P[i])) for i in range(n+1) for j in range(i+1,n+1))
    r=w.max()/w.min(); return min(n*r*diam, n*r*r*dmax)
def split(n,H):
    T=H.copy(); L=np.zeros_like(H); R=np.zeros_like(H); L[0]=T[0]; R[n]=T[n]
    for r in range(1,n+1):
        for j in range(0,n-r+1): T[j]=0.5*(T[j]+T[j+1])
        L[r]=T[0]; R[n-r]=T[n-r]
    return L,R
def pieces(n,H):
    a,b=split(n,H); out=[]
    for x in (a,b):
        c,d=split(n,x)
        for y in (c,d):
            e,f=split(n,y); out+= [e,f]
    return out
