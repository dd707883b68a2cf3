#!/usr/bin/env python
"""GMRES preconditioner study for BIE 5.4 (NEXT-2) on dense oracle matrices
(CPU only): iteration counts to 1e-10 for plain GMRES, the single-sphere
block (self) preconditioner and the exact inverse of the near-field block
operator (diagonal blocks + eq 4.5 near pairs, eta = 1).
    python tools/precond_study.py 40 4      # 40 spheres, p = 4 (6000 unknowns, ~6 min)
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import scipy.sparse.linalg as sla

def geometry(ns, seed, gapmin):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.5, 1.5, ns)
    side = (np.sum(4/3*np.pi*a**3)/0.15)**(1/3)
    c = []
    while len(c) < ns:
        x = rng.uniform(0, side, 3); i = len(c)
        if all(np.linalg.norm(x-y) > a[i]+a[j]+gapmin*min(a[i],a[j]) for j,y in enumerate(c)):
            c.append(x)
    return np.array(c), a

ns, p, eta = int(sys.argv[1]), int(sys.argv[2]), 1.0
c, a = geometry(ns, 3, 0.2)
t = time.time()
A = O.porous_matrix(c, a, p, 1.0, eta)
print("built", A.shape, time.time()-t, flush=True)
nsn = (p+1)*(2*p+2)
n3 = 3*nsn
# block mask: diagonal blocks + near pairs
M = np.zeros_like(A)
near = 0
for t_ in range(ns):
    for s in range(ns):
        if s == t_ or O.is_near(c[s], a[s], c[t_], a[t_], eta):
            M[t_*n3:(t_+1)*n3, s*n3:(s+1)*n3] = A[t_*n3:(t_+1)*n3, s*n3:(s+1)*n3]
            near += (s != t_)
D = np.zeros_like(A)
for t_ in range(ns):
    D[t_*n3:(t_+1)*n3, t_*n3:(t_+1)*n3] = A[t_*n3:(t_+1)*n3, t_*n3:(t_+1)*n3]
print("near pairs", near)
b = -np.tile([0, 0, 1.0], A.shape[0]//3)
def count(Aop, Mop=None):
    it = [0]
    def cb(x): it[0] += 1
    x, info = sla.gmres(Aop, b, M=Mop, rtol=1e-10, restart=400, maxiter=400, callback=cb, callback_type="pr_norm")
    return it[0], info
print("plain", count(A))
Dinv = np.linalg.inv(D)
print("block-diag (self) precond", count(A, Dinv))
Minv = np.linalg.inv(M)
print("near-field block precond (exact inverse)", count(A, Minv))
