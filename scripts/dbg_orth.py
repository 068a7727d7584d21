"""Debug: per-vector norms and scales of the last GMRES cycle basis (cnpint_krylov_basis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2401_16113_b200 import problems
w = synth.C1.with_(alpha=1e-3)
s = problems.make_solver(w, restart_max=w.restart)
b = problems.rhs(w, s)
u = s.empty()
rep = s.gmres(b, u, 1e-12, w.restart)
print(rep["iterations"], rep["history"])
vecs, sc = s.krylov_basis()
for i, (v, c) in enumerate(zip(vecs, sc)):
    vv = b if v is None else v
    print(i, v is None, float(vv.norm()), c, float(vv.norm()) * c, vv.shape)
Q = torch.stack([(b if v is None else v).reshape(-1) * c for v, c in zip(vecs, sc)])
print(Q @ Q.T)
