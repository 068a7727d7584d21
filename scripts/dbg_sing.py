"""Debug: singular variable-row P_1 (reflecting ends) — does K3 flag it?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2401_16113_b200.cnpint import OperatorSpec, Solver
for m in (64, 40, 200):
    i = np.arange(m, dtype=np.float64)
    sub = 1.0 + 0.01 * i; sup = 1.0 + 0.02 * i; sub[0] = 0.0; sup[-1] = 0.0
    diag = -(sub + sup)
    s = Solver(16, 1.0, 1.0, OperatorSpec(dim=1, nx=m, toeplitz=False, sub=sub, diag=diag, sup=sup))
    v = s.to_device(np.random.default_rng(3).standard_normal((16, m)))
    z = s.empty(); s.apply_Pinv(v, z); torch.cuda.synchronize()
    print(m, "max|z|", float(z.abs().max()), "status", s.device_status())
