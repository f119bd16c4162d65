import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import icgen, oracle
import paper_1109_1027_b200 as nl
from icgen import configs
dims = int(sys.argv[1]); n = tuple(int(v) for v in sys.argv[2].split(',')); dt = sys.argv[3]
w = configs.SMALL(dims, n, "dirichlet", dtype=dt, V="harmonic")
psi = icgen.fill(w["ic"], w["grid"], dtype=np.complex64 if dt == "c64" else np.complex128)
S = nl.solver_from_work(w, dt)
L = S.laplacian(torch.from_numpy(psi).cuda()); torch.cuda.synchronize()
Lo = oracle.laplacian(oracle.problem_from_work(w), psi.astype(np.complex128))
print(dims, n, dt, "rel", np.linalg.norm(L.cpu().numpy() - Lo) / np.linalg.norm(Lo), flush=True)
