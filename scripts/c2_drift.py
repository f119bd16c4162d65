"""C2 (1D, 2^22) c64 after 500 steps against the oracle, per variant (numerics check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, oracle
from icgen import configs
import harness as H
w = configs.C2()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
for dtype in ("c64",):
    psi = H.psi0_host(w, dtype)
    P = H.oracle_problem(w)
    dt = 0.8 * oracle.kmax(P, psi.astype(np.complex128))
    ref = oracle.rk4(P, psi.astype(np.complex128), dt, steps)
    for v in (0, 6, 2):
        S = H.gpu_solver(w, dtype, v)
        g = torch.from_numpy(psi).cuda()
        S.rk4(g, dt, steps)
        print(dtype, "variant", v, "rel", H.rel_l2(g.cpu().numpy(), ref), flush=True)
