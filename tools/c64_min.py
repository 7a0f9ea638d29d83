import numpy as np, torch, sys, os
sys.path.insert(0, ".")
import synth as S, oracle as O
import paper_1811_05335_b200 as P
N, M, m, R = 4096, 2048, 8, 32
x = S.jittered(N, 4)
w = np.random.default_rng(1).standard_normal((N, 2*m+1)) * O.slot_live(x, 2*M, m)
plan = P.Plan(x, M, 2.0, m, precision="c64").set_bopt(w, "alg2")
h = torch.randn(R, M, dtype=torch.complex64, device="cuda")
out = plan.adjoint_apply(h); torch.cuda.synchronize()
print("done")
