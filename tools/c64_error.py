"""Diagnostic: where the complex64 error on config 4 (GPU Alg. 2 B_opt) comes from.
Prints GPU-c64 vs oracle with exact or fp32-rounded inputs, and the input-rounding effect alone."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
import synth as S
import paper_1811_05335_b200 as P

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = S.config(cid); x = S.make_nodes(c)
M = c["M"][0] if c["d"] == 1 else tuple(c["M"]); sigma, m = c["sigma"], c["m"]
R = 8
plan = P.Plan(x, M, sigma, m, precision="c64").precompute("alg2")
w = plan.get_bopt()
w32 = w.astype(np.float32).astype(np.float64)
wB = O.window_slot_weights_2d(x, M, sigma, 16) if x.ndim == 2 else O.window_slot_weights(x, M, sigma, 16)
if x.ndim == 2:
    fh = S.blob_image(R, M[0], M[1], 400).reshape(R, -1)
else:
    fh = S.uniform_complex(R, M, 300)
f = O.apply_adjoint(x, M, sigma, 16, wB, 1.0, fh)
f32 = f.astype(np.complex64).astype(np.complex128)
got = plan.apply(torch.from_numpy(f.astype(np.complex64)).cuda()).cpu().numpy().astype(np.complex128)
ref = O.apply_inverse(x, M, sigma, m, w, 1.0, f)
ref32 = O.apply_inverse(x, M, sigma, m, w32, 1.0, f32)
print("max|w|", np.abs(w).max(), "info", plan.info()["n_rank_deficient"])
print("inverse: gpu64 vs oracle(exact inputs)", O.rel_l2(got, ref))
print("inverse: gpu64 vs oracle(fp32 inputs) ", O.rel_l2(got, ref32))
print("inverse: input rounding alone          ", O.rel_l2(ref32, ref))
print("inverse: w rounding alone              ", O.rel_l2(O.apply_inverse(x, M, sigma, m, w32, 1.0, f), ref))
print("inverse: f rounding alone              ", O.rel_l2(O.apply_inverse(x, M, sigma, m, w, 1.0, f32), ref))
print("recovery (c128 oracle)                 ", O.rel_l2(ref, fh))
fn = S.normal_complex(R, x.shape[0], 401)
h = O.apply_inverse(x, M, sigma, 16, wB, 1.0, fn)
h32 = h.astype(np.complex64).astype(np.complex128)
got = plan.adjoint_apply(torch.from_numpy(h.astype(np.complex64)).cuda()).cpu().numpy().astype(np.complex128)
ref = O.apply_adjoint(x, M, sigma, m, w, 1.0, h)
ref32 = O.apply_adjoint(x, M, sigma, m, w32, 1.0, h32)
print("adjoint: gpu64 vs oracle(exact inputs)", O.rel_l2(got, ref))
print("adjoint: gpu64 vs oracle(fp32 inputs) ", O.rel_l2(got, ref32))
print("adjoint: input rounding alone          ", O.rel_l2(ref32, ref))
