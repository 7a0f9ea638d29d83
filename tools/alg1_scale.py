"""Time the GPU Alg. 1 setup (Gram by grid pairs) at config-5 scale and beyond.

    python tools/alg1_scale.py
"""
import os
import sys
import time

import numpy as np

_ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path[:0] = [_ROOT, os.path.join(_ROOT, "tests")]
import paper_1811_05335_b200 as P  # noqa: E402
import synth as S  # noqa: E402

for N, M, m, window in [(1 << 21, 1 << 20, 8, "kb"), (1 << 20, 1 << 21, 8, "kb"), (1 << 20, 1 << 21, 8, "dirichlet")]:
    x = S.jittered(N, 4)
    plan = P.Plan(x, M, 2.0, m, window=window)
    t0 = time.perf_counter()
    plan.precompute("alg1")
    dt = time.perf_counter() - t0
    info = plan.info()
    w = plan.get_bopt()
    print(f"N=2^{N.bit_length()-1} M=2^{M.bit_length()-1} m={m} {window}: Alg. 1 setup {dt:.2f} s, "
          f"rank-deficient {info['n_rank_deficient']}, finite {bool(np.all(np.isfinite(w)))}, "
          f"max|w| {np.abs(w).max():.3g}", flush=True)
