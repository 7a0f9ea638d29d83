"""Time the GPU B_opt setup at full config sizes (configs 1,2,3,5 and optionally 4)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import synth as S
import paper_1811_05335_b200 as P

which = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]
for cid in which:
    c = S.config(cid)
    x = S.make_nodes(c)
    M = c["M"][0] if c["d"] == 1 else c["M"]
    t0 = time.time()
    plan = P.Plan(x, M, c["sigma"], c["m"])
    t1 = time.time()
    plan.precompute("alg1" if c["alg"] == 1 else "alg2")
    t2 = time.time()
    info = plan.info()
    w = plan.get_bopt()
    print(f"config {cid}: plan {t1 - t0:.2f}s precompute {t2 - t1:.2f}s rank_def {info['n_rank_deficient']} "
          f"empty {info['n_empty_cols']} max_col {info['max_col_size']} max|w| {info['max_abs_w']:.3e} "
          f"finite {np.isfinite(w).all()}", flush=True)
