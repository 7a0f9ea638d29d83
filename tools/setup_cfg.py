import sys, time, resource
import numpy as np
import synth as S
import paper_1811_05335_b200 as P
cid = int(sys.argv[1])
c = S.config(cid); x = S.make_nodes(c)
M = c["M"][0] if c["d"] == 1 else c["M"]
print("nodes", x.shape, "rss MB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024, flush=True)
plan = P.Plan(x, M, c["sigma"], c["m"])
print("plan ok rss MB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024, flush=True)
t0 = time.perf_counter(); plan.precompute("alg2"); dt = time.perf_counter() - t0
info = plan.info()
print("precompute", round(dt, 2), "s", {k: info[k] for k in ("n_rank_deficient", "max_col_size", "max_lowrank_rank", "max_abs_w")},
      "rss MB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024, flush=True)
w = plan.get_bopt()
print("bopt", w.shape, np.isfinite(w).all(), flush=True)
