"""bench.py's distributed flow with the REAL library, 2 ranks over gloo on one GPU (the pool has
one GPU per box; the ranks' kernels never wait on each other -- every collective is a gloo CPU
collective): each rank builds its own plan replica and runs the GPU Alg. 2 setup, the ranks
prove they hold bit-identical B_opt (SHA-256 digest all-gather), rank 0 scatters the batch,
every rank applies its shard, rank 0 gathers -- and the gathered outputs must be bit-identical
to ONE plan applied shard by shard (the apply kernels are deterministic), and equal to one plan
applied to the whole batch at once to rounding (the ring kernels' node chunks depend on the batch
size, which changes the straight-line / general code path of some 16-node batches).
Sharding basis: independent right-hand sides for fixed nodes."""
import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        import bench
        import synth as S
        import paper_1811_05335_b200 as P
        from paper_1811_05335_b200 import dist as D
        torch.cuda.set_device(0)
        M, N, m = 1 << 14, 1 << 15, 8
        x = S.jittered(N, 4)
        plan = P.Plan(x, M, 2.0, m, device=0).precompute("alg2")
        info = plan.info()
        digests = D.check_same_bopt(plan.get_bopt(), dist, device=torch.device("cpu"))
        R = 32
        res = bench.run_dist_e2e(plan, R, N, M, torch.complex128, ws, rank, torch.device("cuda", 0), 1, torch, dist,
                                 comm_dev=torch.device("cpu"), return_outputs=True)
        t = D.max_over_ranks(float(rank + 1), dist, device=torch.device("cpu"))
        ok = len(set(digests)) == 1 and t == float(ws) and info["fast_path"] == 2 and info["fused_fft"] == 1
        detail = ""
        if rank == 0:
            F, H, fo, ho = res["outputs"]
            sh_i = torch.cat([plan.apply(F[i:i + R].cuda()).cpu() for i in range(0, ws * R, R)])
            sh_a = torch.cat([plan.adjoint_apply(H[i:i + R].cuda()).cpu() for i in range(0, ws * R, R)])
            same = bool(torch.equal(fo, sh_i) and torch.equal(ho, sh_a))
            one_i = plan.apply(F.cuda()).cpu()
            one_a = plan.adjoint_apply(H.cuda()).cpu()
            rel = max(float((fo - one_i).norm() / one_i.norm()), float((ho - one_a).norm() / one_a.norm()))
            detail = f"bit-identical to shard-wise apply: {same}; vs whole batch rel {rel:.2e}"
            ok = ok and same and rel <= 1e-14
        q.put((rank, ok, detail))
        dist.destroy_process_group()
    except Exception as ex:  # report instead of hanging the other rank
        q.put((rank, False, repr(ex)[:500]))


def test_two_rank_flow_equals_one_plan():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(ws))
    for p in procs:
        p.join(120)
    assert all(ok for _, ok, _ in out), out
