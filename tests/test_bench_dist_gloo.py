"""bench.py's with-communication path (rank 0 scatters inputs, gathers outputs)
with 2 gloo ranks on CPU and a stand-in plan: the collectives line up and every rank's shard
comes back to rank 0 in order."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class FakePlan:
    """inverse: fhat = f[:, :M] * 2; adjoint: f = h tiled to N then * 3 (shapes only)."""

    def __init__(self, N, M):
        self.N, self.M = N, M

    def apply(self, f, out):
        out.copy_(f[:, : self.M] * 2)

    def adjoint_apply(self, h, out):
        out.copy_(torch.cat([h, h], dim=1)[:, : self.N] * 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sys.path.insert(0, ROOT)
    import bench
    R, N, M = 3, 10, 6
    plan = FakePlan(N, M)
    res = bench.run_dist_e2e(plan, R, N, M, torch.complex128, ws, rank, torch.device("cpu"), 2, torch, dist,
                             return_outputs=True)
    same = True
    if rank == 0:
        # every rank's shard came back to rank 0 in order: the gathered outputs equal the
        # stand-in plan applied to the whole batch
        F, H, fo, ho = res["outputs"]
        ref_i = torch.empty_like(fo)
        ref_a = torch.empty_like(ho)
        plan.apply(F, out=ref_i)
        plan.adjoint_apply(H, out=ref_a)
        same = bool(torch.equal(fo, ref_i) and torch.equal(ho, ref_a))
    q.put((rank, res["value"] > 0 and same, res["collective_bytes_per_step"]))
    dist.destroy_process_group()


def test_dist_e2e_collectives_gloo():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get() for _ in range(ws))
    assert all(ok for _, ok, _ in out)
    assert out[0][2] == 3 * 2 * (10 + 6) * 2 * 16
