"""Multi-rank host logic of the RHS-sharded path on CPU (gloo, world_size 2)."""
import importlib.util
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load_dist():
    spec = importlib.util.spec_from_file_location("inft_dist", os.path.join(ROOT, "paper_1811_05335_b200", "dist.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_shard_covers_batch():
    D = _load_dist()
    for R in (0, 1, 7, 64, 512, 513):
        for W in (1, 2, 3, 8):
            got = [D.shard(R, r, W) for r in range(W)]
            assert sum(c for _, c in got) == R
            pos = 0
            for s, c in got:
                assert s == pos
                pos += c
    assert D.shard(512, 3, 8) == (192, 64)  # config 5: 64 RHS per GPU at 8 GPUs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = _load_dist()
    try:
        w = np.random.default_rng(5).standard_normal((100, 17))
        digests = D.check_same_bopt(w, dist)
        ok_same = len(set(digests)) == 1
        w2 = w.copy()
        if rank == 1:
            w2[3, 4] = np.nextafter(w2[3, 4], np.inf)  # a one-ulp change must be detected
        try:
            D.check_same_bopt(w2, dist)
            detected = False
        except RuntimeError:
            detected = True
        t = D.max_over_ranks(1.5 + rank, dist)
        start, count = D.shard(64 * world, rank, world)
        q.put((rank, ok_same, detected, t, start, count))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_same, detected, t, start, count in res:
        assert ok_same and detected
        assert t == 2.5  # max over ranks
        assert (start, count) == (64 * rank, 64)
