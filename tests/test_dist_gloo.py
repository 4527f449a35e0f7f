"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 host logic in paper_2102_13272_b200.dist:
batch sharding, the single broadcast of U, max-over-ranks timing and the verification gather.
The per-rank "layer" here is the FP64 oracle (the GPU kernels need a B200); what is tested is that
sharding by batch + gather reproduces the unsharded result exactly (images are independent, Eq. 2.1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_13272_b200 import dist as nwd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import direct
        # 1) broadcast of U: rank 0's bytes arrive everywhere
        U = torch.arange(4096, dtype=torch.uint8) if rank == 0 else torch.zeros(4096, dtype=torch.uint8)
        nwd.broadcast_filter(U)
        ok_bcast = bool(torch.equal(U, torch.arange(4096, dtype=torch.uint8)))
        # 2) max over ranks
        m = nwd.max_over_ranks(1.5 + rank)
        # 3) shard a batch of 5 images, run the per-image layer, gather
        layer = synth.small(synth.CONFIGS["c2k5"], N=5, H=11, W=9, Cin=3, Cout=2)
        t = synth.make_inputs(layer)
        s0, cnt = nwd.shard(layer.N, world, rank)
        x = t["x"][s0:s0 + cnt].double().numpy()
        y_local = torch.from_numpy(direct.conv2d(x, t["w"].double().numpy(), 1, layer.pad))
        y = nwd.gather_batch(y_local)
        ref = direct.conv2d(t["x"].double().numpy(), t["w"].double().numpy(), 1, layer.pad)
        ok_gather = bool(np.array_equal(y.numpy(), ref))
        q.put((rank, ok_bcast, m, cnt, ok_gather))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for n in (0, 1, 7, 32, 33, 256):
        for ws in (1, 2, 3, 8):
            spans = [nwd.shard(n, ws, r) for r in range(ws)]
            assert sum(c for _, c in spans) == n
            pos = 0
            for s, c in spans:
                assert s == pos
                pos += c
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        nwd.shard(4, 2, 2)


def test_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] for r in res), "broadcast of U"
    assert all(r[2] == 2.5 for r in res), "max over ranks"
    assert [r[3] for r in res] == [3, 2], "shard sizes"
    assert all(r[4] for r in res), "sharded + gathered == unsharded"
