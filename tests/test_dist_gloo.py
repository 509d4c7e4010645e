"""World-size-2 (and 4) gloo tests on CPU for the N > 1 host logic: rank -> (cluster, local
rank) mapping, NCCL unique-id broadcast through torch.distributed, and the exchange
semantics the library implements (every cluster decodes every cluster's payload bytes in
the same tree order) checked against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from gradgen import seed_for, synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, G, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import paper_2205_09470_b200 as nb
        P, c, l = nb.topology_for_rank(rank, world, G)
        uid = nb.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        # the payload exchange: each cluster (G == 1) compresses its own bucket with the
        # oracle, the bytes travel through all_gather, every rank decodes + tree-averages
        codec = O.Codec(method=O.INT8)
        n = 5003
        outs = []
        r = np.zeros(n, np.float32)
        for t in range(3):
            g = synthetic(n, seed_for(c, l, t), "model-like")
            res = O.cluster_step(g, r, codec, t)
            r = res.r_new
            buf = torch.frombuffer(bytearray(res.payload), dtype=torch.uint8)
            allb = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(allb, buf)
            outs.append(O.average([bytes(x.numpy()) for x in allb], n))
        q.put((rank, (P, c, l), len(uid), len(set(ids)), [o.tobytes() for o in outs]))
    finally:
        dist.destroy_process_group()


def _run(world, G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, G, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


@pytest.mark.parametrize("world,G", [(2, 1), (4, 2)])
def test_gloo_topology_uid_and_exchange(world, G):
    res = _run(world, G)
    for rank, (P, c, l), uidlen, nuniq, outs in res:
        assert (P, c, l) == (world // G, rank // G, rank % G)
        assert uidlen == 128 and nuniq == 1          # every rank got the same NCCL unique id
    # every rank averaged the same bytes to the same bits
    assert all(r[4] == res[0][4] for r in res)
    if G == 1:
        # and that equals the single-process oracle step over the same clusters
        n, codec = 5003, O.Codec(method=O.INT8)
        rs = [np.zeros(n, np.float32) for _ in range(world)]
        for t in range(3):
            gs = [synthetic(n, seed_for(c, 0, t), "model-like") for c in range(world)]
            out, rs, _, _ = O.oracle_step(gs, rs, codec, t)
            assert out.tobytes() == res[0][4][t]
