"""Host side of the multi-GPU decision on CPU (-m "not gpu"): the step/exchange orchestration
(paper_2404_16283_b200.run_shard_steps with torch_allgather) over a world-size-2 gloo process
group.  Each rank's 'steps' write rank- and step-stamped blocks; the next step must see every
rank's block of the previous round, in rank order, exactly as the library's steps expect."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
XBYTES = [64, 48, 240, 32]  # per-round block sizes (any positive multiples of 16)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2404_16283_b200 as A
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        send = [torch.empty(b, dtype=torch.uint8) for b in XBYTES]
        recv = [torch.empty(world * b, dtype=torch.uint8) for b in XBYTES]
        seen = []

        def step(s, prev, cur):
            if s > 0:
                blocks = prev.view(world, -1)
                seen.append([int(blocks[g, 0]) * 1000 + int(blocks[g, 1]) for g in range(world)])
                assert blocks.shape[1] == XBYTES[s - 1]
            if cur is not None:
                cur.fill_(0)
                cur[0] = rank + 1
                cur[1] = s
                cur[-1] = 7

        A.run_shard_steps(step, A.torch_allgather(), send, recv)
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_shard_exchange_rank_order_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    got = dict(q.get(timeout=5) for _ in range(world))
    for r in range(world):
        # steps 1..4 see round s-1 blocks from ranks 1..world in rank order
        assert got[r] == [[(g + 1) * 1000 + s for g in range(world)] for s in range(4)]
