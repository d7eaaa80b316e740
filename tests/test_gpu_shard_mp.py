"""The multi-GPU decision across real processes (-m gpu): world-size-2 process group (gloo),
each rank a separate process with its own CUDA context on cuda:0, running the library's five
andes_schedule_shard steps on its contiguous shard; the four exchanges are host-staged gloo
all-gathers (device -> host -> all_gather -> device), i.e. the exact byte blocks an NCCL
all-gather would move.  Every rank's outputs are compared with the CPU oracle's decision on
the whole population (SURVEY 8(c) "Multi-GPU": bit-exact)."""
import os
import socket

import numpy as np
import pytest

from conftest import assert_decision_equal, oracle_decision_cached, snapshot_cached

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, cap, flags, q, comm=False):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import paper_2404_16283_b200 as A
    from conftest import snapshot_cached
    import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        snap = snapshot_cached(name)
        cuts = np.linspace(0, snap.n, world + 1).astype(np.int64)
        mine = W.shard(snap, int(cuts[rank]), int(cuts[rank + 1]))
        ctx = A.Context(max_requests=max(mine.n, 1), max_B=256, max_tokens=mine.n_tokens + 64, device=0)
        req = A.requests_to(mine)
        tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
        sh = ctx.shard_init(world, rank, int(tau.numel()))
        bufs = ctx.alloc_shard_buffers(sh)

        def host_allgather(send, recv):
            h = send.cpu()  # synchronises the producing step
            hr = torch.empty(world * h.numel(), dtype=torch.uint8)
            dist.all_gather(list(hr.chunk(world)), h)
            recv.copy_(hr)

        ag = host_allgather
        if comm:
            # the exchanges as device collectives over peer memory (andes_comm: CUDA IPC mappings of
            # each rank's arena); only the 64-byte handles travel over the host channel, once
            c = A.Comm(world, rank, max(int(x) for x in sh.xbytes), device=0)
            hs = [None] * world
            dist.all_gather_object(hs, c.handle)
            c.connect(hs)
            ag = c.allgather
        out = A.schedule_sharded(ctx, sh, req, mine.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity,
                                 ag, bufs=bufs, preempt_cap=cap, flags=flags)
        if comm:
            # a second decision through the same communicator (sequence numbers and arena parities
            # carry over) must give the same result
            out2 = A.schedule_sharded(ctx, sh, req, mine.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity,
                                      ag, bufs=bufs, preempt_cap=cap, flags=flags)
            torch.cuda.synchronize()
            assert torch.equal(out.scalars, out2.scalars) and torch.equal(out.V, out2.V)
        torch.cuda.synchronize()
        sc = out.scalars.cpu().numpy().view(np.uint32).copy()
        q.put((rank, dict(sc=sc, V=out.V.cpu().numpy(), kstar=out.kstar.cpu().numpy().view(np.uint32),
                          admit=out.admit.cpu().numpy().view(np.uint32)[:sc[2]].copy(),
                          preempt=out.preempt.cpu().numpy().view(np.uint32)[:sc[3]].copy(),
                          mask=out.serve_mask.cpu().numpy()[:mine.n].copy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,cap,flags", [("config2", 16, 1), ("config2", 0xFFFFFFFF, 1 | 16),
                                            ("config3", 16, 1)])
def test_sharded_decision_two_processes(orc, name, cap, flags):
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, cap, flags, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    snap = snapshot_cached(name)
    o = oracle_decision_cached(orc, name, snap, cap=cap, flags=flags)
    mask = np.concatenate([got[r]["mask"] for r in range(world)])
    for r in range(world):
        assert_decision_equal(dict(got[r], mask=mask), o)


@pytest.mark.parametrize("name,cap,flags,world", [("config2", 16, 1, 2), ("config3", 16, 1, 2),
                                                  ("config2", 0xFFFFFFFF, 1 | 16, 3)])
def test_sharded_decision_two_processes_peer_memory(orc, name, cap, flags, world):
    """The same multi-process decision with the four exchanges done on the device by andes_comm
    (CUDA IPC: every rank stores its block into every peer's arena and publishes a flag; no host
    staging, no NCCL), compared with the oracle; two and three processes (uneven shards)."""
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, cap, flags, q, True)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    snap = snapshot_cached(name)
    o = oracle_decision_cached(orc, name, snap, cap=cap, flags=flags)
    mask = np.concatenate([got[r]["mask"] for r in range(world)])
    for r in range(world):
        assert_decision_equal(dict(got[r], mask=mask), o)
