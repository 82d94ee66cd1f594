"""N>1 host logic on CPU: world_size 2/3 gloo processes execute the product's
ring halo plan (imb_ring_plan — the exact op list the NCCL exchange issues)
with torch.distributed send/recv on host slabs, then step the padded slab
with the numpy restatement. The interior must equal the same cells of a
global periodic step (decomposition invariance), the shares come from the
product partitioner on rank 0, and timings reduce by MAX over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, l, iord, nonos, shares, q):
    import torch

    from oracle import oracle as O
    from paper_1507_01265_b200 import fpm, mpdata
    from tests import np_mpdata

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 0 decides the shares with the FPM partitioner and broadcasts them
        if shares is None:
            obj = [None]
            if rank == 0:
                xs = list(range(2, n + 1, 2))
                model = fpm.SpeedFunction(m * l, 2, tuple((x, 1e9 * (1 + 0.01 * (x % 6)))
                                                          for x in xs))
                obj = [fpm.partition_general(fpm.PartitionProblem(n, world, model)).shares]
            dist.broadcast_object_list(obj, src=0)
            shares = obj[0]
        off = mpdata.slab_offsets(shares)
        R = mpdata.step_radius(mpdata.Options(iord, nonos))
        ni = shares[rank]
        g = O.init_fields(0, n, m, l, seed=21)
        pad = np.full((ni + 2 * R, m, l), np.nan)
        pad[R:R + ni] = g[0][off[rank]:off[rank] + ni]
        reqs = []
        for kind, peer, first, planes in mpdata.ring_plan(rank, world, ni, R):
            if kind == "send":
                buf = torch.from_numpy(np.ascontiguousarray(pad[first:first + planes]))
                reqs.append(dist.isend(buf, dst=peer))
            else:
                buf = torch.empty((planes, m, l), dtype=torch.float64)
                reqs.append((dist.irecv(buf, src=peer), buf, first, planes))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                pad[r[2]:r[2] + r[3]] = r[1].numpy()
            else:
                r.wait()
        idx = (np.arange(off[rank] - R, off[rank] + ni + R)) % n
        halo_ok = bool(np.array_equal(pad, g[0][idx]))
        # step the padded window (static fields generated with wrapped halos)
        st = O.init_fields(0, n, m, l, seed=21, i0=off[rank] - R, ni=ni + 2 * R)
        local = np_mpdata.step(pad, st[1], st[2], st[3], st[4], iord=iord, nonos=nonos)[R:R + ni]
        glob = np_mpdata.step(g[0], g[1], g[2], g[3], g[4], iord=iord, nonos=nonos)
        step_ok = bool(np.array_equal(local, glob[off[rank]:off[rank] + ni]))
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, halo_ok, step_ok, float(t.item()), list(shares)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shares,iord,nonos", [
    (2, [7, 9], 2, True), (3, [5, 6, 7], 3, True), (2, [4, 12], 2, False), (3, None, 2, True)])
def test_ring_exchange_and_decomposition(world, shares, iord, nonos):
    n, m, l = 16 if shares is None else sum(shares), 6, 5
    if shares is None:
        n = 18
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, l, iord, nonos, shares, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, halo_ok, step_ok, tmax, sh in res:
        assert halo_ok, f"rank {rank}: halo planes differ from the periodic neighbours"
        assert step_ok, f"rank {rank}: slab step differs from the global step"
        assert tmax == float(world)
        assert sum(sh) == n and len(sh) == world
    assert len({tuple(r[4]) for r in res}) == 1  # every rank got rank 0's shares


def test_ring_plan_shapes():
    from paper_1507_01265_b200 import _lib, mpdata
    assert mpdata.ring_plan(0, 1, 10, 3) == [("send", 0, 3, 3), ("send", 0, 10, 3),
                                             ("recv", 0, 13, 3), ("recv", 0, 0, 3)]
    assert mpdata.ring_plan(0, 4, 8, 2)[0][1] == 3 and mpdata.ring_plan(3, 4, 8, 2)[1][1] == 0
    assert mpdata.slab_offsets([3, 5, 2]) == [0, 3, 8]
    with pytest.raises(_lib.ContractError):
        mpdata.ring_plan(0, 2, 2, 3)
