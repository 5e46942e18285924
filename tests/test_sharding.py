"""Multi-process (gloo, world_size 2, CPU) tests of the signal-sharding host logic:
contiguous shards, and the gather of per-rank results back to rank 0 in global trial order.
The per-rank work is stood in for by a deterministic function of the trial index (no GPU here)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_07407_b200.shard import gather_to_rank0, shard_indices, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 1024, 1025):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, world, r)
                assert 0 <= hi - lo <= -(-n // world)
                seen += list(range(lo, hi))
            assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_solve(trials, k, d):
    """Stand-in for a rank's solves: outputs are a pure function of the trial index."""
    t = torch.tensor(trials, dtype=torch.int64)
    freqs = (t[:, None, None] * 1000 + torch.arange(k)[None, :, None] * 10 + torch.arange(d)[None, None, :]).to(torch.int32)
    coeffs = torch.stack([t.double() + 0.5, -t.double()], -1)[:, None, :].expand(len(trials), k, 2).contiguous()
    count = torch.full((len(trials),), k, dtype=torch.int32)
    return freqs, coeffs, count


def _worker(rank, world, port, n, k, d, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard_indices(n, world, rank)
        outs = _fake_solve(mine, k, d)
        got = gather_to_rank0(list(outs), n, world, rank)
        if rank == 0:
            ref = _fake_solve(list(range(n)), k, d)
            ok = all(torch.equal(a, b) for a, b in zip(got, ref))
            q.put(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 7])
def test_gather_world2_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 3, 4, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


# ------------------------------------------------------------------ line sharding host logic
def test_line_shard_ranges_partition_axes():
    """sfft_line_shard_range (C ABI, host): contiguous, disjoint, covering [0, r), sizes within one, shard 0
    the largest (its line count fixes the tile shapes of every shard); G > r is rejected."""
    import paper_1606_07407_b200 as S
    for r in (1, 2, 3, 10, 20, 50, 500):
        for G in (1, 2, 3, 4, 7, 8):
            if G > r:
                with pytest.raises(S.SfftError):
                    S.sfft_line_shard_range(r, G, 0)
                continue
            rs = [S.sfft_line_shard_range(r, G, g) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == r
            assert all(rs[g][1] == rs[g + 1][0] for g in range(G - 1))
            sizes = [hi - lo for lo, hi in rs]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1 and sizes[0] == max(sizes)


def _line_worker(rank, world, port, r, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1606_07407_b200 as S
        # the communicator bootstrap of comm_init_line_shards: rank 0 draws the NCCL id, the group broadcasts it
        obj = [S.sfft_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        shards = [None] * world
        dist.all_gather_object(shards, S.sfft_line_shard_range(r, world, rank))
        if rank == 0:
            axes = [a for lo, hi in shards for a in range(lo, hi)]
            q.put(len(obj[0]) == 128 and all(i == ids[0] for i in ids) and axes == list(range(r)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("r", [2, 51])
def test_line_shard_bootstrap_world2_gloo(r):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_line_worker, args=(rk, 2, port, r, q)) for rk in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def _peer_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1606_07407_b200 as S
        # the handle exchange of comm_init_line_shards(exchange=1): every rank contributes its 64-byte CUDA IPC
        # handle, every rank receives all of them in rank order (stand-in bytes here: no GPU)
        mine = bytes([rank + 1]) * 64
        got = S.exchange_handles(mine)
        q.put((rank, got == [bytes([g + 1]) * 64 for g in range(world)]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_handle_exchange_world2_gloo():
    """Fused record exchange bootstrap (line_exchange = 1): the all-gather of the ranks' IPC handles."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(rk, 2, port, q)) for rk in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
