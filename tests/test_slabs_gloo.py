"""N > 1 path on CPU: world-size-2 gloo processes run bench.py's rank logic
(slab partition, MAX over ranks of the device time, final slab gather)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1704_08364_b200 import slabs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, e = slabs.rank_slab(n, world, rank)
        # every rank sees the same partition: disjoint, ordered, covering
        got = [None] * world
        dist.all_gather_object(got, (b, e))
        assert got == slabs.split(n, world)
        # job time = max of the per-rank times
        t = slabs.max_over_ranks(10.0 + rank)
        assert t == 10.0 + world - 1
        # each rank "reconstructs" its slab (slice index stamped in); rank 0
        # gathers the volume
        local = torch.arange(b, e, dtype=torch.float32)[:, None, None].expand(e - b, 3, 3).contiguous()
        vol = slabs.gather_slabs(local, n)
        if rank == 0:
            torch.save(vol, os.path.join(out_dir, "vol.pt"))
        else:
            assert vol is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 2048])
def test_two_rank_slab_sharding(tmp_path, n):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    vol = torch.load(tmp_path / "vol.pt")
    assert vol.shape == (n, 3, 3)
    assert torch.equal(vol[:, 0, 0], torch.arange(n, dtype=torch.float32))


def test_split_properties():
    for n in (0, 1, 5, 2048):
        for parts in (1, 2, 3, 8):
            sl = slabs.split(n, parts)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [e - b for b, e in sl]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slabs.rank_slab(4, 2, 2)
