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


def _recon_worker(rank, world, port, out_dir, use_gpu):
    """Each rank reconstructs its z-slab of a small sinogram volume and rank 0
    gathers the image volume (the bench's N > 1 data flow with real work)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        from oracle import bst_oracle as O
        S, N = 7, 32
        rng = np.random.default_rng(11)
        vol = np.stack([O.ellipse_sinogram(O.SHEPP_LOGAN, N, N) for _ in range(S)])
        vol = vol + 0.05 * rng.standard_normal(vol.shape)
        b, e = slabs.rank_slab(S, world, rank)
        if use_gpu:
            from paper_1704_08364_b200 import fourier_bp as F
            torch.cuda.set_device(0)
            sino = torch.from_numpy(vol[b:e].astype(np.float32)).cuda()
            local = F.fbp_volume(sino, F.BstPlan(N, N)).cpu()
        else:
            local = torch.from_numpy(O.fbp_volume(vol[b:e], O.OraclePlan(N, N)))
        got = slabs.gather_slabs(local.contiguous(), S)
        if rank == 0:
            torch.save((got, torch.from_numpy(vol)), os.path.join(out_dir, "recon.pt"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_reconstruction_oracle(tmp_path):
    """world size 2 on CPU: the slabs each rank reconstructs (oracle
    restatement), gathered on rank 0, equal the single-process volume."""
    import numpy as np
    from oracle import bst_oracle as O
    mp.spawn(_recon_worker, args=(2, _free_port(), str(tmp_path), False), nprocs=2, join=True)
    got, vol = torch.load(tmp_path / "recon.pt")
    ref = O.fbp_volume(vol.numpy(), O.OraclePlan(32, 32))
    assert got.shape == (7, 32, 32)
    assert np.array_equal(got.numpy(), ref)


@pytest.mark.gpu
def test_two_rank_slab_reconstruction_gpu(tmp_path):
    """Two gloo ranks sharing GPU 0, each running the CUDA path on its slab:
    the gathered volume is bitwise the single-process fbp_volume."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1704_08364_b200 import fourier_bp as F
    mp.spawn(_recon_worker, args=(2, _free_port(), str(tmp_path), True), nprocs=2, join=True)
    got, vol = torch.load(tmp_path / "recon.pt")
    one = F.fbp_volume(vol.float().cuda(), F.BstPlan(32, 32)).cpu()
    assert torch.equal(got, one)
