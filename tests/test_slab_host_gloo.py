"""Multi-process (world size 2, gloo, CPU) tests of the z-slab decomposition's
host logic: global grid by all-reduce, work histogram -> identical partition
on every rank (apbf_slab_partition, pure host code in libapbf_gpu.so), and
the invariant the GPU path relies on for bit-exactness: concatenating what a
rank receives in source-rank order and stable-sorting by global cell gives
the global stable cell order restricted to the rank's extended slab."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

H = np.float32(0.05)
HALO = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def cells(p, origin, dims):
    c = np.floor((p - origin) / H).astype(np.int64)
    c = np.clip(c, 0, dims - 1)
    return (c[:, 2] * dims[1] + c[:, 1]) * dims[0] + c[:, 0], c[:, 2]


def global_grid(lo, hi):
    origin = (lo - H).astype(np.float32)
    top = (hi + H).astype(np.float32)
    dims = np.maximum(1, np.floor((top - origin) / H).astype(np.int64) + 1)
    return origin, dims


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1608_04721_b200.slab import slab_partition
    rng = np.random.default_rng(5)
    N = 3000
    cloud = np.empty((N, 3), np.float32)
    cloud[:, 0] = rng.uniform(0, 0.6, N)
    cloud[:, 1] = rng.uniform(0, 0.3, N)
    cloud[:, 2] = rng.uniform(0, 1.5, N) ** 1.3  # uneven along the slab axis
    levels = rng.integers(3, 8, N).astype(np.int64)
    b, e = N * rank // world, N * (rank + 1) // world
    mine, mylv = cloud[b:e], levels[b:e]
    # global grid: AABB all-reduce
    lo = torch.from_numpy(mine.min(0).copy())
    hi = torch.from_numpy(mine.max(0).copy())
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    origin, dims = global_grid(lo.numpy(), hi.numpy())
    cid, cz = cells(mine, origin, dims)
    # work histogram (1 + level per particle) -> partition, identical everywhere
    hist = np.zeros(dims[2], np.int64)
    np.add.at(hist, cz, 1 + mylv)
    ht = torch.from_numpy(hist)
    dist.all_reduce(ht)
    part = slab_partition(ht.numpy(), world, HALO)
    assert part is not None
    zlo, zhi = part
    # migration + halo: send every particle whose layer is in q's extended slab
    send = [np.nonzero((cz >= zlo[q] - HALO) & (cz < zhi[q] + HALO))[0] for q in range(world)]
    payload = [(mine[idx], mylv[idx], (b + idx)) for idx in send]
    gathered = [None] * world
    dist.all_gather_object(gathered, payload)
    recv = [gathered[q][rank] for q in range(world)]  # in source-rank order
    pos = np.concatenate([r[0] for r in recv])
    gid = np.concatenate([r[2] for r in recv])
    lcid, lcz = cells(pos, origin, dims)
    local_order = gid[np.argsort(lcid, kind="stable")]
    np.save(os.path.join(out_dir, f"rank{rank}.npy"),
            np.array([zlo, zhi], dtype=np.int64))
    np.save(os.path.join(out_dir, f"order{rank}.npy"), local_order)
    np.save(os.path.join(out_dir, f"grid{rank}.npy"), np.concatenate([origin, dims.astype(np.float32)]))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_decomposition_reproduces_global_order():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npy")) for r in range(world)]
        assert np.array_equal(parts[0], parts[1])  # identical partition on every rank
        zlo, zhi = parts[0]
        assert zlo[0] == 0 and zhi[-1] > zhi[0] and zlo[1] == zhi[0]
        assert (zhi - zlo >= HALO).all()
        grids = [np.load(os.path.join(d, f"grid{r}.npy")) for r in range(world)]
        assert np.array_equal(grids[0], grids[1])
        # the global reference order, restricted to each rank's extended slab
        rng = np.random.default_rng(5)
        N = 3000
        cloud = np.empty((N, 3), np.float32)
        cloud[:, 0] = rng.uniform(0, 0.6, N)
        cloud[:, 1] = rng.uniform(0, 0.3, N)
        cloud[:, 2] = rng.uniform(0, 1.5, N) ** 1.3
        origin, dims = grids[0][:3], grids[0][3:].astype(np.int64)
        gcid, gcz = cells(cloud, origin, dims)
        gorder = np.argsort(gcid, kind="stable")
        for r in range(world):
            sel = gorder[(gcz[gorder] >= zlo[r] - HALO) & (gcz[gorder] < zhi[r] + HALO)]
            assert np.array_equal(np.load(os.path.join(d, f"order{r}.npy")), sel)


def test_partition_balances_work_and_keeps_min_thickness():
    from paper_1608_04721_b200.slab import slab_partition
    hist = np.r_[np.zeros(5), np.full(30, 100), np.full(30, 10)].astype(np.int64)
    lo, hi = slab_partition(hist, 4, 2)
    assert lo[0] == 0 and hi[-1] == hist.shape[0]
    assert np.array_equal(lo[1:], hi[:-1]) and ((hi - lo) >= 2).all()
    work = [hist[a:b].sum() for a, b in zip(lo, hi)]
    assert max(work) <= 1.25 * hist.sum() / 4 + hist.max()
    assert slab_partition(np.ones(5, np.int64), 3, 2) is None
