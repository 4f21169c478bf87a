"""Multi-rank sharding (gloo, world_size 2): the engine's own element-range
split (fb_shard_bounds, the function run_job uses for a device list) gives
contiguous tile-aligned shards that integrate independently and concatenate
to the single-device store bitwise -- the property that lets the GPU path
shard over 8 B200s with no collective.  On CPU the
shards are integrated with the oracle restatement; the gpu-marked variant
integrates each rank's shard with the CUDA engine (both ranks on cuda:0)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1103_0066_b200 as fb

TILE = 288  # fbk::kTile (csrc/fb_internal.h)


def test_shard_bounds_cover_and_align():
    for nslots in (0, 1, 287, 288, 289, 10_000, 1 << 20, 1 << 34):
        for parts in (1, 2, 3, 8):
            b = fb.shard_bounds(nslots, parts)
            assert b[0] == 0 and b[-1] == nslots and len(b) == parts + 1
            assert all(x <= y for x, y in zip(b, b[1:]))
            assert all(x % TILE == 0 for x in b[:-1])
            if nslots >= TILE * parts:  # balanced to within one tile
                sizes = [y - x for x, y in zip(b, b[1:])]
                assert max(sizes) - min(sizes) <= TILE


def test_shard_bounds_rejects_bad_counts():
    with pytest.raises(fb.engine.L.InvalidArgument, match="worker count"):
        fb.shard_bounds(100, 0)
    with pytest.raises(fb.engine.L.InvalidArgument):
        fb.shard_bounds(-1, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, op, dim, bs, prec, q, on_gpu=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Restatement

        import paper_1103_0066_b200 as fb

        ora = Restatement()
        v, c, _ = fb.mesh_prefix(dim, 5000, 0.15, 42)
        nb = dim + 1
        ne = c.size // nb
        nslots = -(-ne // bs) * bs
        full = ora.integrate_mesh(op, v, c, dim, bs=bs, precision=prec)
        nk = full.size // nslots
        b = fb.shard_bounds(nslots, world)
        s0, s1 = b[rank], b[rank + 1]
        # the shard: slots [s0, s1); padding slots replicate element ne-1
        ids = np.minimum(np.arange(s0, s1), ne - 1)
        cs = np.ascontiguousarray(c.reshape(-1, nb)[ids].ravel())
        if on_gpu:
            var = fb.make_variant(op, dim, "f32" if prec == 0 else "f64", "strict", element_batch_size=1)
            part = fb.integrate_mesh(var, torch.from_numpy(v).cuda(), torch.from_numpy(cs).cuda()).cpu().numpy()
            assert fb.kernel_setups(0) > 0  # the kernel was set up on this rank's device
        else:
            part = ora.integrate_mesh(op, v, cs, dim, bs=1, precision=prec)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([part.size]))
        n = int(max(x.item() for x in sizes))
        buf = torch.zeros(n, dtype=torch.float64)
        buf[: part.size] = torch.from_numpy(part.astype(np.float64))
        gathered = [torch.zeros(n, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, buf)
        if rank == 0:
            cat = np.concatenate([g[: int(s.item())].numpy() for g, s in zip(gathered, sizes)])
            q.put(bool(cat.size == nk * nslots and
                       cat.astype(full.dtype).tobytes() == full.tobytes()))
    finally:
        dist.destroy_process_group()


def _run_two_ranks(op, dim, bs, prec, on_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, op, dim, bs, prec, q, on_gpu)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("op,dim,bs,prec", [("elasticity", 2, 128, 0), ("laplacian", 3, 7, 1)])
def test_gloo_two_rank_shards_concatenate_bitwise(op, dim, bs, prec):
    _run_two_ranks(op, dim, bs, prec, on_gpu=False)


@pytest.mark.gpu
@pytest.mark.parametrize("op,dim,bs,prec", [("elasticity", 3, 128, 0), ("laplacian", 2, 5, 1)])
def test_gloo_two_rank_engine_shards_concatenate_bitwise(op, dim, bs, prec):
    """Each rank integrates its engine-split shard with the CUDA engine."""
    _run_two_ranks(op, dim, bs, prec, on_gpu=True)
