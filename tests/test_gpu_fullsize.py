"""Parity at the BASELINE.json configuration sizes.

* 2D P1 elasticity, 1,048,576 elements (configs[1]), f32 and f64, strict:
  the whole store bitwise against the oracle restatement.
* 2D P1 Laplacian, 65,536 elements (configs[0]): bitwise + normwise vs the
  FP64 direct-quadrature oracle on every element, fast mode within tolerance.
* 3D P1 Laplacian, 16,777,216 elements (configs[2]) and one 8,388,608-element
  shard of 3D elasticity-64M (configs[3]): the WHOLE store bitwise against
  the oracle restatement (chunks of 2^21 elements), and size-independent
  properties over the full store on the device: symmetry, zero row sums
  (constants in the null space), elasticity's zero off-diagonal component
  blocks and 0.25-scaled Laplacian diagonal blocks, bitwise.
* >= 1M elements bitwise against the reference build itself (oracle/_ref:
  the unmodified pack_geometry + integrate_batches, src/geometry.cpp:312-351,
  src/engine.cpp:339-376), not only against the restatement.
"""
import numpy as np
import pytest
import torch

import paper_1103_0066_b200 as fb
from oracle.oracle import krows, normwise_error

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _sample(ne):  # fast-mode tolerance checks against the FP64 direct oracle
    idx = np.concatenate([np.arange(min(4096, ne)), np.arange(0, ne, 4096), np.arange(max(0, ne - 4096), ne)])
    return np.unique(idx)


def _device_mesh(dim, ne, jitter):
    v, c, _ = fb.mesh_prefix(dim, ne, jitter, 42)
    return v, c, torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_2d_elasticity_1m_bitwise(restatement, prec):
    v, c, dv, dc = _device_mesh(2, 1 << 20, 0.15)
    var = fb.make_variant("elasticity", 2, prec)
    got = fb.integrate_mesh(var, dv, dc).cpu().numpy()
    want = restatement.integrate_mesh("elasticity", v, c, 2, bs=128, precision=prec)
    assert got.tobytes() == want.tobytes()


def test_2d_laplacian_64k_against_direct_oracle(restatement):
    v, c, dv, dc = _device_mesh(2, 1 << 16, 0.15)
    ne = c.size // 3
    direct = restatement.direct_mesh("laplacian", v, c, 2)
    for prec, tol in (("f64", 1e-13), ("f32", 5e-6)):
        for mode in ("strict", "fast"):
            got = fb.integrate_mesh(fb.make_variant("laplacian", 2, prec, mode), dv, dc).cpu().numpy()
            a = got[: ne * 9].reshape(ne, 3, 3).transpose(0, 2, 1)
            assert normwise_error(a, direct) <= tol
            if mode == "strict":
                want = restatement.integrate_mesh("laplacian", v, c, 2, bs=128, precision=prec)
                assert got.tobytes() == want.tobytes()


def _properties(store, op, dim, ne):
    kr = krows(op, dim)
    nb = dim + 1
    m = store[: ne * kr * kr].view(ne, kr, kr).transpose(1, 2)  # [e][i][j]
    assert torch.equal(m, m.transpose(1, 2)), "not bitwise symmetric"
    if op == "elasticity":
        blocks = m.view(ne, dim, nb, dim, nb)  # [e][c][a][d][b]
        lap = blocks[:, 0, :, 0, :]
        for c in range(dim):
            for d in range(dim):
                blk = blocks[:, c, :, d, :]
                if c == d:
                    assert torch.equal(blk, lap)
                else:
                    assert torch.count_nonzero(blk).item() == 0
        m = lap
    scale = m.abs().amax(dim=(1, 2))
    rows = m.double().sum(dim=2).abs().amax(dim=1)
    tol = 1e-5 if store.dtype == torch.float32 else 1e-13
    assert (rows <= tol * scale.double()).all().item(), "row sums are not ~0"


@pytest.mark.parametrize("op,dim,ne,jitter,prec", [
    ("laplacian", 3, 1 << 24, 0.15, "f32"),
    ("laplacian", 3, 1 << 24, 0.15, "f64"),
    ("elasticity", 3, 1 << 23, 0.0, "f32"),
    ("elasticity", 3, 1 << 23, 0.0, "f64"),
])
def test_large_3d_full_store_bitwise_and_properties(restatement, op, dim, ne, jitter, prec):
    v, c, dv, dc = _device_mesh(dim, ne, jitter)
    var = fb.make_variant(op, dim, prec)
    store = fb.integrate_mesh(var, dv, dc)
    torch.cuda.synchronize()
    _properties(store, op, dim, ne)
    kr2 = krows(op, dim) ** 2
    nb = dim + 1
    chunk = 1 << 21
    for e0 in range(0, ne, chunk):
        e1 = min(ne, e0 + chunk)
        cs = np.ascontiguousarray(c[e0 * nb:e1 * nb])
        want = restatement.integrate_mesh(op, v, cs, dim, bs=1, precision=prec)
        got = store[e0 * kr2:e1 * kr2].cpu().numpy()
        assert got.tobytes() == want.tobytes(), f"elements [{e0}, {e1}) differ"
    assert store.numel() == ne * kr2  # 2^k elements: no padding slots


@pytest.mark.parametrize("op,dim,ne,jitter,prec", [
    ("laplacian", 3, 1 << 21, 0.15, "f32"),
    ("elasticity", 2, 1 << 20, 0.15, "f64"),
    ("elasticity", 3, (1 << 20) + 77, 0.15, "f32"),
])
def test_million_elements_bitwise_against_reference_build(reference, op, dim, ne, jitter, prec):
    """The GPU store equals the unmodified reference engine's store (its own
    pack_geometry + integrate_batches, all host threads) bit for bit,
    padding slots included."""
    import os

    v, c, dv, dc = _device_mesh(dim, ne, jitter)
    got = fb.integrate_mesh(fb.make_variant(op, dim, prec), dv, dc).cpu().numpy()
    want = reference.integrate_mesh(op, v, c, dim, bs=128, ce=2, interleave=True, precision=prec,
                                    workers=os.cpu_count() or 1)
    assert got.size == want.size
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("op,dim,ne,prec,tol", [
    ("laplacian", 3, 1 << 24, "f32", 5e-6),
    ("elasticity", 2, 1 << 20, "f64", 1e-13),
])
def test_fast_mode_at_size_against_direct_oracle(restatement, op, dim, ne, prec, tol):
    """Fast mode (FMA, one reciprocal of det) at a BASELINE size: sampled
    elements within the stated normwise tolerance of the FP64 direct oracle."""
    v, c, dv, dc = _device_mesh(dim, ne, 0.15)
    store = fb.integrate_mesh(fb.make_variant(op, dim, prec, "fast"), dv, dc)
    kr = krows(op, dim)
    idx = _sample(ne)
    got = store.view(-1, kr * kr)[torch.from_numpy(idx).cuda()].cpu().numpy()
    a = got.reshape(-1, kr, kr).transpose(0, 2, 1)
    direct = restatement.direct_mesh(op, v, c, dim, elements=idx)
    assert normwise_error(a, direct) <= tol


def test_store_beyond_2_31_scalars_bitwise_at_the_tail(restatement):
    """3D elasticity f32 with 2^24 + 5 elements: a 2.42 G-scalar store (past
    the int32 index range; element offsets are 64-bit), ragged last tile and
    padded last batch.  The first and last 4096 elements and every 65536th
    in between are bitwise the restatement's."""
    op, dim, ne = "elasticity", 3, (1 << 24) + 5
    v, c, _ = fb.mesh_prefix(dim, ne, 0.0, 42)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    var = fb.make_variant(op, dim, "f32")
    store = fb.integrate_mesh(var, dv, dc)
    kr2 = krows(op, dim) ** 2
    assert store.numel() == var.store_length(ne) and store.numel() > (1 << 31)
    idx = np.unique(np.concatenate([np.arange(4096), np.arange(0, ne, 65536), np.arange(ne - 4096, ne)]))
    cs = np.ascontiguousarray(c.reshape(-1, dim + 1)[idx].ravel())
    want = restatement.integrate_mesh(op, v, cs, dim, bs=1, precision="f32").reshape(-1, kr2)
    got = store.view(-1, kr2)[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert got.tobytes() == want.tobytes()
    # padding slots (ne .. num_batches*bs) replicate the last element
    pad = store.view(-1, kr2)[ne:].cpu().numpy()
    assert pad.shape[0] == var.store_length(ne) // kr2 - ne and pad.shape[0] > 0
    assert all(p.tobytes() == want[-1].tobytes() for p in pad)
