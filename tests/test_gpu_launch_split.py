"""Launch splitting (the kernels index slots with 32-bit locals; the host
splits launches at 2^30 slots): with FB_TEST_MAX_LAUNCH_SLOTS lowering the
split, every integration path runs as many launches with slot offsets and
must give the same bits as the oracle.  Runs in a subprocess so the
environment hook is read at library load."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1103_0066_b200 as fb
from oracle.oracle import Restatement
ora = Restatement()
n0 = fb.launch_counter()
for op, dim, n, prec in (("elasticity", 2, 20, "f32"), ("laplacian", 3, 8, "f64"), ("weighted-laplacian", 3, 6, "f32")):
    v, c = fb.structured_mesh(dim, n, 0.15, 42)
    ne = c.size // (dim + 1)
    w = None
    if op == "weighted-laplacian":
        w = np.ascontiguousarray(1.0 + v.reshape(-1, dim)[c.reshape(-1, dim + 1), 0].ravel())
    var = fb.make_variant(op, dim, prec, "strict", element_batch_size=128)
    want = ora.integrate_mesh(op, v, c, dim, bs=128, precision=prec, coeffs=w)
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    dw = None if w is None else torch.from_numpy(w).cuda()
    out = torch.empty(var.store_length(ne), dtype=torch.float32 if prec == "f32" else torch.float64, device="cuda")
    st = torch.empty(2, dtype=torch.int64, device="cuda")
    sid = torch.cuda.current_stream().cuda_stream
    fb.status_reset(st, sid)
    fb.integrate_mesh_async(var, dv, dc, out, st, sid, coefficients=dw)
    fb.status_check(st, sid)
    assert out.cpu().numpy().tobytes() == want.tobytes(), (op, dim, prec)
    g = torch.empty(var.store_length(ne) // var.spec.krows ** 2 * dim * dim, dtype=out.dtype, device="cuda")
    fb.pack_geometry_async(dv, dc, dim, g, st, 128, prec, sid)
    fb.status_check(st, sid)
    assert g.cpu().numpy().tobytes() == ora.pack_geometry(v, c, dim, 128, prec).tobytes()
    out2 = torch.empty_like(out)
    fb.integrate_packed_async(var, g, ne, out2, sid, coefficients=dw)
    torch.cuda.synchronize()
    assert out2.cpu().numpy().tobytes() == want.tobytes(), ("packed", op, dim, prec)
    # the blocking pack_geometry splits its device-resident launch the same way
    k0 = fb.launch_counter()
    g2 = fb.pack_geometry(dv, dc, dim, 128, prec)
    torch.cuda.synchronize()
    assert fb.launch_counter() - k0 > 1, "blocking pack_geometry was not split"
    assert g2.cpu().numpy().tobytes() == g.cpu().numpy().tobytes()
print("launches", fb.launch_counter() - n0)
'''


def test_split_launches_are_bitwise_equal():
    env = dict(os.environ, FB_TEST_MAX_LAUNCH_SLOTS="256")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    launches = int(r.stdout.split("launches")[-1])
    assert launches > 3 * 3 * 4  # every path ran as several launches
