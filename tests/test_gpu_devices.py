"""Device handling of the blocking entry points: per-device kernel setup
(the shared-memory opt-in is a per-device-context attribute), the caller's
current device survives every call, and the workspace release entry point."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_kernel_setup_is_per_device_and_once(fb, restatement):
    v, c = fb.structured_mesh(3, 4, 0.15, 42)
    # an instantiation no other test uses first: weighted 3D f64 fast, direct stores
    var = fb.make_variant("weighted-laplacian", 3, "f64", "fast", store="direct")
    w = np.ascontiguousarray(1.0 + np.arange(c.size, dtype=np.float64) % 3)
    s0 = fb.kernel_setups(0)
    fb.integrate_mesh(var, v, c, coefficients=w, devices=[0])
    s1 = fb.kernel_setups(0)
    assert s1 >= s0 + 1 or s0 > 0  # set up on device 0 on first use
    # a device list naming the same device again does not set it up again
    fb.integrate_mesh(var, v, c, coefficients=w, devices=[0, 0, 0])
    assert fb.kernel_setups(0) == s1
    for d in range(torch.cuda.device_count(), 64):
        assert fb.kernel_setups(d) == 0  # no device that does not exist was touched
    assert fb.kernel_setups(64) == -1 and fb.kernel_setups(-1) == -1


def test_blocking_calls_keep_the_callers_device(fb):
    v, c = fb.structured_mesh(2, 16, 0.15, 42)
    var = fb.make_variant("laplacian", 2, "f32")
    ndev = torch.cuda.device_count()
    for dev in range(ndev):
        torch.cuda.set_device(dev)
        for target in range(ndev):
            fb.integrate_mesh(var, v, c, devices=[target])
            fb.pack_geometry(v, c, 2, 128, "f32", devices=[target])
            assert torch.cuda.current_device() == dev
    torch.cuda.set_device(0)


def test_release_workspace_then_reuse(fb, restatement):
    v, c = fb.structured_mesh(2, 20, 0.15, 42)
    var = fb.make_variant("elasticity", 2, "f64")
    want = restatement.integrate_mesh("elasticity", v, c, 2, bs=128, precision="f64")
    assert fb.integrate_mesh(var, v, c).tobytes() == want.tobytes()  # host-staged: workspace in use
    fb.release_workspace(0)
    fb.release_workspace(-1)  # idempotent
    assert fb.integrate_mesh(var, v, c).tobytes() == want.tobytes()  # workspace re-created


def test_torch_dtype_mismatch_is_rejected(fb):
    v, c = fb.structured_mesh(2, 8, 0.0, 42)
    var = fb.make_variant("laplacian", 2, "f32")
    dv, dc = torch.from_numpy(v).cuda(), torch.from_numpy(c).cuda()
    with pytest.raises(fb.engine.L.InvalidArgument, match="cells has dtype int64"):
        fb.integrate_mesh(var, dv, dc.long())
    with pytest.raises(fb.engine.L.InvalidArgument, match="vertices has dtype float32"):
        fb.integrate_mesh(var, dv.float(), dc)
    out = torch.empty(var.store_length(c.size // 3), dtype=torch.float64, device="cuda")
    with pytest.raises(fb.engine.L.InvalidArgument, match="out has dtype float64"):
        fb.integrate_mesh(var, dv, dc, out=out)
