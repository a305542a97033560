"""Device rig + tangent frames (hs_rig_frames) against the reference.

Golden vectors: tests/golden/rig.npz (reference rig_evaluate + mesh_frames on a
theta batch incl. an identity pose and a large rotation, and the reference's
DegenerateTriangleError messages) and binding.npz (one more theta).  The device
computes in fp64 and stores fp32 frames, so frames agree to fp32 rounding.  The
polar quaternion is compared as stored (same branch of matrix_to_quat).  A training
step and a render driven by device frames match the same step on host frames.
"""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


class _Rig:
    def __init__(self, d, prefix="rig."):
        self.base_vertices = d[prefix + "base_vertices"]
        self.faces = d[prefix + "faces"]
        self.uv_coords = d[prefix + "uv_coords"]
        self.expr_bases = d[prefix + "expr_bases"]


def _ref_rig():
    return _Rig(golden("binding"))


def _check_frames(out, rot, quat, tri):
    out = out.cpu().numpy().astype(np.float64)
    B, F = rot.shape[:2]
    np.testing.assert_allclose(out[..., 0:9], rot.reshape(B, F, 9), rtol=2e-6, atol=2e-6 * np.abs(rot).max())
    np.testing.assert_allclose(out[..., 9:13], quat, rtol=2e-6, atol=2e-6)
    np.testing.assert_allclose(out[..., 13:22], tri.reshape(B, F, 9), rtol=2e-6, atol=2e-6 * np.abs(tri).max())


def test_rig_frames_match_reference_batch():
    from paper_2503_12886_b200.device import DeviceRig
    d = golden("rig")
    rig = DeviceRig(_ref_rig())
    th = torch.from_numpy(d["theta"].astype(np.float32)).cuda()
    out = rig.frames(th)
    # the device takes theta in fp32: compare against the reference at the fp32 theta
    # (frames are smooth in theta; the fp32 rounding of theta moves them ~1e-7)
    _check_frames(out, d["frames.rotation"], d["frames.quat"], d["frames.tri_vertices"])


def test_mesh_frames_of_vertices_match_reference():
    from paper_2503_12886_b200.device import DeviceRig
    d = golden("rig")
    rig = DeviceRig(_ref_rig())
    out = rig.frames(vertices=torch.from_numpy(d["verts"]).cuda())
    _check_frames(out, d["frames.rotation"], d["frames.quat"], d["frames.tri_vertices"])
    b = golden("binding")
    out = rig.frames(vertices=torch.from_numpy(b["verts"][None]).cuda())
    _check_frames(out, b["frames.rotation"][None], b["frames.quat"][None], b["frames.tri_vertices"][None])


def test_polar_factor_is_a_rotation():
    from paper_2503_12886_b200.device import DeviceRig
    d = golden("rig")
    rig = DeviceRig(_ref_rig())
    out = rig.frames(vertices=torch.from_numpy(d["verts"]).cuda()).cpu().numpy().astype(np.float64)
    q = out[..., 9:13]
    qn = q / np.linalg.norm(q, axis=-1, keepdims=True)
    np.testing.assert_allclose(np.linalg.norm(q, axis=-1), 1.0, atol=1e-6)   # polar factor: |q| = 1
    assert np.isfinite(qn).all()


@pytest.mark.parametrize("case", ["bad_uv", "bad_3d"])
def test_degenerate_triangles_raise_reference_message(case):
    from paper_2503_12886_b200 import _lib as L
    from paper_2503_12886_b200.device import DeviceRig
    d = golden("rig")
    r = _ref_rig()
    if case == "bad_uv":
        r.uv_coords = d["bad_uv.uv_coords"]
    else:
        r.base_vertices, r.expr_bases = d["bad_3d.base_vertices"], d["bad_3d.expr_bases"]
    rig = DeviceRig(r)
    th = torch.from_numpy(d["theta"][:1].astype(np.float32)).cuda()
    msg = str(d[f"{case}.message"])
    with pytest.raises(L.DegenerateTriangleError, match=msg + "$"):
        rig.frames(th)
    assert issubclass(L.DegenerateTriangleError, ValueError)


def test_rig_shape_errors():
    from paper_2503_12886_b200.device import DeviceRig
    rig = DeviceRig(_ref_rig())
    with pytest.raises(ValueError, match="rig expects"):
        rig.frames(torch.zeros(2, 7, device="cuda"))


def test_step_and_render_on_device_frames():
    """A Trainer holding a DeviceRig (frames=None) reproduces the step on host frames."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    import oracle as O
    wl = synth.make_workload(48, 4, 128, distinct_frames=4)
    av = wl.avatar
    mk = lambda: AvatarParams.from_host(O.GSet(*(av.base[a] for a in ("position", "rotation", "scale", "opacity",
                                                                          "color"))),
                                        av.deltas, av.mlp, av.tri_index, av.barycentric)
    th = torch.from_numpy(np.asarray(wl.thetas, np.float32)).cuda()
    tg = torch.from_numpy(wl.targets).cuda()
    fr = torch.from_numpy(wl.frames).cuda()
    cams = torch.from_numpy(np.tile(wl.camera.packed(), (4, 1))).cuda()
    bg = torch.from_numpy(np.asarray(wl.backgrounds, np.float32)).cuda()
    rig = DeviceRig(wl.rig)
    dev_frames = rig.frames(th)
    # host frames were computed from float64 theta; the device from fp32 theta
    np.testing.assert_allclose(dev_frames.cpu().numpy(), wl.frames, rtol=1e-5, atol=1e-5)
    a = Trainer(mk(), 128, 128, 4)
    b = Trainer(mk(), 128, 128, 4, rig=rig)
    ia = a.render(th, fr, cams, bg).clone()
    ib = b.render(th, None, cams, bg)
    assert float((ia - ib).abs().max()) < 1e-3
    for _ in range(2):
        a.step(th, tg, fr, cams, bg)
        b.step(th, tg, None, cams, bg)
    ra, rb = a.result(), b.result()
    assert abs(ra.loss - rb.loss) < 1e-4 * max(1.0, abs(ra.loss))
    ga, gb = a.grads.cpu().numpy(), b.grads.cpu().numpy()
    assert np.linalg.norm(ga - gb) <= 1e-2 * np.linalg.norm(ga)
    # end to end from host arrays without frames (device rig), twice: registration cache
    h = dict(thetas=np.asarray(wl.thetas, np.float32), targets=wl.targets, cameras=np.tile(wl.camera.packed(), (4, 1)),
             backgrounds=np.asarray(wl.backgrounds, np.float32))
    for _ in range(2):
        r = b.step_from_host(h["thetas"], h["targets"], None, h["cameras"], h["backgrounds"])
        assert np.isfinite(r.loss)
    b.close()


def test_compat_mesh_frames_drop_in():
    """compat.mesh_frames / rig_mesh_frames: the reference signatures (S/binding.py:67,
    S/rig.py:57) returning MeshFrames-shaped float64 arrays."""
    from paper_2503_12886_b200 import _lib as L
    from paper_2503_12886_b200 import compat
    d = golden("rig")
    rig = _ref_rig()
    rig.num_expressions = rig.expr_bases.shape[0]
    for b in (0, 2):
        mf = compat.mesh_frames(rig, d["verts"][b])
        np.testing.assert_allclose(mf.rotation, d["frames.rotation"][b], rtol=2e-6, atol=2e-6)
        np.testing.assert_allclose(mf.quat, d["frames.quat"][b], rtol=2e-6, atol=2e-6)
        mf2 = compat.rig_mesh_frames(rig, d["theta"][b])
        np.testing.assert_allclose(mf2.tri_vertices, d["frames.tri_vertices"][b], rtol=2e-6, atol=2e-6)
    bad = _ref_rig()
    bad.uv_coords = d["bad_uv.uv_coords"]
    with pytest.raises(L.DegenerateTriangleError, match=str(d["bad_uv.message"])):
        compat.mesh_frames(bad, d["verts"][0])


def test_step_from_host_prefetch_pipeline():
    """step_from_host with prefetch (double-buffered uploads) gives the same losses as
    uploads on demand, across a sequence of distinct batches."""
    from bench_support import synth
    from paper_2503_12886_b200.device import AvatarParams, DeviceRig, Trainer
    import oracle as O
    wl = synth.make_workload(40, 12, 96, distinct_frames=12)
    av = wl.avatar
    mk = lambda: Trainer(AvatarParams.from_host(O.GSet(*(av.base[a] for a in ("position", "rotation", "scale",
                                                                                   "opacity", "color"))),
                                                av.deltas, av.mlp, av.tri_index, av.barycentric), 96, 96, 4,
                         rig=DeviceRig(wl.rig))
    cams = np.tile(wl.camera.packed(), (4, 1))
    th = np.asarray(wl.thetas, np.float32)
    bg = np.asarray(wl.backgrounds, np.float32)
    batches = [(np.ascontiguousarray(th[i:i + 4]), np.ascontiguousarray(wl.targets[i:i + 4]), None, cams,
                np.ascontiguousarray(bg[i:i + 4])) for i in (0, 4, 8, 0)]
    a, b = mk(), mk()
    la = [a.step_from_host(*x).loss for x in batches]
    lb = [b.step_from_host(*x, prefetch=batches[i + 1] if i + 1 < len(batches) else None).loss
          for i, x in enumerate(batches)]
    np.testing.assert_allclose(lb, la, rtol=1e-6)
    # step_from_host returns at the loss read; the backward and Adam finish later, and the
    # prefetch into a buffer set waits for the step that last read it: the same parameters
    # up to the order of the raster's gradient atomics: Adam turns it into a fraction of
    # a step on near-zero gradients, and colour init can flip on a threshold -- a handful
    # of entries; a clobbered buffer set would change whole gradients
    torch.cuda.synchronize()
    pa, pb = a.av.params.cpu().numpy(), b.av.params.cpu().numpy()
    off = np.abs(pb - pa) > 5e-5 + 1e-3 * np.abs(pa)
    assert off.mean() < 1e-4, (int(off.sum()), pa.size)
    a.close()
    b.close()
