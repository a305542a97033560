"""The host-side workload generators (paper_2503_12886_b200/synth.py) reproduce the
reference's rig, UV binding, mesh frames and init (golden vectors from the reference)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from bench_support import synth


def test_rig_matches_reference():
    d = golden("binding")
    rig = synth.build_head_rig()
    assert np.array_equal(rig.base_vertices, d["rig.base_vertices"])
    assert np.array_equal(rig.faces, d["rig.faces"])
    assert np.array_equal(rig.uv_coords, d["rig.uv_coords"])
    assert np.array_equal(rig.expr_bases, d["rig.expr_bases"])
    np.testing.assert_allclose(synth.rig_evaluate(rig, d["theta"]), d["verts"], rtol=0, atol=1e-14)


def test_bindings_and_frames_match_reference():
    d = golden("binding")
    rig = synth.build_head_rig()
    tri, bary = synth.bind_gaussians(rig, 24)
    assert np.array_equal(tri, d["tri_index"])
    assert np.array_equal(bary, d["barycentric"])
    mf = synth.mesh_frames(rig, synth.rig_evaluate(rig, d["theta"]))
    np.testing.assert_allclose(mf.rotation, d["frames.rotation"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(mf.quat, d["frames.quat"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(mf.tri_vertices, d["frames.tri_vertices"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("uv", [141, 224])
def test_config_gaussian_counts_and_checksums(uv):
    counts = json.load(open(os.path.join(GOLDEN, "counts.json")))
    tri, bary = synth.bind_gaussians(synth.build_head_rig(), uv)
    assert tri.shape[0] == counts[f"uv{uv}"]
    assert synth.bindings_checksum(tri, bary) == counts[f"uv{uv}_checksum"]


def test_init_avatar_matches_reference_train_fixture():
    d = golden("train")
    av = synth.init_avatar(synth.build_head_rig(), uv_resolution=20, num_blendshapes=4, hidden_dim=16)
    assert np.array_equal(av.tri_index, d["tri_index"])
    np.testing.assert_array_equal(av.base["scale"], d["base0.scale"])
    for k in ("w1", "w2", "b1"):
        np.testing.assert_array_equal(av.mlp[k], d["mlp0." + k])


def test_rig_batch_matches_reference():
    """rig.npz: identity pose, large rotation and strong expressions (S/rig.py:57-66,
    S/binding.py:67-115) -- the restatement the device rig is also checked against."""
    d = golden("rig")
    rig = synth.build_head_rig()
    for b, th in enumerate(d["theta"]):
        v = synth.rig_evaluate(rig, th)
        np.testing.assert_allclose(v, d["verts"][b], rtol=0, atol=1e-13)
        mf = synth.mesh_frames(rig, v)
        np.testing.assert_allclose(mf.rotation, d["frames.rotation"][b], rtol=0, atol=1e-12)
        np.testing.assert_allclose(mf.quat, d["frames.quat"][b], rtol=0, atol=1e-11)
        np.testing.assert_allclose(mf.tri_vertices, d["frames.tri_vertices"][b], rtol=0, atol=1e-13)
