"""Model file + sequence loading (paper_2503_12886_b200/io.py) against the reference
(S/model_io.py, S/dataset.py:175-275; golden io.npz written by the reference)."""
import json

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2503_12886_b200 import io as hio

ATTRS = ("position", "rotation", "scale", "opacity", "color")


class _HostAvatar:
    """Duck-typed AvatarParams over host arrays (what save_model reads)."""

    def __init__(self, d):
        self.N = d["model.tri_index"].shape[0]
        self.K = d["model.deltas"].shape[0]
        self.D, self.H = d["model.mlp.w1"].shape
        self._d = d
        self.tri_index = torch.from_numpy(d["model.tri_index"].astype(np.int32))
        self.barycentric = torch.from_numpy(d["model.barycentric"].astype(np.float32))

    def split_host(self):
        d = self._d
        return ({a: d[f"model.base.{a}"] for a in ATTRS}, d["model.deltas"],
                {k: d[f"model.mlp.{k}"] for k in ("w1", "b1", "w2", "b2", "w3", "b3")})


def test_load_reference_model_file(tmp_path):
    d = golden("io")
    p = tmp_path / "m.bin"
    p.write_bytes(d["model.bytes"].tobytes())
    m = hio.load_model(p)
    for a in ATTRS:
        np.testing.assert_array_equal(m.base[a], d[f"model.base.{a}"].astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(m.deltas, d["model.deltas"].astype(np.float32).astype(np.float64))
    for k in ("w1", "b1", "w2", "b2", "w3", "b3"):
        np.testing.assert_array_equal(m.mlp[k], d[f"model.mlp.{k}"].astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(m.tri_index, d["model.tri_index"])
    np.testing.assert_array_equal(m.visited, d["model.visited"])


def test_save_is_byte_identical_to_reference(tmp_path):
    d = golden("io")
    p = tmp_path / "ours.bin"
    hio.save_model(_HostAvatar(d), torch.from_numpy(d["model.visited"].astype(np.uint8)), p)
    assert p.read_bytes() == d["model.bytes"].tobytes()


def test_model_file_errors(tmp_path):
    d = golden("io")
    raw = d["model.bytes"].tobytes()
    cases = {"short": (raw[:10], "file truncated before header"),
             "magic": (b"XXXX" + raw[4:], "bad magic"),
             "version": (raw[:4] + (2).to_bytes(4, "little") + raw[8:], "unsupported version 2"),
             "trunc": (raw[:-200], "file truncated at offset"),
             "trailing": (raw + b"\0", "trailing size mismatch")}
    for name, (data, msg) in cases.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(data)
        with pytest.raises(hio.ModelFileError, match=msg):
            hio.load_model(p)
    assert issubclass(hio.ModelFileError, ValueError)


def _write_sequence(root, d):
    (root / "frames").mkdir(parents=True)
    (root / "params.json").write_text(str(d["seq.params"]))
    (root / "rig.json").write_text(str(d["seq.rig"]))
    for i in range(3):
        (root / "frames" / f"{i:06d}.png").write_bytes(d[f"seq.png{i}"].tobytes())
    (root / "gt_model.bin").write_bytes(d["seq.gt_model"].tobytes())


def test_load_sequence_matches_reference(tmp_path):
    d = golden("io")
    _write_sequence(tmp_path / "seq", d)
    s = hio.load_sequence(tmp_path / "seq")
    assert len(s) == 3
    np.testing.assert_array_equal(s.thetas, d["seq.thetas"])
    np.testing.assert_array_equal(s.images.astype(np.float64) / 255.0, d["seq.images"])
    assert s.rig.param_dim == s.thetas.shape[1]
    cam = s.camera_array()
    assert cam.shape == (16,) and cam[12] > 0


def test_load_sequence_errors(tmp_path):
    d = golden("io")
    with pytest.raises(FileNotFoundError, match="missing params.json"):
        hio.load_sequence(tmp_path)
    root = tmp_path / "seq"
    _write_sequence(root, d)
    (root / "frames" / "000002.png").unlink()
    with pytest.raises(FileNotFoundError, match="missing frame file"):
        hio.load_sequence(root)
    params = json.loads(str(d["seq.params"]))
    params["frame_count"] = 2
    (root / "params.json").write_text(json.dumps(params))
    with pytest.raises(ValueError, match="frame_count 2 does not match theta rows 3"):
        hio.load_sequence(root)
    params = json.loads(str(d["seq.params"]))
    params["theta"] = [t[:-1] for t in params["theta"]]
    (root / "params.json").write_text(json.dumps(params))
    with pytest.raises(ValueError, match="does not match rig parameter dimension"):
        hio.load_sequence(root)
    params = json.loads(str(d["seq.params"]))
    del params["rig"]
    (root / "params.json").write_text(json.dumps(params))
    with pytest.raises(ValueError, match="missing field 'rig'"):
        hio.load_sequence(root)
