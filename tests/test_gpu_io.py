"""Device side of the IO / evaluation row: hs_image_metrics against the
reference's psnr / ssim / l1, model files written from and read into device params
(byte-identical to the reference's), and `evaluate` on a reference-generated sequence
(rendered on the device in fp32 vs the reference's fp64 render)."""
import numpy as np
import pytest
import torch

from conftest import golden
from test_io import _HostAvatar, _write_sequence

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_12886_b200 import build
    build.build()


def test_image_metrics_match_reference():
    from paper_2503_12886_b200 import io as hio
    d = golden("io")
    for i in range(3):
        pred = torch.from_numpy(d[f"metrics{i}.pred"][None]).cuda()
        tgt = torch.from_numpy(d[f"metrics{i}.target"][None]).cuda()
        (p, s, l1), = hio.image_metrics(pred, tgt)
        ref = d[f"metrics{i}.values"]
        np.testing.assert_allclose([p, s, l1], ref, rtol=1e-9, atol=1e-12)


def test_psnr_cap_and_batch():
    from paper_2503_12886_b200 import io as hio
    d = golden("io")
    t = torch.from_numpy(d["metrics1.target"]).cuda()
    exact = (t[..., :3].double() / 255.0 * (t[..., 3:4].double() / 255.0)).float()
    pred = torch.stack([exact, torch.from_numpy(d["metrics1.pred"]).cuda()])
    m = hio.image_metrics(pred, torch.stack([t, t]))
    assert m[0][0] <= 99.0 and m[0][0] > 60.0          # fp32 rounding of the target only
    np.testing.assert_allclose(m[1], d["metrics1.values"], rtol=1e-9)


def test_device_model_file_roundtrip(tmp_path):
    from paper_2503_12886_b200 import io as hio
    from paper_2503_12886_b200.device import AvatarParams
    d = golden("io")
    ref = tmp_path / "ref.bin"
    ref.write_bytes(d["model.bytes"].tobytes())
    m = hio.load_model(ref)
    av, visited = m.to_device()
    assert isinstance(av, AvatarParams) and av.N == d["model.tri_index"].shape[0]
    out = tmp_path / "dev.bin"
    hio.save_model(av, visited, out)
    assert out.read_bytes() == ref.read_bytes()


def test_evaluate_matches_reference(tmp_path):
    from paper_2503_12886_b200 import io as hio
    from paper_2503_12886_b200.device import DeviceRig, Trainer
    d = golden("io")
    _write_sequence(tmp_path / "seq", d)
    seq = hio.load_sequence(tmp_path / "seq")
    gt = hio.load_model(tmp_path / "seq" / "gt_model.bin")
    av, _ = gt.to_device()
    h, w = seq.images.shape[1:3]
    tr = Trainer(av, w, h, 4, color_init=False, rig=DeviceRig(seq.rig))
    ev = hio.evaluate(tr, seq.thetas, seq.images, seq.camera_array())
    ref = d["seq.eval"]
    got = np.array([[f["psnr"], f["ssim"], f["l1"]] for f in ev["frames"]])
    # at ~59 dB one pixel whose alpha >= 1/255 or bbox decision flips between the fp32
    # device render and the fp64 reference moves the PSNR by ~0.1 dB, so compare the
    # MSE with an absolute budget of a few such pixels (3 HW = 6,912 terms here)
    mse_got, mse_ref = 10.0 ** (-got[:, 0] / 10.0), 10.0 ** (-ref[:, 0] / 10.0)
    np.testing.assert_allclose(mse_got, mse_ref, rtol=0, atol=1e-6)
    assert np.sum(np.abs(got[:, 0] - ref[:, 0]) < 1e-3) >= 2          # most frames agree tightly
    np.testing.assert_allclose(got[:, 1], ref[:, 1], atol=1e-4)
    np.testing.assert_allclose(got[:, 2], ref[:, 2], rtol=2e-2, atol=1e-6)
