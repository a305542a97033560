"""Model file, sequence loading and evaluation for the device path.

* ``save_model`` / ``load_model``: the reference's single-file binary format
  (S/model_io.py:1-19 layout: "RGBA", version 1, N K H hidden, float32 base /
  deltas / MLP, u32 triangles, float32 barycentrics, bit-packed visited flags),
  written from and read into the device AvatarParams + visited flags.  Files are
  byte-identical to the reference's for the same model (golden-pinned), so models
  move freely between the two.
* ``load_sequence``: S/dataset.py:241-275 (params.json, rig.json, frames/%06d.png)
  with the reference's checks and messages; images stay u8 RGBA (the PNG bytes, the
  representation the device frame pool and the raster's fused loss consume).
* ``evaluate``: S/train.py:342-360 -- per-frame PSNR / SSIM / L1 against the targets
  composited over black, rendered in batches on the device and scored on the device
  (hs_image_metrics, fp64).
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

MAGIC = b"RGBA"
VERSION = 1
PSNR_CAP = 99.0
ATTRS = ("position", "rotation", "scale", "opacity", "color")


class ModelFileError(ValueError):
    """S/model_io.py:37-38."""


# --------------------------------------------------------------- model file

def save_model(avatar, visited, path):
    """S/model_io.py:41-65 from device state: avatar (AvatarParams), visited ((N,)
    bool/u8 array or tensor; None = all unvisited)."""
    path = Path(path)
    base, deltas, mlp = avatar.split_host()
    n, k, h, hidden = avatar.N, avatar.K, avatar.H, avatar.D
    chunks = [MAGIC, struct.pack("<5I", VERSION, n, k, h, hidden)]

    def put(arr, dtype="<f4"):
        chunks.append(np.ascontiguousarray(arr, dtype=dtype).tobytes())

    for a in ATTRS:
        put(base[a])
    for j in range(k):                      # device block k: [pos 3N | rot 4N | colour 3N]
        put(deltas[j, 0:3 * n])
        put(deltas[j, 3 * n:7 * n])
        put(deltas[j, 7 * n:10 * n])
    for name in ("w1", "b1", "w2", "b2", "w3", "b3"):
        put(mlp[name])
    put(avatar.tri_index.cpu().numpy(), dtype="<u4")
    put(avatar.barycentric.cpu().numpy())
    if visited is None:
        vis = np.zeros(n, bool)
    else:
        vis = visited.cpu().numpy() if hasattr(visited, "cpu") else np.asarray(visited)
    chunks.append(np.packbits(vis.astype(bool)).tobytes())
    path.write_bytes(b"".join(chunks))


@dataclass
class LoadedModel:
    base: dict            # attr -> (N, c) float64 (exact float32 values)
    deltas: np.ndarray    # (K, 10N) float64, block k = [pos (N,3) | rot (N,4) | colour (N,3)] flattened
    mlp: dict
    tri_index: np.ndarray
    barycentric: np.ndarray
    visited: np.ndarray   # (N,) bool

    def to_device(self, device="cuda"):
        """(AvatarParams, visited u8 tensor) on the device."""
        import torch
        from .device import AvatarParams
        g = type("G", (), dict(self.base))()
        av = AvatarParams.from_host(g, self.deltas, self.mlp, self.tri_index, self.barycentric, device=device)
        return av, torch.from_numpy(self.visited.astype(np.uint8)).to(device)


def load_model(path) -> LoadedModel:
    """S/model_io.py:68-110: the same checks and ModelFileError messages."""
    path = Path(path)
    data = path.read_bytes()
    if len(data) < 24:
        raise ModelFileError(f"{path}: file truncated before header")
    if data[:4] != MAGIC:
        raise ModelFileError(f"{path}: bad magic {data[:4]!r}")
    version, n, k, h, hidden = struct.unpack_from("<5I", data, 4)
    if version != VERSION:
        raise ModelFileError(f"{path}: unsupported version {version}")
    offset = 24

    def take(shape, dtype="<f4"):
        nonlocal offset
        count = int(np.prod(shape)) if shape else 1
        nbytes = count * np.dtype(dtype).itemsize
        if offset + nbytes > len(data):
            raise ModelFileError(f"{path}: file truncated at offset {offset}")
        arr = np.frombuffer(data, dtype=dtype, count=count, offset=offset).reshape(shape)
        offset += nbytes
        return arr.astype(np.float64) if dtype == "<f4" else arr

    base = {a: take(s) for a, s in zip(ATTRS, ((n, 3), (n, 4), (n, 3), (n,), (n, 3)))}
    deltas = np.empty((k, 10 * n))
    for j in range(k):
        deltas[j, 0:3 * n] = take((n, 3)).ravel()
        deltas[j, 3 * n:7 * n] = take((n, 4)).ravel()
        deltas[j, 7 * n:10 * n] = take((n, 3)).ravel()
    mlp = {}
    for name, shape in (("w1", (hidden, h)), ("b1", (hidden,)), ("w2", (hidden, hidden)), ("b2", (hidden,)),
                        ("w3", (k, hidden)), ("b3", (k,))):
        mlp[name] = take(shape)
    tri = take((n,), dtype="<u4").astype(np.int64)
    bary = take((n, 3))
    bits_len = (n + 7) // 8
    if offset + bits_len != len(data):
        raise ModelFileError(f"{path}: trailing size mismatch (expected {offset + bits_len} bytes, "
                             f"file has {len(data)})")
    visited = np.unpackbits(np.frombuffer(data, dtype=np.uint8, count=bits_len, offset=offset))[:n].astype(bool)
    return LoadedModel(base, deltas, mlp, tri, bary, visited)


# ------------------------------------------------------------------ sequence

@dataclass
class Sequence:
    """S/dataset.py:37-57 SequenceDataset, images kept as u8 RGBA (T, H, W, 4)."""
    directory: Path
    camera: dict              # Camera.to_dict() fields
    rig: object               # Rig
    thetas: np.ndarray        # (T, H_params) float64
    images: np.ndarray        # (T, H, W, 4) uint8

    def __len__(self):
        return self.thetas.shape[0]

    def camera_array(self) -> np.ndarray:
        c = self.camera
        return np.concatenate([np.asarray(c["rotation"], np.float64).ravel(),
                               np.asarray(c["translation"], np.float64).ravel(),
                               [c["fx"], c["fy"], c["cx"], c["cy"]]]).astype(np.float32)


@dataclass
class Rig:
    """The rig arrays of S/rig.py:18-54 ParametricHeadRig (what DeviceRig consumes)."""
    base_vertices: np.ndarray   # (V, 3)
    faces: np.ndarray           # (F, 3)
    uv_coords: np.ndarray       # (V, 2)
    expr_bases: np.ndarray      # (E, V, 3)
    pose_dim: int = 3

    @property
    def num_faces(self):
        return self.faces.shape[0]

    @property
    def num_expressions(self):
        return self.expr_bases.shape[0]

    @property
    def param_dim(self):
        return self.num_expressions + self.pose_dim


def load_rig(path):
    """S/dataset.py:229-245."""
    path = Path(path)
    try:
        d = json.loads(path.read_text())
    except FileNotFoundError:
        raise FileNotFoundError(f"rig file not found: {path}")
    for key in ("base_vertices", "faces", "uv_coords", "expr_bases"):
        if key not in d:
            raise ValueError(f"{path}: missing field {key!r}")
    return Rig(np.asarray(d["base_vertices"], np.float64), np.asarray(d["faces"], np.int64),
                   np.asarray(d["uv_coords"], np.float64), np.asarray(d["expr_bases"], np.float64),
                   pose_dim=int(d.get("pose_dim", 3)))


def load_sequence(directory) -> Sequence:
    """S/dataset.py:248-275 with the same checks and messages."""
    from PIL import Image
    directory = Path(directory)
    params_path = directory / "params.json"
    if not params_path.exists():
        raise FileNotFoundError(f"missing params.json in {directory}")
    params = json.loads(params_path.read_text())
    for key in ("camera", "theta", "frame_count", "rig"):
        if key not in params:
            raise ValueError(f"{params_path}: missing field {key!r}")
    camera = params["camera"]
    rig = load_rig(directory / params["rig"])
    thetas = np.asarray(params["theta"], dtype=np.float64)
    count = int(params["frame_count"])
    if thetas.ndim != 2 or thetas.shape[0] != count:
        raise ValueError(f"{params_path}: frame_count {count} does not match theta rows "
                         f"{thetas.shape[0] if thetas.ndim == 2 else 'non-tabular'}")
    if thetas.shape[1] != rig.param_dim:
        raise ValueError(f"{params_path}: theta dimension {thetas.shape[1]} does not match "
                         f"rig parameter dimension {rig.param_dim}")
    h, w = int(camera["height"]), int(camera["width"])
    images = np.empty((count, h, w, 4), np.uint8)
    for i in range(count):
        frame_path = directory / "frames" / f"{i:06d}.png"
        if not frame_path.exists():
            raise FileNotFoundError(f"missing frame file {frame_path}")
        with Image.open(frame_path) as im:
            arr = np.asarray(im.convert("RGBA"), dtype=np.uint8)
        if arr.shape[:2] != (h, w):
            raise ValueError(f"{frame_path}: image size {arr.shape[:2]} does not "
                             f"match camera ({h}, {w})")
        images[i] = arr
    return Sequence(directory, camera, rig, thetas, images)


# ---------------------------------------------------------------- evaluation

def image_metrics(pred, targets_u8):
    """Per-frame (psnr, ssim, l1) of pred (B,H,W,3 fp32 device) against targets
    (B,H,W,4 u8 device) composited over black (S/metrics.py:25-85), on the device."""
    import ctypes
    import torch
    from . import _lib as L
    B, H, W = pred.shape[:3]
    sums = torch.empty(B, 5, dtype=torch.float64, device=pred.device)
    L.call("hs_image_metrics", B, H, W, ctypes.c_void_p(pred.data_ptr()), ctypes.c_void_p(targets_u8.data_ptr()),
           ctypes.c_void_p(sums.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    s = sums.cpu().numpy()
    n = 3.0 * H * W
    out = []
    for b in range(B):
        mse = s[b, 0] / n
        p = PSNR_CAP if mse <= 0.0 else min(10.0 * np.log10(1.0 / mse), PSNR_CAP)
        ssim = float(np.mean(s[b, 2:5] / ((H - 10) * (W - 10))))
        out.append((float(p), ssim, float(s[b, 1] / n)))
    return out


def evaluate(trainer, thetas, images_u8, cameras, frame_indices=None):
    """S/train.py:342-360 on the device: renders the frames (black background, the
    Trainer's DeviceRig for mesh frames) in batches of trainer.B and scores them."""
    import torch
    B = trainer.B
    idx = list(frame_indices) if frame_indices is not None else list(range(len(thetas)))
    dev = trainer.av.device
    cams = torch.as_tensor(np.asarray(cameras, np.float32)).to(dev)
    zero = torch.zeros(B, 3, dtype=torch.float32, device=dev)
    per_frame = []
    for s in range(0, len(idx), B):
        chunk = idx[s:s + B]
        th = np.zeros((B, thetas.shape[1]), np.float32)
        th[:len(chunk)] = np.asarray(thetas)[chunk]
        tg = np.zeros((B,) + images_u8.shape[1:], np.uint8)
        tg[:len(chunk)] = images_u8[chunk]
        img = trainer.render(torch.from_numpy(th).to(dev), None, cams, zero)
        m = image_metrics(img, torch.from_numpy(tg).to(dev))
        for j, i in enumerate(chunk):
            per_frame.append({"frame": i, "psnr": m[j][0], "ssim": m[j][1], "l1": m[j][2]})
    return {"frames": per_frame,
            "mean_psnr": float(np.mean([f["psnr"] for f in per_frame])),
            "mean_ssim": float(np.mean([f["ssim"] for f in per_frame])),
            "mean_l1": float(np.mean([f["l1"] for f in per_frame]))}
