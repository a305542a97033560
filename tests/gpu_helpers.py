"""Helpers shared by the GPU tests and scripts: read the device's fp32 stage outputs so
the oracle can replay the same decisions (SURVEY §8c stage-wise protocol)."""
import numpy as np

ATTRS = ("position", "rotation", "scale", "opacity", "color")


def unpack_bbox(rec):
    bits = np.ascontiguousarray(rec).view(np.uint32)
    lo = lambda v: (v & 0xFFFF).astype(np.int16).astype(np.int32)
    hi = lambda v: (v >> 16).astype(np.int16).astype(np.int32)
    return np.stack([lo(bits[..., 7]), hi(bits[..., 7]), lo(bits[..., 8]), hi(bits[..., 8])], axis=-1)


def replay_from_trainer(tr):
    """Per-frame {index, order, bbox} of the last projection (needs tr.radius captured)."""
    B, N = tr.B, tr.av.N
    rec = tr.records.view(B, N, 12).cpu().numpy()
    rad = tr.radius.view(B, N).cpu().numpy()
    dep = tr.depth.view(B, N).cpu().numpy()
    out = []
    for b in range(B):
        idx = np.flatnonzero(rad[b] > 0)
        out.append({"index": idx, "order": np.argsort(dep[b, idx], kind="stable"),
                    "bbox": unpack_bbox(rec[b, idx])})
    return out


def normwise(a, b, scale=None):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.linalg.norm(b) if scale is None else scale
    return float(np.linalg.norm(a - b) / max(den, 1e-300))
