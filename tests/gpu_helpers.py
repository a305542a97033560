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


def device_signs(tr):
    """(B, H, W, 3) int8 L1 signs of the last forward raster (pix_state bits 26..31)."""
    st = tr.pix_state.view(tr.B, tr.H, tr.W).cpu().numpy().view(np.uint32) >> 26
    out = np.zeros((tr.B, tr.H, tr.W, 3), np.int8)
    for c in range(3):
        s2 = (st >> (2 * c)) & 3
        out[..., c] = np.where(s2 == 1, 1, np.where(s2 == 2, -1, 0))
    return out


class MaskedReplay:
    """Trainer.debug_before_backward hook for a stage-exact step comparison.

    Between the device's forward raster and its adjoint it (1) captures the replay
    (kept set, depth order, integer bbox) and the device's per-pixel L1 signs, (2)
    runs the oracle's own float64 forward of every frame in the device's order,
    compares transmittance and L1 sign per pixel, and flags, with
    ``oracle.flip_mask``, the pixels where an alpha / ellipse / termination decision
    is within fp32 noise of its threshold -- on the oracle's float64 splats and on
    the device's fp32 splats -- and (3) clears the sign bits of the flagged pixels
    on the device.  The oracle's train_step then gets the same signs and mask
    (``replay``), so every remaining gradient entry must agree."""

    def __init__(self, O, model, cam, thetas, frames_list, targets=None, backgrounds=None):
        self.O, self.model, self.cam = O, model, cam
        self.thetas, self.frames = thetas, frames_list
        self.targets, self.backgrounds = targets, backgrounds
        self.replay = None
        self.report = {}

    def __call__(self, tr):
        import torch
        O = self.O
        torch.cuda.synchronize()
        replay = replay_from_trainer(tr)
        signs = device_signs(tr)
        B, N = tr.B, tr.av.N
        rec = tr.records.view(B, N, 12).cpu().numpy().astype(np.float64)
        rad = tr.radius.view(B, N).cpu().numpy().astype(np.float64)
        pT = tr.pix_T.view(B, tr.H, tr.W).cpu().numpy().astype(np.float64)
        masks = np.zeros((B, tr.H, tr.W), np.uint8)
        rep = dict(masked=0, pixels=B * tr.H * tr.W, t_maxabs=0.0, sign_flips=0,
                   sign_flip_max_absdiff=0.0)
        for b in range(B):
            world, _ = self.O.frame_forward(self.model, self.thetas[b], self.frames[b])
            sp = O.preprocess(world, self.cam)
            r = replay[b]
            assert np.array_equal(sp.index, r["index"]), "kept sets differ"
            O.flip_mask(sp, self.cam, order=r["order"], bbox=r["bbox"], out=masks[b])
            if self.targets is not None:
                img, aux = O.rasterize(sp, self.cam, self.backgrounds[b], order=r["order"], bbox=r["bbox"])
            i = r["index"]
            sp.mean2d, sp.conic = rec[b, i, 0:2].copy(), rec[b, i, 2:5].copy()
            sp.opacity, sp.radius = rec[b, i, 5].copy(), rad[b, i].copy()
            O.flip_mask(sp, self.cam, order=r["order"], bbox=r["bbox"], out=masks[b])
            ok = masks[b] == 0
            if self.targets is not None:
                rep["t_maxabs"] = max(rep["t_maxabs"], float(np.abs(pT[b] - aux.transmittance)[ok].max(initial=0)))
                tgt = O.composite_over(np.asarray(self.targets[b], np.float64) / 255.0, self.backgrounds[b])
                d = img - tgt
                osign = np.sign(d).astype(np.int8)
                flip = (osign != signs[b]) & ok[:, :, None]
                rep["sign_flips"] += int(flip.sum())
                if flip.any():
                    rep["sign_flip_max_absdiff"] = max(rep["sign_flip_max_absdiff"], float(np.abs(d[flip]).max()))
            r["signs"] = signs[b]
            r["gmask"] = masks[b].astype(bool)
        rep["masked"] = int(masks.sum())
        self.report = rep
        self.replay = replay
        m = torch.from_numpy(masks.reshape(-1).astype(bool)).to(tr.pix_state.device)
        ps = tr.pix_state
        ps.copy_(torch.where(m, ps & 0x03FFFFFF, ps))


def rel_fail(a, b, rtol=1e-3, floor_frac=1e-5, scale=None):
    """Entrywise |a-b| <= max(floor, rtol*max(|a|,|b|)) with floor = floor_frac * max|b|
    (or * scale).  Returns (failing entries, worst rel err above the floor, the
    smallest floor_frac under which nothing fails).  The floor is the fp32
    cancellation floor: gradient entries are sums over pixels (and frames) whose
    terms cancel, so an entry far below the tensor's maximum carries an absolute
    rounding error set by its terms, not by its value."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    ref = np.abs(b).max(initial=0.0) if scale is None else scale
    ref = max(ref, 1e-30)
    floor = floor_frac * ref
    diff = np.abs(a - b)
    sc = np.maximum(np.abs(a), np.abs(b))
    over = diff > rtol * sc
    bad = (diff > floor) & over
    r = np.where(diff <= floor, 0.0, diff / np.maximum(sc, 1e-300))
    need = float(diff[over].max(initial=0.0) / ref)
    return int(bad.sum()), float(r.max(initial=0.0)), need
