"""TEST INFRASTRUCTURE ONLY -- the bit-exact CPU oracle for batched tile binning.

The reference has no tile binning: it composites with one global stable depth
sort per frame (S/render.py:221-223) and scatters each splat over its pixel bbox
(S/render.py:248-251).  This restatement derives the
(frame, tile, depth) key list the device path must reproduce BIT-EXACTLY, from
the device path's own fp32 mean2d / radius / depth / opacity / valid:

1. skip n unless valid and opacity >= 1/255 (such splats never composite,
   S/render.py:239-240);
2. pixel bbox in IEEE fp32, one rounding per op, no FMA:
   r_lo = max(0, ceil((my - rad) - 0.5)), r_hi = min(H-1, floor((my + rad) - 0.5)),
   likewise for columns; skip if empty;
3. tiles ty in [r_lo//16, r_hi//16], tx in [c_lo//16, c_hi//16], id ty*TX + tx;
4. key = frame << (tile_bits+32) | tile << 32 | float_bits(depth), value = n,
   emitted n ascending, then ty, then tx;
5. stable sort by key (equal depth bits resolve to lower n = the reference's
   tie-break);
6. ranges[frame, tile] = [first, last+1), empty tiles [0, 0).

With conic and qmax (the training path, hs_project_avatar_fwd given tile_rects) step 3
keeps only the tiles some pixel of which the splat's alpha >= 1/255 ellipse can reach
(tile_reaches below, the device's hs_common.cuh:tile_reaches in the same fp32 operations),
for rectangles of at most 32 tiles; larger rectangles keep every tile.  The culled keys
composite nothing (every pixel of such a tile fails the reference's q <= qmax test,
S/render.py:260-262), so the rendered result is the same.
"""

from __future__ import annotations

import numpy as np

TILE = 16
ALPHA_CUTOFF_F32 = np.float32(1.0 / 255.0)


def bit_length(x: int) -> int:
    return int(x).bit_length()


def key_layout(batch: int, width: int, height: int):
    tiles_x = (width + TILE - 1) // TILE
    tiles_y = (height + TILE - 1) // TILE
    tiles = tiles_x * tiles_y
    tile_bits = bit_length(tiles - 1)
    frame_bits = bit_length(batch - 1)
    return tiles_x, tiles_y, tiles, tile_bits, frame_bits


def pixel_bbox(mean2d, radius, width, height):
    """Step 2 in fp32.  mean2d (..., 2), radius (...) float32 -> int32 (..., 4)
    (r_lo, r_hi, c_lo, c_hi); empty boxes have lo > hi."""
    mx = np.asarray(mean2d[..., 0], np.float32)
    my = np.asarray(mean2d[..., 1], np.float32)
    rad = np.asarray(radius, np.float32)
    half = np.float32(0.5)
    with np.errstate(invalid="ignore", over="ignore"):
        r_lo = np.ceil((my - rad) - half)
        r_hi = np.floor((my + rad) - half)
        c_lo = np.ceil((mx - rad) - half)
        c_hi = np.floor((mx + rad) - half)
    lim = np.float32(2.0 ** 30)
    r_lo = np.clip(np.nan_to_num(r_lo, nan=lim), -lim, lim).astype(np.int64)
    r_hi = np.clip(np.nan_to_num(r_hi, nan=-lim), -lim, lim).astype(np.int64)
    c_lo = np.clip(np.nan_to_num(c_lo, nan=lim), -lim, lim).astype(np.int64)
    c_hi = np.clip(np.nan_to_num(c_hi, nan=-lim), -lim, lim).astype(np.int64)
    r_lo = np.maximum(r_lo, 0)
    r_hi = np.minimum(r_hi, height - 1)
    c_lo = np.maximum(c_lo, 0)
    c_hi = np.minimum(c_hi, width - 1)
    return np.stack([r_lo, r_hi, c_lo, c_hi], axis=-1).astype(np.int32)


MASK_TILES = 32


def tile_reaches(mx, my, a, b, c, qmax, rl, rh, cl, ch, tx, ty):
    """Vectorised hs_common.cuh:tile_cull + tile_reaches: fp32, one rounding per op, the
    correctly rounded reciprocals of a and c, fmin/fmax (NaN-ignoring) clamps.  All
    arguments are arrays of one shape."""
    f = np.float32
    xs = np.maximum(tx * TILE, cl)
    xe = np.minimum(tx * TILE + TILE - 1, ch)
    ys = np.maximum(ty * TILE, rl)
    ye = np.minimum(ty * TILE + TILE - 1, rh)
    with np.errstate(all="ignore"):
        det = a * c - b * b
        pd = (det > 0) & (a > 0) & (c > 0)
        half = f(0.5)
        dxlo = (xs.astype(f) + half) - mx
        dxhi = (xe.astype(f) + half) - mx
        dylo = (ys.astype(f) + half) - my
        dyhi = (ye.astype(f) + half) - my
        zero = f(0.0)
        inv_a = np.where(pd, f(1.0) / a, f(0.0)).astype(f)
        inv_c = np.where(pd, f(1.0) / c, f(0.0)).astype(f)
        dxv = np.fmin(np.fmax(zero, dxlo), dxhi)
        dyv = np.fmin(np.fmax(((-b) * dxv) * inv_c, dylo), dyhi)
        dyh = np.fmin(np.fmax(zero, dylo), dyhi)
        dxh = np.fmin(np.fmax(((-b) * dyh) * inv_a, dxlo), dxhi)
        b2 = f(2.0) * b
        qv = ((a * dxv) * dxv + (b2 * dxv) * dyv) + (c * dyv) * dyv
        qh = ((a * dxh) * dxh + (b2 * dxh) * dyh) + (c * dyh) * dyh
        cull = (np.fmin(qv, qh) * f(0.999) - f(1e-3)) > qmax
    return ~pd | ~cull


def bin_batch(mean2d, radius, depth, opacity, valid, width, height, conic=None, qmax=None):
    """All inputs per (frame, Gaussian): mean2d (B, N, 2), radius/depth/opacity
    (B, N) float32, valid (B, N) bool; conic (B, N, 3) and qmax (B, N) float32 turn on
    the tile cull.  Returns dict with keys (u64), values (u32), ranges (B, tiles, 2) u32,
    bbox (B, N, 4) int32, counts (B, N) u32."""
    mean2d = np.asarray(mean2d, np.float32)
    radius = np.asarray(radius, np.float32)
    depth = np.asarray(depth, np.float32)
    opacity = np.asarray(opacity, np.float32)
    valid = np.asarray(valid, bool)
    B, N = radius.shape
    tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
    bbox = pixel_bbox(mean2d, radius, width, height)
    live = valid & (opacity >= ALPHA_CUTOFF_F32) & (bbox[..., 0] <= bbox[..., 1]) & (bbox[..., 2] <= bbox[..., 3])
    ty0 = bbox[..., 0] // TILE
    ty1 = bbox[..., 1] // TILE
    tx0 = bbox[..., 2] // TILE
    tx1 = bbox[..., 3] // TILE
    counts = np.where(live, (ty1 - ty0 + 1) * (tx1 - tx0 + 1), 0).astype(np.int64)
    total = int(counts.sum())
    depth_bits = depth.view(np.uint32).astype(np.uint64)
    bs, ns = np.nonzero(counts)           # row-major: b, then n ascending (emission order)
    c = counts[bs, ns]
    nx = np.repeat((tx1 - tx0 + 1)[bs, ns], c)
    local = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(c) - c, c)
    ty = np.repeat(ty0[bs, ns], c) + local // nx        # ty major, then tx
    tx = np.repeat(tx0[bs, ns], c) + local % nx
    frames = np.repeat(bs, c).astype(np.uint64)
    vals = np.repeat(ns, c).astype(np.uint32)
    dbits = np.repeat(depth_bits[bs, ns], c)
    if conic is not None:
        conic = np.asarray(conic, np.float32)
        qmax = np.asarray(qmax, np.float32)
        rep = lambda x: np.repeat(x[bs, ns], c)
        keep = (rep(counts) > MASK_TILES) | tile_reaches(
            rep(mean2d[..., 0]), rep(mean2d[..., 1]), rep(conic[..., 0]), rep(conic[..., 1]), rep(conic[..., 2]),
            rep(qmax), rep(bbox[..., 0]).astype(np.int64), rep(bbox[..., 1]).astype(np.int64),
            rep(bbox[..., 2]).astype(np.int64), rep(bbox[..., 3]).astype(np.int64), tx, ty)
        ty, tx, frames, vals, dbits = ty[keep], tx[keep], frames[keep], vals[keep], dbits[keep]
        kept = np.zeros(counts.shape, np.int64)
        np.add.at(kept, (np.repeat(bs, c)[keep], np.repeat(ns, c)[keep]), 1)
        counts = kept
        total = int(counts.sum())
    tile_ids = (ty * tiles_x + tx).astype(np.uint64)
    keys = (frames << np.uint64(tile_bits + 32)) | (tile_ids << np.uint64(32)) | dbits
    order = np.argsort(keys, kind="stable")
    keys = keys[order]
    vals = vals[order]
    ranges = np.zeros((B, tiles, 2), np.uint32)
    if total:
        ft = (keys >> np.uint64(32)).astype(np.int64)          # frame * 2^tile_bits + tile
        starts = np.flatnonzero(np.r_[True, ft[1:] != ft[:-1]])
        ends = np.r_[starts[1:], total]
        fr = ft[starts] >> tile_bits
        tl = ft[starts] & ((1 << tile_bits) - 1)
        ranges[fr, tl, 0] = starts
        ranges[fr, tl, 1] = ends
    return {"keys": keys, "values": vals, "ranges": ranges, "bbox": bbox,
            "counts": counts.astype(np.uint32), "tile_bits": tile_bits, "frame_bits": frame_bits,
            "tiles_x": tiles_x, "tiles_y": tiles_y}


def lexsort_check(res, depth):
    """Appendix B item 7: the sorted list equals np.lexsort((n, depth_bits, tile, frame))."""
    keys = res["keys"]
    vals = res["values"].astype(np.int64)
    tile_bits = res["tile_bits"]
    frame = (keys >> np.uint64(tile_bits + 32)).astype(np.int64)
    tile = ((keys >> np.uint64(32)) & np.uint64((1 << tile_bits) - 1)).astype(np.int64)
    dbits = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    o = np.lexsort((vals, dbits, tile, frame))
    return np.array_equal(o, np.arange(keys.size))
