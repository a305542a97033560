"""Device-resident training / rendering on one B200 (the fast API: torch tensors in, no host copies).

This is the B200 replacement of the reference's ``train_step`` (S/train.py:214-260)
and its render path (S/dataset.py:163-172, S/train.py:333-339).  The frame batch
is a grid dimension of every kernel: one launch per stage per batch, and exactly
ONE device->host read per step (the key total + error word after the tile-count
scan, needed to size the sort), mirroring the paper's single GPU->CPU sync
between the projection and rasterization stages (PAPER.md:156,
S/scheduler.py:64-72).

Step (N Gaussians, K bases, B frames):
  [rig_frames: theta -> mesh frames, when the Trainer holds a DeviceRig]
  -> mlp_fwd -> blend_fwd -> project_avatar_fwd (+ tile counts) -> bin_scan -> [sync]
  -> bin_emit -> sort_pairs -> tile_ranges -> raster_fwd (+ L1 loss, colour-init
  sums) -> loss_reduce -> raster_bwd -> project_avatar_bwd -> blend_bwd -> mlp_bwd
  -> [bucketed allreduce of the flat gradient, multi-GPU] -> Adam + colour init.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

ATTRS = ("position", "rotation", "scale", "opacity", "color")
ADAM_BETAS = (0.9, 0.999)       # S/optim.py:19-21
ADAM_EPS = 1e-8
TILE = 16


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    """The current CUDA stream as a raw handle for the C ABI.  (Straight from the torch
    stream registry: torch.cuda.current_stream() re-resolves the device through
    availability checks on every call, ~10 us of host time a step's worth of calls.)"""
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_12886_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    L.load()


def default_lrs(lr_position=0.0008, lr_opacity=0.25, lr_scale=0.025, lr_rotation=0.005, lr_color=0.0125,
                delta_position_scale=0.05, delta_rotation_scale=0.5, delta_color_scale=0.5, lr_mlp=0.001):
    """Per-group learning rates in hs_adam order (S/train.py:43-51, :63-68):
    base position, rotation, color, scale, opacity, delta position, rotation, color, mlp."""
    return [lr_position, lr_rotation, lr_color, lr_scale, lr_opacity, lr_position * delta_position_scale,
            lr_rotation * delta_rotation_scale, lr_color * delta_color_scale, lr_mlp]


def lrs_from_config(cfg):
    """Learning rates from a reference-style TrainConfig (duck typed)."""
    return default_lrs(cfg.lr_position, cfg.lr_opacity, cfg.lr_scale, cfg.lr_rotation, cfg.lr_color,
                       cfg.delta_position_scale, cfg.delta_rotation_scale, cfg.delta_color_scale, cfg.lr_mlp)


def key_layout(batch, width, height):
    tiles_x = (width + TILE - 1) // TILE
    tiles_y = (height + TILE - 1) // TILE
    tiles = tiles_x * tiles_y
    tile_bits = int(tiles - 1).bit_length()
    frame_bits = int(batch - 1).bit_length()
    return tiles_x, tiles_y, tiles, tile_bits, frame_bits


def camera_array(camera) -> np.ndarray:
    """(16,) float32 [R 9 | t 3 | fx fy cx cy] from a reference-style Camera (S/render.py:40-84)."""
    return np.concatenate([np.asarray(camera.rotation, np.float64).ravel(),
                           np.asarray(camera.translation, np.float64).ravel(),
                           [camera.fx, camera.fy, camera.cx, camera.cy]]).astype(np.float32)


def frames_array(frames) -> np.ndarray:
    """(F, 22) float32 from a reference-style MeshFrames (S/binding.py:47-53)."""
    f = np.asarray(frames.rotation).shape[0]
    return np.concatenate([np.asarray(frames.rotation, np.float64).reshape(f, 9),
                           np.asarray(frames.quat, np.float64).reshape(f, 4),
                           np.asarray(frames.tri_vertices, np.float64).reshape(f, 9)], axis=1).astype(np.float32)


# --------------------------------------------------------------------- model

class AvatarParams:
    """Device-resident reduced-blendshape avatar (S/model.py:98-127 AvatarModel).

    params: flat fp32 [base 14N | deltas K*10N | mlp] (include/hs_api.h layout),
    tri_index int32 (N,), barycentric fp32 (N, 3).
    """

    def __init__(self, N, K, H, D, device="cuda"):
        require_cuda()
        self.N, self.K, self.H, self.D = int(N), int(K), int(H), int(D)
        self.mlp_size = int(L.load().hs_mlp_size(self.H, self.D, self.K))
        self.size = 14 * self.N + 10 * self.K * self.N + self.mlp_size
        self.device = torch.device(device)
        self.params = torch.zeros(self.size, dtype=torch.float32, device=self.device)
        self.tri_index = torch.zeros(self.N, dtype=torch.int32, device=self.device)
        self.barycentric = torch.zeros(self.N, 3, dtype=torch.float32, device=self.device)

    # views ------------------------------------------------------------
    @property
    def base14(self):
        return self.params[:14 * self.N]

    @property
    def deltas(self):
        return self.params[14 * self.N:14 * self.N + 10 * self.K * self.N]

    @property
    def mlp(self):
        return self.params[14 * self.N + 10 * self.K * self.N:]

    def base_view(self, name):
        n = self.N
        off = {"position": (0, 3), "rotation": (3 * n, 4), "color": (7 * n, 3), "scale": (10 * n, 3),
               "opacity": (13 * n, 1)}[name]
        v = self.params[off[0]:off[0] + off[1] * n]
        return v if name == "opacity" else v.view(n, off[1])

    # conversion -------------------------------------------------------
    @staticmethod
    def pack_base(base) -> np.ndarray:
        return np.concatenate([np.asarray(base.position).ravel(), np.asarray(base.rotation).ravel(),
                               np.asarray(base.color).ravel(), np.asarray(base.scale).ravel(),
                               np.asarray(base.opacity).ravel()])

    @staticmethod
    def pack_deltas(deltas) -> np.ndarray:
        if isinstance(deltas, np.ndarray):
            return deltas.reshape(-1)
        return np.concatenate([np.concatenate([np.asarray(d.position).ravel(), np.asarray(d.rotation).ravel(),
                                               np.asarray(d.color).ravel()]) for d in deltas])

    @staticmethod
    def pack_mlp(mlp) -> np.ndarray:
        get = (lambda k: mlp[k]) if isinstance(mlp, dict) else (lambda k: getattr(mlp, k))
        return np.concatenate([np.asarray(get(k)).ravel() for k in ("w1", "b1", "w2", "b2", "w3", "b3")])

    @classmethod
    def from_host(cls, base, deltas, mlp, tri_index, barycentric, device="cuda"):
        """From reference-style objects (GaussianSet, list[DeltaSet] or (K,10N) array,
        MlpWeights or dict, bindings arrays)."""
        get = (lambda k: mlp[k]) if isinstance(mlp, dict) else (lambda k: getattr(mlp, k))
        w1 = np.asarray(get("w1"))
        N = np.asarray(base.position).shape[0]
        K = np.asarray(get("w3")).shape[0]
        self = cls(N, K, w1.shape[1], w1.shape[0], device)
        self.load_host(base, deltas, mlp)
        self.tri_index.copy_(torch.from_numpy(np.asarray(tri_index, np.int32)))
        self.barycentric.copy_(torch.from_numpy(np.asarray(barycentric, np.float32).reshape(N, 3)))
        return self

    def load_host(self, base, deltas, mlp):
        flat = np.concatenate([self.pack_base(base), self.pack_deltas(deltas), self.pack_mlp(mlp)]).astype(np.float32)
        if flat.size != self.size:
            raise ValueError(f"parameter count {flat.size} != {self.size}")
        self.params.copy_(torch.from_numpy(flat))

    def host_flat(self) -> np.ndarray:
        return self.params.detach().cpu().numpy()

    def split_host(self, flat=None, dtype=np.float64):
        """(base dict, deltas (K,10N), mlp dict) numpy (float64, or views of ``flat``
        with dtype=None) from the device copy."""
        flat = self.host_flat() if flat is None else flat
        return split_flat(flat, self.N, self.K, self.H, self.D, dtype)


def split_flat(flat, N, K, H, D, dtype=np.float64):
    flat = np.asarray(flat, dtype)
    n = N
    base = {"position": flat[0:3 * n].reshape(n, 3), "rotation": flat[3 * n:7 * n].reshape(n, 4),
            "color": flat[7 * n:10 * n].reshape(n, 3), "scale": flat[10 * n:13 * n].reshape(n, 3),
            "opacity": flat[13 * n:14 * n].copy()}
    o = 14 * n
    deltas = flat[o:o + 10 * K * n].reshape(K, 10 * n)
    o += 10 * K * n
    mlp = {}
    for k, shape in (("w1", (D, H)), ("b1", (D,)), ("w2", (D, D)), ("b2", (D,)), ("w3", (K, D)), ("b3", (K,))):
        sz = int(np.prod(shape))
        mlp[k] = flat[o:o + sz].reshape(shape)
        o += sz
    return base, deltas, mlp


# -------------------------------------------------------------------- binning

class DeviceRig:
    """Device copy of the head rig (S/rig.py:18-54 ParametricHeadRig) that turns
    rig parameters into mesh frames on the GPU (hs_rig_frames):
    rig_evaluate (S/rig.py:57-66) + mesh_frames (S/binding.py:67-115).

    ``rig`` is any object with base_vertices (V,3), faces (F,3), uv_coords (V,2) and
    expr_bases (E,V,3) -- the reference's rig or io.Rig."""

    def __init__(self, rig, device="cuda"):
        require_cuda()
        f64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(device)
        self.base = f64(rig.base_vertices)
        self.bases = f64(rig.expr_bases)
        self.uv = f64(rig.uv_coords)
        self.faces = torch.from_numpy(np.ascontiguousarray(rig.faces, np.int32)).to(device)
        self.V, self.F, self.E = self.base.shape[0], self.faces.shape[0], self.bases.shape[0]
        if self.bases.shape[1:] != (self.V, 3) or self.uv.shape != (self.V, 2):
            raise ValueError("rig arrays have inconsistent shapes")
        self.err = torch.full((1,), -1, dtype=torch.int64, device=device)
        self.device = device

    @property
    def param_dim(self):
        return self.E + 3

    def frames(self, thetas=None, vertices=None, out=None, err=None):
        """(B, F, 22) fp32 frames of thetas (B, E+3) fp32 or of vertices (B, V, 3) fp64.
        With err=None the call checks the error word (a host sync) and raises the
        reference's DegenerateTriangleError; with a caller err word it is async."""
        src = thetas if vertices is None else vertices
        if src is None:
            raise ValueError("need thetas or vertices")
        B = src.shape[0]
        if vertices is None and thetas.shape[-1] != self.param_dim:
            raise ValueError(f"theta has shape {tuple(thetas.shape)}, rig expects (B, {self.param_dim})")
        if out is None:
            out = torch.empty(B, self.F, 22, dtype=torch.float32, device=self.device)
        check = err is None
        if check:
            err = self.err
            err.fill_(-1)
        L.call("hs_rig_frames", B, self.V, self.F, self.E, _p(self.base), _p(self.bases), _p(self.faces),
               _p(self.uv), _p(thetas), _p(vertices), _p(out), _p(err), _stream())
        if check:
            L.raise_device_error(int(err.item()) & 0xFFFFFFFFFFFFFFFF)
        return out


class Binner:
    """Batched tile binning shared by training, rendering and the compat path:
    project-stage outputs -> (keys, values, ranges) with one host read."""

    def __init__(self, device):
        self.device = device
        self.cap = 0
        self.keys = self.vals = self.keys_alt = self.vals_alt = self.ws = None
        self.summary_host = torch.empty(4, dtype=torch.int64, pin_memory=True)
        self.offsets = None
        self.summary = torch.empty(4, dtype=torch.int64, device=device)
        self.depth_range = torch.empty(2, dtype=torch.int32, device=device)
        self._depth_range_init = None
        self._depth_range_clean = False     # hs_tile_scan reset it (no fallback that step)
        self.depth_bits = (0, 0)
        self.passes = 0
        self.ranges = None
        self.result = None
        self.order = None
        self._ordered = None
        self.tile_counts = None
        self.order_ready = False
        self.rects = None
        self.mode = None             # how the last bin() built its lists
        self.longest = 0             # longest (frame, tile) list of the last tile-major binning
        self.fork = None             # hs_fork_create context (side stream of the list sorts)
        self._d2h = None             # stream of the step's summary read
        # tile-major binning writes the (frame, tile) key of every entry only when asked
        # (checkers); the raster reads values and ranges only
        self.write_keys = True

    def __del__(self):
        try:
            if self.fork is not None and self.fork.value:
                with torch.cuda.device(self._fork_dev):
                    L.load().hs_fork_destroy(self.fork)
                self.fork = None
        except Exception:
            pass

    def _ensure(self, total):
        if total <= self.cap and self.keys is not None:
            return
        cap = max(int(total * 1.25) + 1024, 1 << 16)
        d = self.device
        self.keys = torch.empty(cap, dtype=torch.int64, device=d)
        self.keys_alt = torch.empty(cap, dtype=torch.int64, device=d)
        self.vals = torch.empty(cap, dtype=torch.int32, device=d)
        self.vals_alt = torch.empty(cap, dtype=torch.int32, device=d)
        ws = int(L.load().hs_sort_workspace_size(cap))
        self.ws = torch.empty(ws, dtype=torch.uint8, device=d)
        self.cap = cap

    def reset_depth_range(self):
        """{0xFFFFFFFF, 0}: the projection atomically narrows it to the depths that emit keys.
        (A device-to-device copy: element assignment from a host scalar would be a
        pageable host->device copy, which blocks the host until the stream drains.)  After a
        tile-major binning that needed no fallback, hs_tile_scan has already reset it."""
        if self._depth_range_clean:
            self._depth_range_clean = False
            return self.depth_range
        if self._depth_range_init is None:
            self._depth_range_init = torch.tensor([-1, 0], dtype=torch.int32, device=self.device)
        self.depth_range.copy_(self._depth_range_init)
        return self.depth_range

    def scan(self, block_sums, nblocks, err, overlap=None):
        """Exclusive scan of the per-block tile counts + the step's single D2H read
        (key total, error word, depth-bit range).  ``overlap`` (a callable) enqueues
        work that needs no host answer after the read: the host then waits on the
        read's event only, while the GPU runs that work."""
        if self.offsets is None or self.offsets.numel() < nblocks:
            self.offsets = torch.empty(max(nblocks, 1), dtype=torch.int32, device=self.device)
        L.call("hs_bin_scan", nblocks, _p(block_sums), _p(self.offsets), _p(err), _p(self.depth_range),
               _p(self.summary), _stream())
        self.summary_host.copy_(self.summary, non_blocking=True)
        ready = torch.cuda.Event()
        ready.record()
        if overlap is not None:
            overlap()
        ready.synchronize()
        total = int(self.summary_host[0])
        code = int(self.summary_host[1]) & 0xFFFFFFFFFFFFFFFF
        dr = int(self.summary_host[2]) & 0xFFFFFFFFFFFFFFFF
        self.depth_bits = (dr & 0xFFFFFFFF, dr >> 32)
        return total, code

    def sort_mask(self, tile_bits, frame_bits):
        """Key bits the sort must resolve: the frame/tile bits plus the depth bits below
        the highest bit in which the smallest and largest emitted depth differ."""
        lo, hi = self.depth_bits
        depth_width = (lo ^ hi).bit_length() if lo <= hi else 32
        return (((1 << (tile_bits + frame_bits)) - 1) << 32) | ((1 << depth_width) - 1)

    def depth_order(self, B, N, depth):
        """Two-level binning, stage 1 (hs_depth_order): the (frame, Gaussian) items in
        stable depth order.  Needs only the projection's outputs (no host read), so it
        is enqueued before the scan and runs while the host waits for the key total."""
        items = B * N
        d = self.device
        if self.order is None or self.order.numel() < items:
            mk = lambda: torch.empty(items, dtype=torch.int32, device=d)
            self.order, self.order_alt, self.dkeys_a, self.dkeys_b = mk(), mk(), mk(), mk()
            self.dws = torch.empty(int(L.load().hs_sort_workspace_size(items)), dtype=torch.uint8, device=d)
            nb = int(L.load().hs_scan_blocks(items))
            self.sblock_sums = torch.empty(nb, dtype=torch.int32, device=d)
            self.sblock_offs = torch.empty(nb, dtype=torch.int32, device=d)
        L.call("hs_depth_order", items, _p(depth), _p(self.depth_range), _p(self.order), _p(self.order_alt),
               _p(self.dkeys_a), _p(self.dkeys_b), _p(self.dws), self.dws.numel(), _stream())
        self._ordered = (B, N)

    def bin(self, B, N, width, height, records, depth, counts, total, rects=None):
        """rects: the projection's tile_rects when it had them (its counts then hold only the
        kept tiles, which the emitters must reproduce)."""
        if self._ordered == (B, N):
            return self._bin_two_level(B, N, width, height, records, counts, total, rects)
        tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
        self._ensure(total)
        s = _stream()
        nr = B << tile_bits
        if self.ranges is None or self.ranges.numel() < 2 * nr:
            self.ranges = torch.empty(2 * nr, dtype=torch.int32, device=self.device)
        ranges = self.ranges[:2 * nr]
        ranges.zero_()
        if total:
            L.call("hs_bin_emit", B, N, width, height, _p(records), _p(depth), _p(counts), _p(self.offsets),
                   _p(rects), _p(self.keys), _p(self.vals), s)
            alt = ctypes.c_int(0)
            mask = self.sort_mask(tile_bits, frame_bits)
            self.passes = sum(1 for sh in range(0, 64, 8) if (mask >> sh) & 0xFF)
            L.call("hs_sort_pairs", total, ctypes.c_uint64(mask), _p(self.keys), _p(self.vals),
                   _p(self.keys_alt), _p(self.vals_alt), _p(self.ws), self.ws.numel(), ctypes.byref(alt), s)
            keys, vals = (self.keys_alt, self.vals_alt) if alt.value else (self.keys, self.vals)
            L.call("hs_tile_ranges", total, _p(keys), _p(ranges), s)
        else:
            keys, vals = self.keys, self.vals
        self.result = (keys[:total], vals[:total], ranges, tile_bits, tiles)
        return self.result

    def _fill_longest(self, B, N, width, height, depth, ranges, s):
        L.call("hs_tile_fill_longest", B, N, width, height, _p(depth), _p(ranges), _p(self.lists),
               _p(self.list_counts), self.list_half, _p(self.summary), self.cap, _p(self.vals), s)

    def _bin_two_level(self, B, N, width, height, records, counts, total, rects=None):
        """Stage 2: emission in depth order with 32-bit (frame, tile) keys and a stable
        sort of those keys alone (frame + tile bits: 2 passes at C2) -- the same
        per-tile lists as the one-level (frame, tile, depth) sort."""
        self._ordered = None
        tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
        self._ensure(total)
        s = _stream()
        nr = B << tile_bits
        if self.ranges is None or self.ranges.numel() < 2 * nr:
            self.ranges = torch.empty(2 * nr, dtype=torch.int32, device=self.device)
        ranges = self.ranges[:2 * nr]
        ranges.zero_()
        k32, k32_alt = self.keys.view(torch.int32), self.keys_alt.view(torch.int32)
        if total:
            L.call("hs_bin_emit_sorted", B, N, width, height, _p(records), _p(counts), _p(rects), _p(self.order),
                   _p(self.sblock_sums), _p(self.sblock_offs), _p(k32), _p(self.vals), s)
            alt = ctypes.c_int(0)
            mask = (1 << (tile_bits + frame_bits)) - 1
            self.passes = sum(1 for sh in range(0, 32, 8) if (mask >> sh) & 0xFF)
            L.call("hs_sort_pairs32", total, ctypes.c_uint32(mask), _p(k32), _p(self.vals), _p(k32_alt),
                   _p(self.vals_alt), _p(self.ws), self.ws.numel(), ctypes.byref(alt), s)
            keys, vals = (k32_alt, self.vals_alt) if alt.value else (k32, self.vals)
            L.call("hs_tile_ranges32", total, _p(keys), _p(ranges), s)
        else:
            keys, vals = k32, self.vals
        self.result = (keys[:total], vals[:total], ranges, tile_bits, tiles)
        return self.result


    def tile_count_buffer(self, B, width, height):
        """The zeroed per-(frame, tile) counters, for a projection that counts the tiles
        itself (hs_project_avatar_fwd's tile_counts); then bin_tiles(counted=True)."""
        tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
        nseg = B << tile_bits
        d = self.device
        if self.tile_counts is None or self.tile_counts.numel() < nseg:
            self.tile_counts = torch.zeros(nseg, dtype=torch.int32, device=d)
            self.cursor = torch.empty(nseg, dtype=torch.int32, device=d)
            self.lists = torch.empty(2 * nseg, dtype=torch.int32, device=d)
            self.list_half = 8 + (nseg + 1023) // 1024
            self.list_counts = torch.zeros(1 + 2 * self.list_half, dtype=torch.int32, device=d)
        return self.tile_counts

    def tile_rects_buffer(self, B, N, width, height):
        """Per-item packed tile rectangles (hs_project_avatar_fwd's tile_rects) for the
        fill, or None when an image axis has more than 256 tiles."""
        tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
        if tiles_x > 256 or tiles_y > 256:
            return None
        if self.rects is None or self.rects.numel() < 2 * B * N:
            self.rects = torch.empty(2 * B * N, dtype=torch.int32, device=self.device)
        return self.rects[:2 * B * N]

    def bin_tiles(self, B, N, width, height, records, depth, counts, err, after_scan=None, counted=False,
                  rects=None, speculate=None):
        """Tile-major binning (hs_tile_count / hs_tile_scan / hs_tile_fill) with the
        step's single host read: the scatter and the per-list sorts are enqueued before
        the host waits, sized by the previous step's capacity; a step that needs more
        re-runs them on grown buffers.  Lists longer than hs_tile_sort_cap() fall back to
        the two-level sort for that step.  ``after_scan(ranges, tile_bits, scanned)`` enqueues
        work that needs only the ranges (the raster's tile order; ``scanned`` is the event
        after the scan).  Returns (key total, error word)."""
        tiles_x, tiles_y, tiles, tile_bits, frame_bits = key_layout(B, width, height)
        nseg = B << tile_bits
        d = self.device
        self.tile_count_buffer(B, width, height)
        if self.ranges is None or self.ranges.numel() < 2 * nseg:
            self.ranges = torch.empty(2 * nseg, dtype=torch.int32, device=d)
        ranges = self.ranges[:2 * nseg]
        s = _stream()
        if not counted:
            L.call("hs_tile_count", B, N, width, height, _p(records), _p(counts), _p(self.tile_counts), s)
        L.call("hs_tile_scan", B, width, height, _p(self.tile_counts), _p(ranges), _p(self.cursor),
               _p(self.lists), _p(self.list_counts), self.list_half, _p(err), _p(self.depth_range), _p(self.summary),
               s)
        # the summary's D2H copy runs on a side stream behind the scan, so the compute
        # stream goes straight on to the scatter (a copy in its own order would hold the
        # scatter back by the copy's latency)
        scanned = torch.cuda.Event()
        scanned.record()
        if self._d2h is None:
            self._d2h = torch.cuda.Stream(device=torch.cuda.current_device())
        self._d2h.wait_event(scanned)
        with torch.cuda.stream(self._d2h):
            self.summary_host.copy_(self.summary, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self._d2h)
        if self.keys is None:
            self._ensure(4 * B * N)         # a first guess; grown below when short

        if self.fork is None:
            self._fork_dev = torch.cuda.current_device()
            self.fork = ctypes.c_void_p(L.load().hs_fork_create())
            if not self.fork.value:
                raise RuntimeError(f"hs_fork_create: {L.last_error()}")

        # lists past the warp-run sorts expected (the previous batch had them: render
        # batches of crowded tiles): the fill sorts them too, first on its side stream,
        # instead of a CTA sort enqueued after the summary read
        forked_longest = _cta_sort_min() <= self.longest <= tile_sort_cap()

        def fill():
            L.call("hs_tile_fill", B, N, width, height, _p(records), _p(counts), _p(rects), _p(depth), _p(ranges),
                   _p(self.cursor), _p(self.lists), _p(self.list_counts), self.list_half, _p(self.summary), self.cap,
                   _p(self.keys) if self.write_keys else None, _p(self.vals),
                   L.FILL_CTA_SORT if forked_longest else 0, self.fork, s)
        fill()                              # first: the GPU reaches it right after the scan
        self.order_ready = False
        if after_scan is not None:
            self.order_ready = after_scan(ranges, tile_bits, scanned)
        # the consumer of the lists, enqueued before the host reads the summary: it runs
        # right after the fill unless the device-side guard (hs_raster_guard_t) finds the
        # lists incomplete, in which case it exits and spec_valid tells the caller to
        # launch it again once the rare case is handled
        cap_at_fill = self.cap
        self.spec_valid = False
        if speculate is not None:
            guard = L.RasterGuard(self.summary.data_ptr(), cap_at_fill,
                                  tile_sort_cap() if forked_longest else _cta_sort_min() - 1)
            speculate(self.vals[:cap_at_fill], ranges, tile_bits, guard)
        ready.synchronize()
        total = int(self.summary_host[0])
        code = int(self.summary_host[1]) & 0xFFFFFFFFFFFFFFFF
        dr = int(self.summary_host[2]) & 0xFFFFFFFFFFFFFFFF
        self.depth_bits = (dr & 0xFFFFFFFF, dr >> 32)
        self.longest = int(self.summary_host[3])
        self.mode = "tiles"
        regrown = total > self.cap
        if regrown:
            self._ensure(total)
            self.cursor[:nseg].copy_(ranges.view(-1, 2)[:, 0])
            fill()
        huge = _cta_sort_min() <= self.longest <= tile_sort_cap()
        self.launches_extra = int(forked_longest) * (1 + int(regrown))
        if huge and not forked_longest:
            # lists long enough for the shared-memory CTA sort, not expected: after the fill
            self._fill_longest(B, N, width, height, depth, ranges, s)
            self.launches_extra += 1
        self._depth_range_clean = self.longest <= tile_sort_cap()
        self.spec_valid = (speculate is not None and total <= cap_at_fill and code == L.HS_NO_ERROR
                           and (self.longest < _cta_sort_min() or (forked_longest and huge)))
        if self.longest > tile_sort_cap():
            # a list too long to sort in shared memory: the global two-level sort
            # (whose ranges replace the ones the tile order was built from)
            self.order_ready = False
            self.depth_order(B, N, depth)
            self._bin_two_level(B, N, width, height, records, counts, total, rects)
            self.mode = "two_level"
            return total, code
        k32 = self.keys.view(torch.int32)
        self.result = (k32[:total], self.vals[:total], ranges, tile_bits, tiles)
        return total, code


_SORT_CAP = None
_CTA_MIN = None


def _cta_sort_min():
    global _CTA_MIN
    if _CTA_MIN is None:
        _CTA_MIN = int(L.load().hs_tile_cta_sort_min())
    return _CTA_MIN


def tile_sort_cap():
    global _SORT_CAP
    if _SORT_CAP is None:
        _SORT_CAP = int(L.load().hs_tile_sort_cap())
    return _SORT_CAP


def launches_tiles(binner):
    """Kernel launches issued by Binner.bin_tiles: count, scan, scatter, the four list
    sorts (warp, CTA-cooperative, long-list, 64-bit fallback) (+ the two-level fallback's)."""
    n = 5 + getattr(binner, "launches_extra", 0)   # (the count runs inside the projection)
    if binner.mode == "two_level":
        n += 6 + launches_binning(1, binner.passes, True)
    return n


def launches_binning(total, passes, two_level=False):
    """Kernel launches issued by Binner.bin (emit (3 for the sorted emission), histogram,
    digit scan, one per pass, ranges) -- for the bench's gpu_launches count."""
    if not total:
        return 0
    return (3 if two_level else 1) + 2 + passes + 1


# -------------------------------------------------------------------- trainer

@dataclass
class StepResult:
    loss: float
    black_l1: np.ndarray
    per_frame: np.ndarray
    total_keys: int


class Trainer:
    """One batched training step per call, entirely on device.

    Mirrors S/train.py:214-260 (``train_step``) + the Adam groups (:164-199) and
    colour init (:258-278).  ``process_group`` (torch.distributed, NCCL) shards the
    global batch: every rank renders its frames and the flat gradient buffer is
    allreduced once per step; grads are scaled by 1/global_batch.
    """

    def __init__(self, avatar: AvatarParams, width, height, batch, lrs=None, color_init=True, threshold=0.1,
                 process_group=None, global_batch=None, frame_offset=0, rig: DeviceRig = None, deterministic=False):
        require_cuda()
        self.av = avatar
        # bitwise run-to-run reproducible gradients: the fused raster accumulates the splat
        # gradients and colour-init sums in int64 fixed point (HS_RASTER_DETERMINISTIC);
        # every other reduction of the step is already in a fixed order
        self.deterministic = bool(deterministic)
        self.rig = rig              # DeviceRig: frames computed from theta on device
        self.fused_raster = True    # hs_raster_train (False: hs_raster_fwd + hs_raster_bwd)
        self.two_level_binning = True   # depth order + 32-bit tile sort (False: one 64-bit sort)
        self.tile_binning = True        # tile-major binning (the two flags above: its fallback / off)
        self.W, self.H = int(width), int(height)
        self.B = int(batch)
        self.global_batch = int(global_batch or batch)
        self.frame_offset = int(frame_offset)
        self.lrs = (ctypes.c_float * 9)(*(lrs or default_lrs()))
        self.color_init = bool(color_init)
        self.threshold = float(threshold)
        self.pg = process_group
        self.step_count = 0
        d = avatar.device
        N, K, B, D = avatar.N, avatar.K, self.B, avatar.D
        self.tiles_x, self.tiles_y, self.tiles, self.tile_bits, self.frame_bits = key_layout(B, self.W, self.H)
        f32 = dict(dtype=torch.float32, device=d)
        self.grads = torch.zeros(avatar.size, **f32)
        self.m = torch.zeros(avatar.size, **f32)
        self.v = torch.zeros(avatar.size, **f32)
        self.visited = torch.zeros(N, dtype=torch.uint8, device=d)
        self.psi = torch.empty(B, K, **f32)
        self.gpsi = torch.empty(B, K, **f32)
        self.cache = torch.empty(B, 4 * D, **f32)
        self.mlp_scratch = torch.empty(B * (K + 2 * D) + 16, **f32)
        self.raw10 = torch.empty(B * 10 * N, **f32)
        self.records = torch.empty(B * N * 12, **f32)
        self.depth = torch.empty(B * N, **f32)
        self.radius = None          # optional debug output (set to a tensor to capture)
        # checker hook (unfused raster only): called on the host between the forward
        # raster and the adjoint; may edit pix_state (e.g. clear the L1 sign bits of
        # pixels a parity test excludes) on the current stream
        self.debug_before_backward = None
        self.capture_pixels = False     # fused raster also writes pix_T / pix_state (checker)
        self.speculative = True         # enqueue the raster before the step's host sync (guarded)
        self.profile_speculative = False  # keep speculating while stage events are recorded
        self.counts = torch.empty(B * N, dtype=torch.int32, device=d)
        self.nblocks = int(L.load().hs_scan_blocks(B * N))
        self.block_sums = torch.empty(self.nblocks, dtype=torch.int32, device=d)
        self.err = torch.full((1,), -1, dtype=torch.int64, device=d)
        self.pix_T = torch.empty(B * self.H * self.W, **f32)
        self.pix_state = torch.empty(B * self.H * self.W, dtype=torch.int32, device=d)
        self.maxw = torch.zeros(B * N, **f32)
        self.wsums = torch.zeros(B * N * 4, **f32)
        self.loss_partials = torch.empty(B * self.tiles * L.LOSS_PARTIALS_PER_TILE, **f32)
        self.loss_out = torch.empty(2 * B + 1, **f32)
        self.g_splat = torch.empty(B * N * 9, **f32)
        if self.deterministic:
            self.g_splat_fx = torch.empty(B * N * 9, dtype=torch.int64, device=d)
            self.wsums_fx = torch.empty(B * N * 4, dtype=torch.int64, device=d)
        # the persistent raster's work counters + item order (zeroed once; per Trainer, so
        # Trainers on different streams / devices never share raster state)
        self.raster_ws = torch.zeros(int(L.load().hs_raster_workspace_size(B, self.W, self.H)), dtype=torch.uint8,
                                     device=d)
        self.g_raw14 = torch.empty(B * 14 * N, **f32)
        self.nparts = int(L.load().hs_blend_bwd_partials(N))
        self.gpsi_partials = torch.empty(B * K * self.nparts, **f32)
        self.n_init = torch.zeros(1, dtype=torch.int32, device=d)
        self.packed = torch.empty(N, dtype=torch.int64, device=d)
        self.est4 = torch.empty(N * 4, **f32)
        self.binner = Binner(d)
        self.binner.write_keys = False
        self.last_total = 0
        self.launches = 0           # libhs_b200 kernel launches issued so far
        self.events = None          # {stage: [(start, end), ...]} when profiling is enabled
        self._ci_done = False
        self._comm = None
        self._bucket_events = []
        self._rig_frames = None
        self._rig_event = None
        self._order_event = None
        self._cur = None                # the compute stream of the step in flight
        self._read_loss = False         # step_from_host: copy the losses to the host in the step
        self._slot_free = [None, None]  # step_from_host: per input buffer set, its last step's end
        self._loss_event = None
        self._side = None               # side stream: rig || mlp_fwd + blend_fwd, loss || backward,
        self._side_events = []          # base/delta Adam || mlp_bwd
        self._last_frames = None
        self._copy = None               # H2D copy stream of step_from_host
        self._targets_ready = None
        self._registered = {}           # page-locked caller arrays
        self._staging = {}
        self._dev_in = {}
        self._slot = 0                  # input buffer set of the next uploaded step
        self._pending = None            # (batch key, device inputs, event, slot) of a prefetch
        # host staging for the end-to-end path (pinned)

    # --------------------------------------------------------------- profiling
    def enable_profiling(self, on=True):
        """Record CUDA events around every stage (on the launching stream)."""
        self.events = {} if on else None

    def _mark(self, name):
        if self.events is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.setdefault(name, []).append([ev, None])
        return name

    def _done(self, name):
        if name is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events[name][-1][1] = ev

    def stage_ms(self):
        """{stage: total ms} over everything recorded since enable_profiling()."""
        torch.cuda.synchronize()
        return {k: sum(a.elapsed_time(b) for a, b in v) for k, v in (self.events or {}).items()}

    def _call(self, stage, name, *args, kernels=1):
        m = self._mark(stage)
        L.call(name, *args)
        self._done(m)
        self.launches += kernels

    # ------------------------------------------------------------------ forward
    def _frames(self, thetas, frames):
        if frames is not None:
            return frames
        if self.rig is None:
            raise ValueError("frames is None and the Trainer has no DeviceRig")
        if self._rig_frames is None:
            self._rig_frames = torch.empty(self.B, self.rig.F, 22, dtype=torch.float32, device=self.av.device)
        # the rig depends on theta only: it runs on a side stream concurrently with
        # mlp_fwd + blend_fwd, and project_fwd waits for it
        side = self._side_stream()
        side.wait_stream(self._cur)
        with torch.cuda.stream(side):
            m = self._mark("rig_frames")
            self.rig.frames(thetas, out=self._rig_frames, err=self.err)     # errors surface at the scan read
            self._done(m)
            ev = torch.cuda.Event()
            ev.record(side)
        self._rig_event = ev
        self.launches += 1
        return self._rig_frames

    def _tile_order(self, ranges, tile_bits, scanned):
        """The raster's longest-first tile order, built on the side stream while the
        lists are scattered and sorted; the raster waits for ``_order_event``."""
        side = self._side_stream()
        side.wait_event(scanned)
        with torch.cuda.stream(side):
            L.call("hs_raster_tile_order", self.B, self.W, self.H, _p(ranges), tile_bits, _p(self.raster_ws),
                   _stream())
            ev = torch.cuda.Event()
            ev.record(side)
        self._order_event = ev
        self.launches += 1
        return True

    def _side_stream(self):
        if self._side is None:
            # (HS_SIDE_PRIORITY=-1: the side stream -- rig, loss reduction, the one-rank Adam --
            # at high priority)
            self._side = torch.cuda.Stream(device=self.av.device,
                                           priority=int(os.environ.get("HS_SIDE_PRIORITY", "0")))
        return self._side

    def _forward_project(self, thetas, frames, cameras, zero=(None, None, None), order=False, speculate=None):
        av = self.av
        N, K, B = av.N, av.K, self.B
        self._cur = torch.cuda.current_stream()     # the step's compute stream (looked up once)
        s = _stream()
        frames = self._frames(thetas, frames)
        self._call("mlp_fwd", "hs_mlp_fwd", B, av.H, av.D, K, _p(av.mlp), _p(thetas), _p(self.cache), _p(self.psi),
                   _p(self.err), s)
        self._call("blend_fwd", "hs_blend_fwd", N, K, B, _p(av.base14), _p(av.deltas), _p(self.psi),
                   _p(self.raw10), s)
        F = frames.shape[-2] if frames.dim() == 3 else frames.numel() // (B * 22)
        # tile-major binning: the projection counts the tiles in the same pass
        tile_counts = self.binner.tile_count_buffer(B, self.W, self.H) if self.tile_binning else None
        rects = self.binner.tile_rects_buffer(B, N, self.W, self.H) if self.tile_binning else None
        if self._rig_event is not None:
            self._cur.wait_event(self._rig_event)
            self._rig_event = None
        self._call("project_fwd", "hs_project_avatar_fwd", B, N, F, self.W, self.H, _p(self.raw10), _p(av.base14),
                   _p(av.tri_index), _p(av.barycentric), _p(frames), _p(cameras), _p(self.records), _p(self.depth),
                   _p(self.counts), _p(self.block_sums), _p(self.binner.reset_depth_range()), _p(self.radius),
                   *(_p(z) for z in zero), _p(tile_counts), _p(rects), _p(self.err), s)
        if self.tile_binning:
            m = self._mark("bin_tiles")
            total, code = self.binner.bin_tiles(B, N, self.W, self.H, self.records, self.depth, self.counts,
                                                self.err, self._tile_order if order else None, counted=True,
                                                rects=rects, speculate=speculate)
            self._done(m)
            self.launches += launches_tiles(self.binner)
            # (the scan reset the error word after reading it into the summary)
            L.raise_device_error(code, self.frame_offset)
            self.last_total = total
            self._last_frames = frames
            return F, self.binner.result
        overlap = None
        if self.two_level_binning:
            def overlap():      # the depth order runs while the host waits for the key total
                self.binner.depth_order(B, N, self.depth)
            self.launches += 6        # depth order: histogram, digit scan, 4 passes
        m = self._mark("bin_scan+sync")
        total, code = self.binner.scan(self.block_sums, self.nblocks, self.err, overlap)
        self._done(m)
        self.launches += 1
        # the error word also carries a colour-init failure of the previous step's
        # fused Adam (read here, at the step's one host sync); reset after reading
        self.err.fill_(-1)
        L.raise_device_error(code, self.frame_offset)
        self.last_total = total
        self._last_frames = frames
        m = self._mark("bin_sort")
        res = self.binner.bin(B, N, self.W, self.H, self.records, self.depth, self.counts, total)
        self._done(m)
        self.launches += launches_binning(total, self.binner.passes, self.two_level_binning)
        return F, res

    def _cameras(self, cameras):
        if cameras.dim() == 1:
            cameras = cameras.view(1, 16).expand(self.B, 16).contiguous()
        return cameras

    # --------------------------------------------------------------------- step
    def step(self, thetas, targets, frames, cameras, backgrounds) -> StepResult:
        """thetas (B,H) f32, targets (B,H,W,4) u8 straight RGBA, frames (B,F,22) f32
        (or None: computed from thetas by the Trainer's DeviceRig),
        cameras (B,16) or (16,) f32, backgrounds (B,3) f32 -- all on the device."""
        av = self.av
        N, K, B = av.N, av.K, self.B
        cameras = self._cameras(cameras)
        self._bucket_events = []
        ci = self.color_init and not self._all_visited()
        det = self.deterministic and self.fused_raster
        # the raster's accumulators are zero-filled by the projection pass (the int64
        # fixed-point ones of the deterministic mode by a memset)
        zero = (None if det else self.g_splat, self.maxw if ci else None, self.wsums if ci and not det else None)
        if det:
            self.g_splat_fx.zero_()
            if ci:
                self.wsums_fx.zero_()
        self._order_event = None
        flags = L.RASTER_LOSS
        if ci:
            flags |= L.RASTER_MAXW_UNVISITED | L.RASTER_WSUMS
        if det:
            flags |= L.RASTER_DETERMINISTIC
        # d loss_b / d pred = sign / (H W 3) / B_global  (S/metrics.py:19-22, S/train.py:244)
        grad_scale = 1.0 / (self.H * self.W * 3.0) / self.global_batch

        def raster(vals, ranges, tile_bits, guard=None):
            # forward + adjoint of every pixel block in one pass (hs_raster_train)
            s = _stream()
            if self._targets_ready is not None:     # step_from_host: targets arrive on the copy stream
                self._cur.wait_event(self._targets_ready)
                self._targets_ready = None
            fl, kernels = flags, 2                  # tile order + the fused raster
            if self._order_event is not None:       # built on the side stream (see _tile_order)
                self._cur.wait_event(self._order_event)
                if self.binner.order_ready and (guard is not None or self.binner.mode == "tiles"):
                    fl |= L.RASTER_ORDER_READY
                    kernels = 1                     # (the order was counted in _tile_order)
            self._call("raster", "hs_raster_train", B, N, self.W, self.H, fl, _p(self.records), _p(vals),
                       _p(ranges), tile_bits, _p(backgrounds), _p(targets), _p(self.visited), _p(self.maxw),
                       _p(self.wsums_fx if det else self.wsums), _p(self.loss_partials), ctypes.c_float(grad_scale),
                       _p(self.g_splat_fx if det else self.g_splat),
                       _p(self.pix_T) if self.capture_pixels else None,
                       _p(self.pix_state) if self.capture_pixels else None,
                       ctypes.byref(guard) if guard is not None else None, _p(self.raster_ws), s, kernels=kernels)

        # fused raster: enqueued speculatively before the step's host sync (device-guarded,
        # see Binner.bin_tiles), so the GPU goes from the list sorts straight into it.  Not
        # while profiling: the stage events would then bracket the raster inside bin_tiles.
        spec = raster if (self.fused_raster and self.tile_binning and self.speculative and (self.events is None or self.profile_speculative)) else None
        F, (keys, vals, ranges, tile_bits, tiles) = self._forward_project(thetas, frames, cameras, zero,
                                                                          order=self.fused_raster, speculate=spec)
        frames = self._last_frames
        s = _stream()
        if self.fused_raster:
            if spec is None or not self.binner.spec_valid:
                raster(vals, ranges, tile_bits)
            if det:
                self._call("raster", "hs_fixed_to_float", B * N * 9, _p(self.g_splat_fx), _p(self.g_splat), 0, s)
                if ci:
                    self._call("raster", "hs_fixed_to_float", B * N * 4, _p(self.wsums_fx), _p(self.wsums), 1, s)
            if ci and self.pg is not None:
                self._color_collectives()   # on the comm stream, overlapping the rest of the backward
            # the loss is only read after the step: reduce it on the side stream
            side = self._side_stream()
            side.wait_stream(self._cur)
            with torch.cuda.stream(side):
                self._call("loss_reduce", "hs_loss_reduce", B, tiles, self.W, self.H, _p(self.loss_partials),
                           _p(self.loss_out), _stream(), kernels=2)
                if self._read_loss:      # step_from_host: the D2H read right behind the reduction
                    self._loss_host.copy_(self.loss_out, non_blocking=True)
                loss_ev = torch.cuda.Event()
                loss_ev.record(side)
            self._side_events.append(loss_ev)
            self._loss_event = loss_ev
        else:
            if self._targets_ready is not None:
                self._cur.wait_event(self._targets_ready)
                self._targets_ready = None
            self._call("raster_fwd", "hs_raster_fwd", B, N, self.W, self.H, flags, _p(self.records), _p(vals),
                       _p(ranges), tile_bits, _p(backgrounds), _p(targets), None, _p(self.visited), _p(self.pix_T),
                       _p(self.pix_state), None, _p(self.maxw), _p(self.wsums), _p(self.loss_partials), None,
                       _p(self.raster_ws), s)
            if ci and self.pg is not None:
                self._color_collectives()   # on the comm stream, overlapping the backward
            self._call("loss_reduce", "hs_loss_reduce", B, tiles, self.W, self.H, _p(self.loss_partials),
                       _p(self.loss_out), s, kernels=2)
            if self.debug_before_backward is not None:
                self.debug_before_backward(self)
            self._call("raster_bwd", "hs_raster_bwd", B, N, self.W, self.H, _p(self.records), _p(vals),
                       _p(ranges), tile_bits, _p(backgrounds), _p(self.pix_T), _p(self.pix_state), None,
                       ctypes.c_float(grad_scale), _p(self.g_splat), L.RASTER_RAW_MEAN, _p(self.raster_ws), s)
        # (both rasters leave g_splat's mean entries as the raw sums: the projection adjoint
        # applies the conic)
        self._call("project_bwd", "hs_project_avatar_bwd", B, N, F, _p(self.raw10), _p(av.base14), _p(av.tri_index),
                   _p(av.barycentric), _p(frames), _p(cameras), _p(self.g_splat), 1, _p(self.g_raw14), s)
        nparts = ctypes.c_int(0)
        self._call("blend_bwd", "hs_blend_bwd", N, K, B, _p(av.deltas), _p(self.psi), _p(self.g_raw14),
                   _p(self.grads), _p(self.grads[14 * N:]), _p(self.gpsi_partials), ctypes.byref(nparts), s,
                   kernels=int(L.load().hs_blend_bwd_kernels(N, K, B)))
        buckets = self.buckets()
        ci_mode = (2 if self.pg is not None else 1) if ci else 0
        self.step_count += 1
        if self.pg is not None:           # base + delta buckets reduce while mlp_bwd runs
            self._allreduce_buckets(buckets[:-1])
        else:
            # one rank: Adam on base + deltas (+ colour init) needs only blend_bwd's output;
            # it runs on the side stream while mlp_bwd runs
            side = self._side_stream()
            side.wait_stream(self._cur)
            with torch.cuda.stream(side):
                m = self._mark("adam")
                self._adam(0, 14 * N + 10 * K * N, ci_mode, _stream())
                self._done(m)
                ev = torch.cuda.Event()
                ev.record(side)
            self._side_events.append(ev)
        self._call("mlp_bwd", "hs_mlp_bwd", B, av.H, av.D, K, _p(av.mlp), _p(thetas), _p(self.cache),
                   _p(self.gpsi_partials), nparts.value, _p(self.gpsi), _p(self.mlp_scratch),
                   _p(self.grads[14 * N + 10 * K * N:]), s, kernels=2)
        if self.pg is not None:
            self._allreduce_buckets(buckets[-1:])
            # multi-tensor Adam per bucket (each waits only for its own reduction), colour
            # init fused into the bucket holding the base colours
            m = self._mark("adam")
            for i, (lo, hi) in enumerate(buckets):
                self._cur.wait_event(self._bucket_events[i])
                self._adam(lo, hi, ci_mode, s)
            self._done(m)
        else:
            m = self._mark("adam_mlp")
            self._adam(14 * N + 10 * K * N, av.size, 0, s)
            self._done(m)
        for ev in self._side_events:      # the step ends when the side-stream work has
            self._cur.wait_event(ev)
        self._side_events = []
        return self.loss_out

    def _adam(self, lo, hi, ci_mode, stream):
        av = self.av
        L.call("hs_adam_fused", av.N, av.K, av.mlp_size, _p(av.params), _p(self.grads), _p(self.m), _p(self.v),
               self.lrs, self.step_count, ADAM_BETAS[0], ADAM_BETAS[1], ADAM_EPS, lo, hi, ci_mode, self.B,
               _p(self.maxw), _p(self.wsums), _p(self.packed), _p(self.est4), ctypes.c_float(self.threshold),
               _p(self.visited), _p(self.n_init), _p(self.err), stream)
        self.launches += 1

    def buckets(self):
        """Flat-gradient buckets [lo, hi): the base block (holds the colour segment
        that colour init writes), the deltas in 4 basis groups, then the MLP (which
        is produced last, by mlp_bwd).  Boundaries are multiples of N (float4 Adam)."""
        av = self.av
        N, K = av.N, av.K
        out = [(0, 14 * N)]
        per = max(1, -(-K // 4))
        for k0 in range(0, K, per):
            out.append((14 * N + 10 * N * k0, 14 * N + 10 * N * min(K, k0 + per)))
        out.append((14 * N + 10 * K * N, av.size))
        return out

    def _comm_stream(self):
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=self.av.device)
        return self._comm

    def _allreduce_buckets(self, buckets):
        """Allreduce-sum each bucket on the comm stream after the work enqueued so far
        on the compute stream; records one event per bucket for its Adam launch."""
        import torch.distributed as dist
        comm = self._comm_stream()
        ready = torch.cuda.Event()
        ready.record()
        m = self._mark("allreduce")
        with torch.cuda.stream(comm):
            comm.wait_event(ready)
            for lo, hi in buckets:
                dist.all_reduce(self.grads[lo:hi], op=dist.ReduceOp.SUM, group=self.pg)
                ev = torch.cuda.Event()
                ev.record(comm)
                self._bucket_events.append(ev)
        self._done(m)

    def result(self) -> StepResult:
        """Host copy of the last step's losses (a device->host read)."""
        lo = self.loss_out.cpu().numpy()
        B = self.B
        return StepResult(float(lo[2 * B]), lo[B:2 * B].copy(), lo[:B].copy(), self.last_total)

    def _all_visited(self):
        # visited is one-way; the host answer is cached once color_init_done() saw True
        return self._ci_done

    def color_init_done(self) -> bool:
        """Host check (a sync) of ColorInitState.done (S/color_init.py:28-30)."""
        self._ci_done = bool(self.visited.bool().all().item())
        return self._ci_done

    def _color_collectives(self):
        """Multi-GPU colour-init exchange on the comm stream right after
        the forward raster: pack -> allreduce-MAX -> select -> allreduce-SUM.  The
        apply is fused into the Adam launch of the base bucket."""
        import torch.distributed as dist
        av = self.av
        comm = self._comm_stream()
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(comm):
            comm.wait_event(ready)
            cs = ctypes.c_void_p(comm.cuda_stream)
            L.call("hs_color_pack", self.B, av.N, self.frame_offset, _p(self.maxw), _p(self.visited),
                   _p(self.packed), cs)
            dist.all_reduce(self.packed, op=dist.ReduceOp.MAX, group=self.pg)
            L.call("hs_color_select", self.B, av.N, self.frame_offset, _p(self.packed), _p(self.wsums),
                   _p(self.est4), _p(self.err), cs)
            dist.all_reduce(self.est4, op=dist.ReduceOp.SUM, group=self.pg)
        self.launches += 2


    # ------------------------------------------------------------------ render
    def render(self, thetas, frames, cameras, backgrounds, out=None):
        """Forward-only batched render (S/dataset.py:163-172 without the mesh rig):
        returns images (B, H, W, 3) fp32 = C + T * background."""
        av = self.av
        cameras = self._cameras(cameras)
        self._order_event = None
        if out is None:
            out = torch.empty(self.B, self.H, self.W, 3, dtype=torch.float32, device=av.device)

        def raster(vals, ranges, tile_bits, guard=None):
            flags = L.RASTER_IMAGE
            if self._order_event is not None:       # built on the side stream (see _tile_order)
                self._cur.wait_event(self._order_event)
                if self.binner.order_ready and (guard is not None or self.binner.mode == "tiles"):
                    flags |= L.RASTER_ORDER_READY
            self._call("raster_fwd", "hs_raster_fwd", self.B, av.N, self.W, self.H, flags, _p(self.records),
                       _p(vals), _p(ranges), tile_bits, _p(backgrounds), None, None, None, None, None, _p(out),
                       None, None, None,
                       ctypes.byref(guard) if guard is not None else None, _p(self.raster_ws), _stream())

        spec = raster if (self.tile_binning and self.speculative and (self.events is None or self.profile_speculative)) else None
        F, (keys, vals, ranges, tile_bits, tiles) = self._forward_project(thetas, frames, cameras, order=True,
                                                                          speculate=spec)
        if spec is None or not self.binner.spec_valid:
            raster(vals, ranges, tile_bits)
        return out

    # -------------------------------------------------------------- end to end
    def _host_view(self, name, arr, dtype):
        """A CPU tensor over the caller's host array that the GPU can DMA from.

        Conforming arrays (C-contiguous, right dtype) are page-locked in place once
        (cudaHostRegister) and cached by address, so a caller cycling through a few
        frame buffers pays no host copy per step; anything else is copied into a
        pinned staging buffer."""
        a = np.asarray(arr)
        if a.dtype == dtype and a.flags.c_contiguous and a.nbytes >= (1 << 16):
            # register the array that owns the memory (views of one buffer share it)
            root = a
            while isinstance(root.base, np.ndarray):
                root = root.base
            if not root.flags.c_contiguous:
                root = a
            key = (root.__array_interface__["data"][0], root.nbytes)
            hit = self._registered.get(key)
            if hit is None:
                t = torch.from_numpy(root)
                if L.load().hs_host_register(ctypes.c_void_p(t.data_ptr()), root.nbytes) == L.HS_OK:
                    if len(self._registered) >= 32:          # bounded: drop the oldest
                        old_key, (old_a, old_t) = next(iter(self._registered.items()))
                        torch.cuda.synchronize()
                        L.load().hs_host_unregister(ctypes.c_void_p(old_t.data_ptr()))
                        del self._registered[old_key]
                    hit = self._registered[key] = (root, t)  # keeps the memory alive
                # else: overlapping / unsupported range -> pinned staging below
            if hit is not None:
                return torch.from_numpy(a)
        a = np.ascontiguousarray(a, dtype)
        st = self._staging.get(name)
        if st is None or st.shape != a.shape:
            st = self._staging[name] = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        st.numpy()[...] = a
        return st

    def _device_buf(self, name, host, slot=0):
        key = (slot, name)
        d = self._dev_in.get(key)
        if d is None or d.shape != host.shape or d.dtype != host.dtype:
            d = self._dev_in[key] = torch.empty(host.shape, dtype=host.dtype, device=self.av.device)
        return d

    @staticmethod
    def _batch_key(arrays):
        return tuple((k, id(v), np.asarray(v).__array_interface__["data"][0], np.shape(v))
                     for k, v in sorted(arrays.items()) if v is not None)

    def _upload(self, slot, arrays):
        """Every input of one step H2D on the copy stream into buffer set `slot`;
        returns (device tensors, completion event)."""
        dt = {"thetas": np.float32, "targets": np.uint8, "frames": np.float32, "cameras": np.float32,
              "backgrounds": np.float32}
        dev = {}
        if self._slot_free[slot] is not None:
            # the step that last read this buffer set may still be in its backward
            self._copy.wait_event(self._slot_free[slot])
        with torch.cuda.stream(self._copy):
            for k, v in arrays.items():
                if v is None:
                    continue
                h = self._host_view(f"{k}{slot}", v, dt[k])
                d = self._device_buf(k, h, slot)
                d.copy_(h, non_blocking=True)
                dev[k] = d
            ev = torch.cuda.Event()
            ev.record(self._copy)
        return dev, ev

    def step_from_host(self, thetas, targets, frames, cameras, backgrounds, prefetch=None):
        """End-to-end step through host buffers (numpy): H2D copies, the device step
        and the D2H read of the losses.  Returns StepResult once the losses are on the
        host; the step's backward and Adam may still be running (stream-ordered before
        anything the caller enqueues next; torch.cuda.synchronize() waits for them).

        The small inputs go first on the compute stream; the targets (the bulk of the
        bytes) go on a copy stream and only the forward raster waits for them, so
        their transfer overlaps the MLP, blend, projection and sort.  frames may be
        None when the Trainer holds a DeviceRig (mesh frames computed from theta).

        ``prefetch`` = the next step's (thetas, targets, frames, cameras, backgrounds):
        its copies are enqueued on the copy stream right after this step's kernels
        (double-buffered device inputs), so they run under this step's compute and the
        next call finds its inputs on the device -- the input pipeline of a training loop."""
        if self._copy is None:
            self._copy = torch.cuda.Stream(device=self.av.device)
            self._loss_host = torch.empty(2 * self.B + 1, dtype=torch.float32, pin_memory=True)
        arrays = {"thetas": thetas, "targets": targets, "frames": frames, "cameras": cameras,
                  "backgrounds": backgrounds}
        key = self._batch_key(arrays)
        cur = torch.cuda.current_stream()
        if self._pending is not None and self._pending[0] == key:
            _, dev, ev, slot = self._pending
            self._pending = None
            cur.wait_event(ev)
            d = dev["targets"]
        else:
            if self._pending is not None:
                # a prefetch of a different batch may still be writing (device side) into
                # the buffer set and pinned staging this upload reuses: let it land first
                self._pending[2].synchronize()
                self._pending = None
            slot = self._slot
            small = {"thetas": (thetas, np.float32), "cameras": (cameras, np.float32),
                     "backgrounds": (backgrounds, np.float32)}
            if frames is not None:
                small["frames"] = (frames, np.float32)
            dev = {}
            for k, (v, dt) in small.items():
                h = self._host_view(f"{k}{slot}", v, dt)
                dd = self._device_buf(k, h, slot)
                dd.copy_(h, non_blocking=True)
                dev[k] = dd
            h = self._host_view(f"targets{slot}", targets, np.uint8)
            d = self._device_buf("targets", h, slot)
            self._copy.wait_stream(cur)
            with torch.cuda.stream(self._copy):
                d.copy_(h, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(self._copy)
            self._targets_ready = ready
        # the losses are reduced and copied to the host on the side stream right after the
        # forward raster; the host waits for that copy only, not for the backward and
        # Adam, so it enqueues the next step while this one finishes
        self._read_loss = self.fused_raster
        try:
            self.step(dev["thetas"], d, dev.get("frames"), dev["cameras"], dev["backgrounds"])
        finally:
            self._read_loss = False
        loss_ready = self._loss_event if self.fused_raster else None
        if loss_ready is None:
            self._loss_host.copy_(self.loss_out, non_blocking=True)
        done = torch.cuda.Event()
        done.record(cur)                  # this buffer set is free once the step has finished
        self._slot_free[slot] = done
        self._slot = 1 - slot
        if prefetch is not None:
            nxt = dict(zip(("thetas", "targets", "frames", "cameras", "backgrounds"), prefetch))
            ndev, nev = self._upload(self._slot, nxt)
            self._pending = (self._batch_key(nxt), ndev, nev, self._slot)
        if loss_ready is not None:
            loss_ready.synchronize()
        else:
            cur.synchronize()
        lo = self._loss_host.numpy()
        B = self.B
        return StepResult(float(lo[2 * B]), lo[B:2 * B].copy(), lo[:B].copy(), self.last_total)

    def close(self):
        """Unregister the page-locked caller arrays of step_from_host."""
        if self._registered:
            torch.cuda.synchronize()
            for a, t in self._registered.values():
                L.load().hs_host_unregister(ctypes.c_void_p(t.data_ptr()))
            self._registered.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def h2d_bytes(self, F, frames=True):
        return self.B * (self.av.H * 4 + self.H * self.W * 4 + (F * 22 * 4 if frames else 0) + 16 * 4 + 3 * 4)

    def d2h_bytes(self):
        return (2 * self.B + 1) * 4
