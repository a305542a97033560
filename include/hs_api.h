/*
 * hs_api.h -- C ABI of the B200 (sm_100a) RGBAvatar training hot path.
 *
 * One shared library, libhs_b200.so (paper_2503_12886_b200/lib/), built from
 * paper_2503_12886_b200/csrc/*.cu with nvcc -gencode arch=compute_100a,code=sm_100a.
 *
 * Calling convention
 *   - Every buffer argument is a caller-owned DEVICE pointer (e.g. a torch
 *     tensor's data_ptr()); sizes are plain integers.  No torch types.
 *   - Every call enqueues work on the caller-given stream (a cudaStream_t passed
 *     as void*; NULL = legacy default stream) and returns without synchronizing.
 *   - No allocation happens inside the library.  Scratch is sized by the
 *     hs_*_size queries and allocated by the caller.
 *   - Return value: HS_OK or an HS_ERR_* status; hs_last_error() returns a
 *     thread-local message for the last failing call on the calling thread.
 *   - Re-entrant per stream; no global mutable state besides the thread-local
 *     error string.
 *
 * Data layout (fp32 unless stated; N Gaussians, K blendshapes, B frames):
 *   params   flat [base 14N | deltas K*10N | mlp]  with
 *            base  = [position 3N | rotation 4N (wxyz) | color 3N | scale 3N | opacity N]
 *            delta = [position 3N | rotation 4N | color 3N]        (one block per k)
 *            mlp   = [w1 D*H | b1 D | w2 D*D | b2 D | w3 K*D | b3 K]  (row-major)
 *            raw values: log-scale, opacity/color logits (S/gaussians.py:24-69).
 *   grads    same layout as params (the NCCL allreduce payload).
 *   raw10    B x [position 3N | rotation 4N | color 3N]  blended (pre-activation)
 *   g_raw14  B x 14N, the base layout.
 *   world14  B x 14N activated world Gaussians, the base layout (compat path).
 *   frames   B x F x 22: [rotation 9 (row-major, columns T,B,N) | quat 4 | tri 9
 *            (vertex-major)]  (S/binding.py:47-53 MeshFrames).
 *   cameras  B x 16: [R 9 row-major world->camera | t 3 | fx fy cx cy]
 *            (S/render.py:40-84).  All frames of a call share width/height.
 *   records  B x N x 12 splat records written by project:
 *            [mx my | conic a b c | opacity | qmax | bbox_rows | bbox_cols | r g b]
 *            bbox_* pack (lo | hi << 16) as uint32 bits; qmax = 2 ln(255 op) + 1e-9.
 *   depth    B x N camera-space z of each splat; counts B x N tiles touched.
 *   keys     uint64  frame << (tile_bits+32) | tile << 32 | float_bits(depth)
 *   values   uint32  Gaussian index n
 *   ranges   B x 2^tile_bits x uint2 [start, end) into the sorted key list
 *            (tile_bits = bit length of tiles-1; index = key >> 32)
 *   pixel    B x H x W: T_final (fp32) and state (uint32: stop | sign bits << 26)
 *   g_splat  B x N x 9 [g_mean x y | g_conic a 2b c | g_opacity | g_color r g b]
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/headsplat):
 *   see the per-function comments.
 */
#ifndef HS_API_H
#define HS_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HS_OK = 0,
    HS_ERR_SHAPE = 1,      /* -> ValueError          (e.g. model.py:133-134, render.py:56-59) */
    HS_ERR_NONFINITE = 2,  /* -> FloatingPointError  (render.py:204-208) */
    HS_ERR_ZERO_QUAT = 3,  /* -> FloatingPointError  (model.py:224-227) */
    HS_ERR_COLOR_INIT = 4, /* -> RuntimeError        (color_init.py:59-63) */
    HS_ERR_CUDA = 5
};

/* Error-code word written with atomicMin by device kernels (HS_NO_ERROR = none):
 *   bits 62-63 stage (0 frame-forward checks, 1 preprocess checks)
 *   bits 40-61 frame, bits 32-39 attribute, bits 0-31 Gaussian index
 * stage 0 attributes: 0 non-finite theta (model.py:135-136), 1 zero-norm quat (model.py:224-227)
 * stage 1 attributes: 0 position, 1 rotation, 2 scale, 3 opacity, 4 color (render.py:204-208)
 * stage 2 attribute 0: colour-init eligibility inconsistency (color_init.py:59-63)
 * stage 3 attributes: 0 degenerate UV triangle, 1 degenerate 3D triangle (binding.py:104-109);
 *         the index field holds the face */
#define HS_NO_ERROR 0xFFFFFFFFFFFFFFFFull

const char *hs_last_error(void);
int hs_version(void);
int hs_device_sm_count(int device);

/* ---- MLP (model.py:130-142 map_params, :145-162 mlp_backward) ----------- */
/* psi[B,K] and the per-frame cache[B, 4D] = (z1, h1, z2, h2); err gets a stage-0
 * attribute-0 code for a non-finite theta row. */
int hs_mlp_fwd(int B, int H, int D, int K, const float *mlp, const float *theta,
               float *cache, float *psi, unsigned long long *err, void *stream);
/* Sums the weight gradients over the B frames in frame order into g_mlp (written).
 * gpsi_partials[B*K][num_partials] come from hs_blend_bwd; scratch >= B*(K+2D) floats. */
int hs_mlp_bwd(int B, int H, int D, int K, const float *mlp, const float *theta,
               const float *cache, const float *gpsi_partials, int num_partials,
               float *gpsi, float *scratch, float *g_mlp, void *stream);
/* Number of floats in the mlp block. */
int64_t hs_mlp_size(int H, int D, int K);

/* ---- Blend (model.py:165-185 blend, :188-216 blend_backward + train.py:253-255) */
/* raw10[b] = base10 + sum_k psi[b,k] * delta_k  (k ascending, psi==0 skipped, fmaf). */
int hs_blend_fwd(int64_t N, int K, int B, const float *base14, const float *deltas,
                 const float *psi, float *raw10, void *stream);
/* Reduces over all B frames in-kernel:  g_base14 = sum_b g_raw14[b];
 * g_deltas[k] = sum_b psi[b,k] g_raw10[b];  gpsi partial sums per block.
 * Both outputs are written (not accumulated).  Returns the partial count in
 * *num_partials; gpsi_partials needs hs_blend_bwd_partials(N) * B * K floats.
 * Up to 16 frames: one fused pass (TMA tiles when N % 128 == 0 and the buffers are
 * 16-byte aligned, else register streaming); more frames (8-byte aligned buffers,
 * N >= 17): one streaming pass for g_base / g_deltas over all frames, then g_psi per
 * 128 frames -- no read-modify-write passes over the outputs. */
int hs_blend_bwd(int64_t N, int K, int B, const float *deltas, const float *psi,
                 const float *g_raw14, float *g_base14, float *g_deltas,
                 float *gpsi_partials, int *num_partials, void *stream);
int hs_blend_bwd_partials(int64_t N);
/* Kernel launches hs_blend_bwd issues for these sizes (aligned buffers). */
int hs_blend_bwd_kernels(int64_t N, int K, int B);

/* ---- Projection (render.py:132-230 preprocess; model.py:219-234 activate;
 *      binding.py:174-188 transform_to_deformed) -------------------------- */
/* Fused activate + transform + project for B frames x N Gaussians in one launch.
 * Writes records, depth, counts (tiles touched) and one partial sum of counts per
 * 256 items (block_sums[ceil(B*N/256)]); err gets the first error code. */
int hs_project_avatar_fwd(int B, int64_t N, int F, int width, int height,
                          const float *raw10, const float *base14, const int32_t *tri_index,
                          const float *bary, const float *frames, const float *cameras,
                          float *records, float *depth, uint32_t *counts,
                          uint32_t *block_sums, uint32_t *depth_range, float *radius,
                          float *zero_gsplat, float *zero_maxw, float *zero_wsums,
                          uint32_t *tile_counts, uint32_t *tile_rects, unsigned long long *err,
                          void *stream);
/* (zero_gsplat [B*N*9], zero_maxw [B*N], zero_wsums [B*N*4]: optional accumulators of
 *  the step's raster, zero-filled in the same pass -- NULL to skip.  tile_counts
 *  [B << tile_bits]: optional, hs_tile_count done in the same pass (zero on entry).
 *  tile_rects [B*N*2]: optional, per item its tile rectangle packed ty0 | ty1 << 8 | tx0 << 16
 *  | tx1 << 24 (ty0 > ty1 for items without keys) and a kept-tile mask (bit dy * w + dx;
 *  all ones for rectangles of more than 32 tiles), for hs_tile_fill / hs_bin_emit*; at most
 *  256 tiles per image axis.  With tile_rects the binning culls the tiles no pixel of which
 *  the splat's alpha >= 1/255 ellipse reaches (exact, oracle/binning.py:tile_mask): counts,
 *  tile_counts and every emitter then hold only the kept tiles.)
 * Projection of already-activated world Gaussians (compat preprocess).
 * radius (B*N, 0 for culled splats), x_cam (B*N*3) and cov_cam (B*N*9) are
 * optional outputs (NULL to skip) in both projection calls. */
int hs_project_world_fwd(int B, int64_t N, int width, int height, const float *world14,
                         const float *cameras, float *records, float *depth,
                         uint32_t *counts, uint32_t *block_sums, uint32_t *depth_range,
                         float *radius, float *x_cam, float *cov_cam, unsigned long long *err,
                         void *stream);
/* Adjoint of hs_project_avatar_fwd (render.py:432-497 _preprocess_backward,
 * binding.py:191-204 transform_backward, model.py:237-248 activate_backward):
 * g_splat[B,N,9] -> g_raw14[B,14N] (written).  raw_mean != 0: g_splat's mean entries are the
 * HS_RASTER_RAW_MEAN sums (hs_raster_train's), converted here with the recomputed conic. */
int hs_project_avatar_bwd(int B, int64_t N, int F, const float *raw10, const float *base14,
                          const int32_t *tri_index, const float *bary, const float *frames,
                          const float *cameras, const float *g_splat, int raw_mean, float *g_raw14,
                          void *stream);
/* Adjoint of hs_project_world_fwd: g_splat -> g_world14[B,14N] (written). */
int hs_project_world_bwd(int B, int64_t N, const float *world14, const float *cameras,
                         const float *g_splat, float *g_world14, void *stream);

/* ---- Binning (new; replaces render.py:221-223 + :380-386) */
int hs_scan_blocks(int64_t num_items);  /* = ceil(num_items / 256) */
/* Exclusive scan of block_sums -> block_offsets; summary[0] = total keys,
 * summary[1] = *err, summary[2] = depth_range[0] | depth_range[1] << 32 (float bits of
 * the smallest / largest depth that emits keys; depth_range = {0xFFFFFFFF, 0} before
 * the projection, optional).  The caller copies summary to pinned host memory: the
 * one device->host read of a training step. */
int hs_bin_scan(int num_blocks, const uint32_t *block_sums, uint32_t *block_offsets,
                const unsigned long long *err, const uint32_t *depth_range,
                unsigned long long *summary, void *stream);
/* Writes keys/values in (frame, n, ty, tx) order.  tile_rects: the projection's (NULL when
 * it had none): only the kept tiles of each item's rectangle are emitted. */
int hs_bin_emit(int B, int64_t N, int width, int height, const float *records,
                const float *depth, const uint32_t *counts, const uint32_t *block_offsets,
                const uint32_t *tile_rects, uint64_t *keys, uint32_t *values, void *stream);
/* Bytes of scratch for hs_sort_pairs. */
size_t hs_sort_workspace_size(int64_t num_keys);
/* Stable LSD radix sort (onesweep: one histogram kernel, then one decoupled
 * look-back kernel per 8-bit pass) of (keys, values) by the key bits in bit_mask;
 * digit windows outside the mask must be constant over the keys.  Ping-pongs
 * between (keys, values) and (keys_alt, values_alt); *result_in_alt tells which
 * pair holds the sorted output. */
int hs_sort_pairs(int64_t num_keys, uint64_t bit_mask, uint64_t *keys, uint32_t *values,
                  uint64_t *keys_alt, uint32_t *values_alt, void *workspace,
                  size_t workspace_bytes, int *result_in_alt, void *stream);
/* Diagnostics (-DHS_BIN_STATS builds; zeros otherwise): [keys emitted, keys whose
 * splat provably contributes to no pixel of the tile]; synchronous copy to host_out[2]. */
int hs_bin_stats(unsigned long long *host_out, int reset);
/* ---- Two-level binning (the training path): the same per-tile lists with 32-bit
 * sort keys.
 * hs_depth_order: stable sort of the B*N (frame, Gaussian) items by their float depth
 *   bits -> order[j] = item index (ties to the lower index).  Always 4 passes; the
 *   8-bit windows that depth_range ({min, max} emitted depth bits, written by the
 *   projection) shows constant copy through, so no host read is needed -- it can run
 *   while the host waits for hs_bin_scan.  keys_a/keys_b/order_alt are scratch (B*N),
 *   workspace hs_sort_workspace_size(B*N) bytes.
 * hs_bin_emit_sorted: each item in depth order writes its tiles' 32-bit keys
 *   frame << tile_bits | tile and values n (block sums + scan + emission); block_sums /
 *   block_offsets hold hs_scan_blocks(B*N) words.
 * hs_sort_pairs32: hs_sort_pairs for 32-bit keys (frame/tile bits only: 2 passes).
 * hs_tile_ranges32: ranges from the sorted 32-bit keys (zero-filled by the caller). */
int hs_depth_order(int64_t num_items, const float *depth, const uint32_t *depth_range, uint32_t *order,
                   uint32_t *order_alt, uint32_t *keys_a, uint32_t *keys_b, void *workspace,
                   size_t workspace_bytes, void *stream);
int hs_bin_emit_sorted(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                       const uint32_t *tile_rects, const uint32_t *order, uint32_t *block_sums,
                       uint32_t *block_offsets, uint32_t *keys, uint32_t *values, void *stream);
int hs_sort_pairs32(int64_t num_keys, uint32_t bit_mask, uint32_t *keys, uint32_t *values,
                    uint32_t *keys_alt, uint32_t *values_alt, void *workspace, size_t workspace_bytes,
                    int *result_in_alt, void *stream);
int hs_tile_ranges32(int64_t num_keys, const uint32_t *keys, uint32_t *ranges, void *stream);

/* ---- Tile-major binning (the training path; same lists as the sorts above)
 * hs_tile_count: each (frame, splat) with counts[i] > 0 adds one to every tile of its
 *   pixel bbox in tile_counts [B << tile_bits] (zero on entry; hs_tile_scan re-zeroes it).
 * hs_tile_scan: ranges [2 * (B << tile_bits)] (every entry written), scatter cursors
 *   [B << tile_bits], summary [4] = {key total, error word, depth range as hs_bin_scan,
 *   longest list} -- err is reset to HS_NO_ERROR after the read, and depth_range to
 *   {~0, 0} unless the longest list exceeds hs_tile_sort_cap() -- and, in lists
 *   [2 * (B << tile_bits)] / list_counts [1 + 2 * list_half, zero on first use; list_half
 *   >= 8 + ceil((B << tile_bits) / 1024), the same in every call], the lists the fill sorts
 *   per CTA (list_counts alternates halves between steps: no reset is needed).
 * hs_tile_fill: values [key total] (keys, when not NULL: the (frame, tile) key of each entry --
 *   the raster needs only values and ranges, so the training step passes NULL), each
 *   entry from the items' tile_rects (NULL: from the records' bboxes and counts); each
 *   list of at most hs_tile_cta_sort_min() - 1 entries in (depth, Gaussian index) order --
 *   the reference order.  Skipped on the device when summary[0] > capacity (grow the
 *   buffers, reset the cursors to the range starts and call again).  Longer lists are
 *   scattered but sorted by hs_tile_fill_longest (up to hs_tile_sort_cap()) or, past the
 *   cap, not at all: then bin that step with the two-level sort instead.
 *   With a fork context (hs_fork_create, caller-owned) the short lists sort on the
 *   context's side stream concurrently with the long ones, and the caller's stream joins
 *   it before the call returns (stream-ordered like any other call); fork == NULL sorts
 *   both on the caller's stream.  A context serves one caller at a time (one per Trainer
 *   / thread), so calls with different contexts are re-entrant. */
int hs_tile_sort_cap(void);
/* A fork context: a non-blocking side stream and two events on the device current at
 * creation; destroy it on the same device. */
void *hs_fork_create(void);
void hs_fork_destroy(void *fork);
/* Lists of hs_tile_cta_sort_min()..hs_tile_sort_cap() entries are sorted by
 * hs_tile_fill_longest (one CTA each), which the caller enqueues after hs_tile_fill when
 * the summary's longest list is in that range (arguments as hs_tile_fill). */
int hs_tile_cta_sort_min(void);
int hs_tile_fill_longest(int B, int64_t N, int width, int height, const float *depth, const uint32_t *ranges,
                         uint32_t *lists, uint32_t *list_counts, int list_half,
                         const unsigned long long *summary, uint64_t capacity, uint32_t *values, void *stream);
int hs_tile_count(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                  uint32_t *tile_counts, void *stream);
int hs_tile_scan(int B, int width, int height, uint32_t *tile_counts, uint32_t *ranges, uint32_t *cursor,
                 uint32_t *lists, uint32_t *list_counts, int list_half, unsigned long long *err,
                 uint32_t *depth_range, unsigned long long *summary, void *stream);
int hs_tile_fill(int B, int64_t N, int width, int height, const float *records, const uint32_t *counts,
                 const uint32_t *tile_rects, const float *depth, const uint32_t *ranges, uint32_t *cursor,
                 uint32_t *lists,
                 uint32_t *list_counts, int list_half, const unsigned long long *summary, uint64_t capacity,
                 uint32_t *keys, uint32_t *values, int flags, void *fork, void *stream);
/* hs_tile_fill flags: HS_FILL_CTA_SORT also sorts the lists of
 * hs_tile_cta_sort_min()..hs_tile_sort_cap() entries (a no-op on the device when there are
 * none), first on the fork's side stream -- for a caller that expects such lists (its
 * previous batch had them); otherwise hs_tile_fill_longest after the summary read. */
#define HS_FILL_CTA_SORT 1
/* ranges[frame*tiles + tile] = [start, end); caller zero-fills ranges first. */
int hs_tile_ranges(int64_t num_keys, const uint64_t *keys, uint32_t *ranges, void *stream);

/* ---- Raster (render.py:233-273 _composite_kernel, :339-377 _weight_sums_kernel,
 *      metrics.py:10-22 l1_loss, :80-85 composite_over, train.py:238-247) ----
 * The raster kernels are persistent: their work counters and item order live in a
 * caller-provided workspace of hs_raster_workspace_size(B, width, height) bytes
 * (16-byte aligned, zero-filled once at allocation; every launch leaves the counters
 * zeroed).  Launches on different workspaces are independent (re-entrant: several
 * streams / devices); launches sharing one workspace must be stream-ordered. */
enum {
    HS_RASTER_LOSS = 1,          /* fused L1 loss vs targets (u8 RGBA) composited over bg */
    HS_RASTER_IMAGE = 2,         /* write image[B,H,W,3] */
    HS_RASTER_MAXW_ALL = 4,      /* max blend weight per (frame, Gaussian) */
    HS_RASTER_MAXW_UNVISITED = 8,/* same, only for Gaussians with visited[n] == 0 */
    HS_RASTER_WSUMS = 16,        /* colour-init sums (sum w*target, sum w) for the same set */
    HS_RASTER_WSUMS_IMAGE = 32,  /* weight sums against wsum_image[B,H,W,3] (fp32) instead of the target */
    HS_RASTER_ORDER_READY = 64,  /* hs_raster_train / hs_raster_fwd: the tile order hs_raster_tile_order
                                    built for these ranges is in place (the call skips building it) */
    HS_RASTER_DETERMINISTIC = 128, /* hs_raster_train / hs_raster_fwd: g_splat and wsums are int64
                                    fixed-point accumulators (zeroed by the caller, converted with
                                    hs_fixed_to_float): bitwise run-to-run reproducible sums */
    HS_RASTER_RAW_MEAN = 256     /* hs_raster_bwd: g_splat[0:2] hold the raw sums (-sum dq dx, -sum dq dy)
                                    (g_mean = [[a b][b c]] times them, a b c the conic) -- what
                                    hs_raster_train always writes and hs_project_avatar_bwd takes */
};
size_t hs_raster_workspace_size(int B, int width, int height);
/* Optional guard of a raster enqueued before the host has read the step's binning summary
 * (hs_tile_scan's summary): the launch exits at once -- leaving every output untouched --
 * unless summary[0] <= capacity (the fill ran), summary[3] <= longest_max (every list
 * sorted by hs_tile_fill) and summary[1] == HS_NO_ERROR.  The caller re-launches it after
 * handling the rare case.  NULL (or summary NULL): no guard. */
typedef struct {
    const unsigned long long *summary;
    uint64_t capacity;
    uint32_t longest_max;
} hs_raster_guard_t;
/* The persistent raster's longest-list-first tile order for these ranges, written into
 * the workspace; lets a caller build it off the critical path (e.g. on a side stream
 * while the lists are sorted) and pass HS_RASTER_ORDER_READY to the raster that uses
 * the same workspace (ordered after this call and after the workspace's last raster). */
int hs_raster_tile_order(int B, int width, int height, const uint32_t *ranges, int tile_bits, void *workspace,
                         void *stream);
/* loss_partials holds B * num_tiles * HS_LOSS_PARTIALS_PER_TILE floats (one (L1,
 * black L1) pair per pixel block of the kernel, at most 8 per tile), reduced by
 * hs_loss_reduce. */
#define HS_LOSS_PARTIALS_PER_TILE 16
/* pix_T / pix_state (both or neither; both with the colour-init flags): per-pixel final
 * transmittance and stop index for a later hs_raster_bwd.  NULL: a forward no adjoint
 * follows (render) -- not tracked, not written. */
int hs_raster_fwd(int B, int64_t N, int width, int height, int flags, const float *records,
                  const uint32_t *values, const uint32_t *ranges, int tile_bits,
                  const float *backgrounds, const uint8_t *targets, const float *wsum_image,
                  const uint8_t *visited, float *pix_T, uint32_t *pix_state, float *image,
                  float *maxw, float *wsums, float *loss_partials, const hs_raster_guard_t *guard,
                  void *workspace, void *stream);
/* Adjoint (render.py:276-336 _backward_kernel).  grad_image (B,H,W,3) may be NULL:
 * then the L1 gradient sign(pred - target) * grad_scale recorded by the forward is used.
 * g_splat must be zero-filled by the caller (accumulated with atomics after a warp reduce).
 * flags: 0 (g_splat as documented) or HS_RASTER_RAW_MEAN. */
int hs_raster_bwd(int B, int64_t N, int width, int height, const float *records,
                  const uint32_t *values, const uint32_t *ranges, int tile_bits,
                  const float *backgrounds, const float *pix_T, const uint32_t *pix_state,
                  const float *grad_image, float grad_scale, float *g_splat, int flags, void *workspace,
                  void *stream);
/* Training-step raster: hs_raster_fwd (HS_RASTER_LOSS plus the colour-init flags)
 * and hs_raster_bwd with the L1 gradient sign(pred - target) * grad_scale, fused per
 * pixel block -- T, stop and the gradient stay in registers and the adjoint reuses
 * the forward's per-batch hit masks.  pix_T / pix_state are written only when
 * non-NULL.  g_splat must be zero-filled; loss_partials as hs_raster_fwd.  g_splat's mean
 * entries are the HS_RASTER_RAW_MEAN sums (the conic is applied by hs_project_avatar_bwd). */
int hs_raster_train(int B, int64_t N, int width, int height, int flags, const float *records,
                    const uint32_t *values, const uint32_t *ranges, int tile_bits,
                    const float *backgrounds, const uint8_t *targets, const uint8_t *visited,
                    float *maxw, float *wsums, float *loss_partials, float grad_scale, float *g_splat,
                    float *pix_T, uint32_t *pix_state, const hs_raster_guard_t *guard, void *workspace,
                    void *stream);
/* Diagnostics: raster counters accumulated when built with -DHS_RASTER_STATS (zeros
 * otherwise); synchronous copy to host_out[16]:
 *   forward [warp iterations, pixel tests, q <= qmax, alpha >= 1/255, iterations with
 *   no q pass, full-cover iterations, staged batches, 0], adjoint iterations by the
 *   number of contributing lanes [0, 1, 2, 3-4, 5-8, 9-16, 17-32, 0]. */
int hs_raster_stats(unsigned long long *host_out, int reset);
/* Diagnostics (-DHS_RASTER_TIMING builds only): per persistent raster warp of the last
 * launch, host_out[3 w .. 3 w + 2] = start and end %globaltimer (ns) and items processed. */
int hs_raster_warp_times(unsigned long long *host_out, int n);
/* out[i] = fixed[i] * 2^-48 (sums == 0: splat gradients) or * 2^-40 (sums != 0: the
 * colour-init weight sums) -- the HS_RASTER_DETERMINISTIC accumulators as float. */
int hs_fixed_to_float(int64_t n, const long long *fixed, float *out, int sums, void *stream);
/* loss_out[b] = sum|pred-target| / (H*W*3), loss_out[B+b] = black-bg L1,
 * loss_out[2B] = mean over frames. */
int hs_loss_reduce(int B, int num_tiles, int width, int height, const float *loss_partials,
                   float *loss_out, void *stream);

/* ---- Optimizer (optim.py:28-40; groups train.py:164-199) ---------------- */
/* lrs[9] = base position, rotation, color, scale, opacity, delta position,
 * rotation, color, mlp.  step >= 1 (bias correction). */
int hs_adam(int64_t N, int K, int64_t mlp_size, float *params, const float *grads,
            float *m, float *v, const float *lrs, int step, float beta1, float beta2,
            float eps, void *stream);
/* The same update restricted to flat elements [begin, end) -- one call per
 * allreduce bucket, so the update of bucket i overlaps the reduction of bucket
 * i+1 -- optionally fused with the colour-init apply that the
 * reference runs right after Adam (train.py:258-278; moments untouched):
 *   ci_mode 0: none;
 *   ci_mode 1: single rank -- hs_color_init semantics from maxw/wsums of B frames;
 *   ci_mode 2: across ranks -- hs_color_apply semantics from packed/est4 (after
 *              hs_color_pack/select and their two allreduces).
 * With ci_mode != 0 a range that touches the base-colour segment [7N, 10N) must
 * hold all of it.  Vectorised (float4) when N, begin and end are multiples of 4. */
int hs_adam_fused(int64_t N, int K, int64_t mlp_size, float *params, const float *grads,
                  float *m, float *v, const float *lrs, int step, float beta1, float beta2,
                  float eps, int64_t begin, int64_t end, int ci_mode, int B, const float *maxw,
                  const float *wsums, const int64_t *packed, const float *est4, float threshold,
                  uint8_t *visited, int *n_init, unsigned long long *err, void *stream);

/* ---- Colour init (train.py:263-278, color_init.py:45-80, model.py:260-263) */
/* best frame = first argmax_b maxw[b,n]; need = !visited && best > threshold;
 * base color[n] <- logit(clip(num/den, 1e-4, 1-1e-4)); visited[n] = 1.
 * n_init (optional, device int) counts initialized Gaussians. */
int hs_color_init(int B, int64_t N, const float *maxw, const float *wsums, float threshold,
                  uint8_t *visited, float *params, int *n_init, unsigned long long *err,
                  void *stream);
/* Multi-GPU colour init, three steps around two allreduces:
 *  pack:   packed[n] = max_b (float_bits(maxw[b,n]) << 32 | 0xFFFFFFFF - (frame_offset+b)),
 *          0 for visited n -- an allreduce-MAX picks the largest weight, then the
 *          smallest global frame (the reference's first-max argmax);
 *  select: est4[n] = (num/den rgb, 1) where this rank owns the winning frame, else 0
 *          -- then allreduce-SUM;
 *  apply:  need = !visited && weight > threshold -> logit write + visited. */
int hs_color_pack(int B, int64_t N, int frame_offset, const float *maxw, const uint8_t *visited,
                  int64_t *packed, void *stream);
int hs_color_select(int B, int64_t N, int frame_offset, const int64_t *packed, const float *wsums,
                    float *est4, unsigned long long *err, void *stream);
int hs_color_apply(int64_t N, const int64_t *packed, const float *est4, float threshold,
                   uint8_t *visited, float *params, int *n_init, void *stream);

/* ---- Device rig + tangent frames -------------------------
 * rig.py:57-66 rig_evaluate, quatmath.py:152-161 axis_angle_to_matrix,
 * binding.py:67-115 mesh_frames (_tbn_batch, polar_rotation), quatmath.py:105-149
 * matrix_to_quat.  frames[B][F][22] fp32 = [TBN 3x3 row-major (columns T, B, N) |
 * quaternion of its polar rotation factor (wxyz, unnormalised) | triangle
 * vertices 3x3], the layout hs_project_avatar_fwd reads.  Rig data in fp64
 * (base_vertices V x 3, expr_bases E x V x 3, uv_coords V x 2), faces int32 F x 3,
 * theta B x (E + 3) fp32 (expressions, then the axis-angle pose).  With
 * `vertices` (B x V x 3 fp64) non-NULL, theta is ignored and only mesh_frames
 * runs.  Degenerate triangles set a stage-3 error code in *err (face index). */
int hs_rig_frames(int B, int V, int F, int E, const double *base_vertices, const double *expr_bases,
                  const int32_t *faces, const double *uv_coords, const float *theta,
                  const double *vertices, float *frames, unsigned long long *err, void *stream);

/* ---- Device frame pool (stream.py:27-86) -------------------
 * out[r] = pool[slots[r]] for num_rows rows of row_bytes bytes each: the online
 * step gathers its sampled frames (u8 RGBA images, thetas) from the HBM-resident
 * pool into the step's contiguous buffers.  slots is a device int32 array. */
int hs_gather_rows(int num_rows, int64_t row_bytes, const int32_t *slots, const void *pool, void *out,
                   void *stream);

/* ---- Evaluation metrics (train.py:342-360, metrics.py:25-85) ----
 * For each frame b of pred (B,H,W,3 fp32) against target_rgba (B,H,W,4 u8)
 * composited over black, accumulates in fp64 (written, not accumulated):
 *   sums[5b + 0] = sum (pred - target)^2        -> psnr = 10 log10(3HW / sum), cap 99
 *   sums[5b + 1] = sum |pred - target|          -> l1 = sum / (3HW)
 *   sums[5b + 2 + c] = sum of the SSIM map of channel c over the (H-10)(W-10)
 *                      valid positions (Gaussian window 11, sigma 1.5, k1 .01, k2 .03)
 * H, W >= 11. */
int hs_image_metrics(int B, int H, int W, const float *pred, const uint8_t *target_rgba, double *sums,
                     void *stream);

/* Page-lock / release a host buffer for the end-to-end input path (failures leave no
 * sticky CUDA error; HS_ERR_CUDA + hs_last_error). */
int hs_host_register(void *ptr, size_t bytes);
int hs_host_unregister(void *ptr);

/* ---- Elementwise compat ops (model.py:219-248, binding.py:174-204) ------- */
int hs_activate_fwd(int64_t N, const float *raw14, float *act14, unsigned long long *err, void *stream);
int hs_activate_bwd(int64_t N, const float *raw14, const float *act14, const float *g_act14,
                    float *g_raw14, void *stream);
int hs_transform_fwd(int64_t N, const float *tangent14, const float *frames,
                     const int32_t *tri_index, const float *bary, float *world14, void *stream);
int hs_transform_bwd(int64_t N, const float *tangent14, const float *frames,
                     const int32_t *tri_index, const float *g_world14, float *g_tangent14,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HS_API_H */
