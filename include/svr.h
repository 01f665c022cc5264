/* svr.h -- C-ABI of the B200-native sparse-dense SDF rendering path
 * (libsvr_b200.so, built from paper_2305_13220_b200/csrc/).
 *
 * Drop-in boundary for the reference `svrecon` grid/renderer API
 * (/root/reference/proj/src/core/grid.hpp:100-223, allocation.hpp:22-29,
 * grid_io.hpp:14-15, renderer ops specified in SPEC.md:268-327).  The reference is a
 * C++ class library with no FFI of its own; each entry point below names the reference
 * member it replaces.  Plain pointers and sizes only -- no Eigen, no torch types.
 *
 * Memory: every array argument may be HOST memory (pageable or pinned) or DEVICE
 * memory on the grid's GPU; the library inspects each pointer
 * (cudaPointerGetAttributes).  A call whose array arguments are all device pointers is
 * asynchronous on the grid's stream (svr_grid_set_stream); a call with any host array
 * stages through device scratch and returns after the results are on the host.
 *
 * Errors: never throws across the ABI.  Status codes mirror the reference exceptions
 * (proj/src/core/errors.hpp:8-31) and svr_last_error() returns the thread's last
 * message.  Queries of unallocated / unobserved space are flags, not errors
 * (grid.cpp:240-261).
 *
 * Threading: one handle = one device + one stream.  Calls on one handle must be
 * serialised by the caller; activation must not overlap rendering.
 * Block resolution is specialised to 8 (the paper's 8^3 blocks); other
 * values return SVR_ERR_CONFIG.  Block coordinates must lie in [-2^20, 2^20) per axis
 * (64-bit packed keys, 21 bits per axis).
 */
#ifndef SVR_H
#define SVR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVR_ABI_VERSION 1

#define SVR_OK 0
#define SVR_ERR_CONFIG 2   /* ConfigError   (errors.hpp:12-15) */
#define SVR_ERR_DATA 3     /* DataError     (errors.hpp:17-20) */
#define SVR_ERR_DIVERGED 4 /* DivergedError (errors.hpp:22-25) */
#define SVR_ERR_CAPACITY 5 /* CapacityError (errors.hpp:27-31); see report->unallocated */
#define SVR_ERR_CUDA 6     /* CUDA runtime / device failure */

#define SVR_INVALID_BLOCK 0xFFFFFFFFu /* SparseDenseGrid::kInvalidBlock (grid.hpp:102) */

#define SVR_LOOKUP_AUTO 0  /* dense AABB index when it fits, else hash */
#define SVR_LOOKUP_HASH 1  /* always probe the hash table */
#define SVR_LOOKUP_DENSE 2 /* require the dense AABB index */

typedef struct svr_grid svr_grid;

/* Camera (camera.hpp:16-29): pinhole, camera-to-world x_w = R x_c + t, R row-major. */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R[9];
    double t[3];
} svr_camera;

/* AllocationReport (allocation.hpp:13-17) + CapacityError::unallocated_blocks. */
typedef struct {
    uint64_t blocks_added;
    uint64_t blocks_requested;
    uint64_t pixels_used;
    uint64_t unallocated;
} svr_alloc_report;

typedef struct {
    double voxel_size;
    int32_t block_res;
    int32_t label_channels;
    uint64_t capacity;
    uint64_t block_count;
    uint64_t hash_slots;
    int32_t bounds_lo[3]; /* min block coordinate (grid.hpp:222), valid iff block_count */
    int32_t bounds_hi[3]; /* max block coordinate */
    int32_t lookup_mode;  /* SVR_LOOKUP_HASH or SVR_LOOKUP_DENSE actually in use */
    int32_t device;
    uint64_t device_bytes; /* device memory owned by the handle */
} svr_grid_info;

typedef struct {
    uint64_t rays;           /* rays in the last render_forward */
    uint64_t samples;        /* marched samples (sum of per-ray counts) */
    uint64_t valid_samples;  /* samples whose 8 corners were all allocated and observed */
} svr_render_stats;

const char* svr_last_error(void);
int svr_abi_version(void);
int svr_device_count(int32_t* n);

/* SparseDenseGrid(voxel_size, block_res, label_channels, capacity) (grid.hpp:104-107).
 * capacity 0 = kDefaultCapacity (2^21).  Payload memory grows on demand. */
int svr_grid_create(double voxel_size, int32_t block_res, int32_t label_channels,
                    uint64_t capacity, int32_t device, svr_grid** out);
int svr_grid_destroy(svr_grid* g);
/* Bind the handle to a CUDA stream (cudaStream_t; cudaStreamLegacy = (void*)1 selects the
 * legacy default stream).  NULL restores a private non-blocking stream.  Device inputs must
 * be complete in the order of this stream when a call is issued. */
int svr_grid_set_stream(svr_grid* g, void* cuda_stream);
int svr_grid_synchronize(svr_grid* g);
/* Orders the handle's stream after the handle's pending internal work (a deferred
 * svr_grad_zero_active zeroing) without blocking the host; every call but render_forward
 * does this. */
int svr_grid_join(svr_grid* g);
int svr_grid_get_info(svr_grid* g, svr_grid_info* out);
int svr_grid_set_lookup(svr_grid* g, int32_t mode);
/* Performance knobs (results are unaffected; unknown keys -> SVR_ERR_CONFIG):
 *   "ray_sort"      bit 1: order the march by origin + octahedral direction; bit 0: order
 *                   forward / backward by the Morton code of each ray's first-sample block;
 *                   default 3 = both (random ray batches; a full image in raster order is
 *                   coherent already and renders faster with 0)
 *   "sort_min_rays" default 32768: smaller batches skip both orderings
 *   "records"       0/1, default 1: the forward leaves 32 B per sample so the backward skips
 *                   the re-gather (0 for inference: no backward context)
 *   "bwd_pipe"      0/1, default 1: the persistent cp.async.bulk-pipelined backward (needs
 *                   records and max_samples <= 64)
 *   "march_jump"    0/1, default 1: exact empty-space jumps over the block-distance field
 *   "zero_fused"    0/1, default 1: svr_grad_zero_active defers the zeroing to the next
 *                   render_forward's warps; every other call runs it first.  0: in order at
 *                   once
 *   "host_async"    0/1: render_forward / render_backward given PINNED host arrays return
 *                   without waiting; the transfers run on two internal copy streams through
 *                   double-buffered device slots so one step's copies overlap the previous
 *                   step's kernels; host outputs are valid, and host inputs may be reused,
 *                   only after svr_grid_synchronize
 *   "fuse_batch"    frames per fusion launch, 0 = auto */
int svr_grid_set_tuning(svr_grid* g, const char* key, int64_t value);

/* save_grid / load_grid (grid_io.cpp:37-97): SDGV v1; load keeps index = record order. */
int svr_grid_load_sdgv(const char* path, int32_t device, svr_grid** out);
int svr_grid_save_sdgv(svr_grid* g, const char* path);

/* allocate_block (grid.cpp:88-108) applied to coords[n][3] in order; idx_out[n] gets the
 * existing or new index.  Partial allocation then SVR_ERR_CAPACITY at capacity. */
int svr_grid_allocate_blocks(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out);
/* allocate_for_points (allocation.cpp:45-54): block of each point + L-inf dilation.
 * New blocks get indices in ascending packed-key (z, y, x) order. */
int svr_grid_activate_points(svr_grid* g, const double* xyz, uint64_t n, int32_t dilation,
                             svr_alloc_report* report);
/* allocate_for_frames (allocation.cpp:56-83): depth[n_frames][H][W] (<= 0 invalid),
 * optional per-frame ScaleField grids scales[n_frames][sf_rows][sf_cols] (NULL = 1). */
int svr_grid_activate_depth(svr_grid* g, const float* depth, const svr_camera* cams,
                            uint32_t n_frames, const double* scales, int32_t sf_rows,
                            int32_t sf_cols, int32_t dilation, svr_alloc_report* report);
/* find_block (grid.hpp:156) for coords[n][3]; SVR_INVALID_BLOCK when absent. */
int svr_grid_find(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out);
/* block_coord(i) for all blocks: out[block_count][3]. */
int svr_grid_coords(svr_grid* g, int32_t* out);

/* VoxelBlock payload (grid.hpp:62-66) for blocks [first, first+n), reference layout per
 * block: sdf[512], weight[512] (valid iff > 0), rgb[512][3], logits[512][C].
 * Any pointer may be NULL to skip that channel. */
int svr_grid_set_payload(svr_grid* g, uint32_t first, uint32_t n, const float* sdf,
                         const float* weight, const float* rgb, const float* logits);
int svr_grid_get_payload(svr_grid* g, uint32_t first, uint32_t n, float* sdf, float* weight,
                         float* rgb, float* logits);

/* query_sdf_with_gradient + color_at + logits_at over CornerCacheD (grid.cpp:157-261),
 * fp64 with the reference's operation order: x[n][3] -> sdf[n], grad[n][3], rgb[n][3],
 * logits[n][C], valid[n].  Invalid -> zeros.  Any output may be NULL. */
int svr_query(svr_grid* g, const double* x, uint64_t n, double* sdf, double* grad, double* rgb,
              double* logits, uint8_t* valid);

/* march_ray (grid.cpp:263-353) for o[n][3], d[n][3] (unit): counts[n],
 * t[n][max_samples], delta[n][max_samples] (bit-exact fp64).  t/delta may be NULL. */
int svr_march(svr_grid* g, const double* o, const double* d, uint64_t n, double step,
              uint32_t max_samples, uint32_t* counts, double* t, double* delta);

/* render_ray forward for n rays: rgb[n][3], depth[n], normal[n][3]
 * (world, un-normalised), wsum[n]; n_samples[n] optional.  Retains the context that
 * svr_render_backward consumes (device ray buffers must stay valid until then). */
int svr_render_forward(svr_grid* g, const double* o, const double* d, uint64_t n, double step,
                       uint32_t max_samples, double beta, float* rgb, float* depth,
                       float* normal, float* wsum, uint32_t* n_samples);
/* backward_step render part: upstream d_rgb[n][3], d_depth[n],
 * d_normal[n][3] of the last forward; accumulates into the grid's gradient planes
 * (grad_sdf / grad_color, grid.hpp:69) and marks active blocks. */
int svr_render_backward(svr_grid* g, const float* d_rgb, const float* d_depth,
                        const float* d_normal);
int svr_render_get_stats(svr_grid* g, svr_render_stats* out);

/* Gradient planes. grad_get: g_sdf[A][512], g_rgb[A][512][3]. */
int svr_grad_zero(svr_grid* g);
int svr_grad_get(svr_grid* g, float* g_sdf, float* g_rgb);
/* Active blocks (touched by a valid sample since the last grad_zero):
 * mask[A] (0/1, optional) and/or the ascending index list + count.  When every requested
 * output is device memory the call is stream-ordered with no host synchronisation (list then
 * receives A slots, entries past *count unspecified); a host count or list synchronises. */
int svr_active_blocks(svr_grid* g, uint8_t* mask, uint32_t* list, uint64_t* count);
/* Multi-GPU plumbing (device pointers): mark blocks from a union mask, then pack /
 * unpack the gradients of `blocks[n]` as [n][512][4] floats (g_sdf, g_r, g_g, g_b). */
int svr_active_set_mask(svr_grid* g, const uint8_t* mask);
int svr_grad_pack(svr_grid* g, const uint32_t* blocks, uint64_t n, float* out);
int svr_grad_unpack(svr_grid* g, const uint32_t* blocks, uint64_t n, const float* in);
/* Zero the gradients of the active blocks only and clear the active mask.  Stream-ordered;
 * with "zero_fused" (default) the zeros are stored by the next svr_render_forward's kernel,
 * and any other call on the handle (reads included) runs the pending zeroing first, so every
 * observable result is as if it ran here. */
int svr_grad_zero_active(svr_grid* g);

/* --- the losses / update around the rendering path ---------- */

/* sample_uniform (grid.cpp:355-370): n points uniform over the union of
 * allocated block volumes (uniform block, then uniform inside it), deterministic for a
 * seed.  The device uses a counter-based splitmix64 stream, NOT the reference's
 * mt19937_64 + libstdc++ distributions (whose stream is library-specific).
 * out[n][3]; SVR_ERR_DATA on an empty grid (grid.cpp:358). */
int svr_sample_uniform(svr_grid* g, uint64_t n, uint64_t seed, double* out);
/* Eikonal regulariser (Eq. 16/18): over the valid points of
 * x[n][3], loss = mean (|grad f(x)| - 1)^2 with f the fp64 trilinear interpolant; adds
 * scale * dloss/dsdf to the sdf gradient plane through the analytic trilinear weight
 * derivatives and marks active blocks.  *loss (mean) and *n_valid are returned. */
int svr_eikonal(svr_grid* g, const double* x, uint64_t n, double scale, double* loss,
                uint64_t* n_valid);
/* RMSProp on the active blocks (SPEC.md:320-327 refine, grid.hpp:70 rms_* buffers):
 * v = alpha v + (1 - alpha) g^2,  theta -= lr g / (sqrt(v) + eps)  for sdf and rgb, then the
 * active gradients are zeroed and the active mask cleared (fused).  State lives in the
 * handle (allocated on first use). */
int svr_rmsprop_step(svr_grid* g, float lr, float alpha, float eps);

/* ---- multi-GPU gradient reduction over peer memory ----
 * The NCCL path (svr_active_blocks -> svr_grad_pack -> all-reduce -> svr_grad_unpack) has a
 * fused alternative that reads and writes the ranks' gradient planes directly over NVLink:
 * every rank exports its plane (svr_grad_ipc_handle), opens the others' (svr_ipc_open, a
 * CUDA IPC mapping), and after a cross-rank barrier each rank reduces its 1/world slice of
 * the common ascending active-row list, summing in rank order and storing the sum into every
 * plane (svr_grad_peer_allreduce); a second barrier completes the step.  peer_planes[q] is
 * rank q's plane in this process (NULL at q == rank = own); world <= 8.  Handles stay valid
 * while the grid does not grow (re-export after allocating blocks). */
#define SVR_IPC_HANDLE_BYTES 64
int svr_grad_ipc_handle(svr_grid* g, void* handle_out, uint64_t* plane_bytes);
/* The gradient plane itself (float4 [capacity][512], device memory of the handle's GPU).
 * Work that reads it outside this API must follow svr_grid_join / svr_grid_synchronize (a
 * deferred svr_grad_zero_active zeroing may still be pending). */
int svr_grad_plane(svr_grid* g, void** ptr_out, uint64_t* plane_bytes);
int svr_ipc_open(const void* handle, int32_t device, void** ptr_out);
int svr_ipc_close(void* ptr);
int svr_grad_peer_allreduce(svr_grid* g, void* const* peer_planes, uint32_t world, uint32_t rank,
                            const uint32_t* rows, uint64_t n_rows);

/* ---- the whole reduction without host synchronisation ----
 * svr_reduce_grads: one process driving one handle per device (the replicas of one grid):
 * afterwards every handle holds the summed gradients of all handles in its active blocks
 * and the union active set.  Every step is stream-ordered on the handles' streams (cross-
 * device event waits, no host synchronisation) when the devices reach each other's memory
 * (NVLink / NVSwitch peer access, or handles sharing a device): union of the u8 flags by peer
 * reads, ascending compaction, each handle sums its 1/n slice of the rows over the n planes in
 * handle order and stores the sum into all n planes.  Otherwise (or mode SVR_REDUCE_NCCL) it
 * uses NCCL, loaded at run time: ncclCommInitAll over the handles' devices (one handle per
 * device), grouped ncclAllReduce(MAX) of the flags, pack -> grouped ncclAllReduce(SUM) ->
 * unpack; that path reads the union count on the host once.  Replaces the reference's
 * per-worker accumulation (proj/src/core/parallel.cpp:35-63). */
#define SVR_REDUCE_AUTO 0
#define SVR_REDUCE_PEER 1
#define SVR_REDUCE_NCCL 2
int svr_reduce_grads(svr_grid* const* grids, uint32_t n);
int svr_reduce_grads_ex(svr_grid* const* grids, uint32_t n, int32_t mode);

/* Multi-process form (one rank per GPU, e.g. torchrun): every rank exports its handle's
 * gradient plane, active flags and two interprocess events (svr_peer_export_get), the
 * exports are exchanged by any host channel, and svr_peer_group_open maps the others'.  One
 * reduction is three phases per rank, each stream-ordered:
 *   SVR_REDUCE_PUBLISH  record "backward done"
 *   SVR_REDUCE_SUM      wait every rank's "done"; union, compaction, own slice of the sum
 *                       over all planes; record "reduced"
 *   SVR_REDUCE_ADOPT    wait every rank's "reduced"; adopt the union active set
 * The caller runs a host-side barrier between consecutive phases (every rank must have
 * recorded an event before any rank waits on it) -- a CPU rendezvous, not a device
 * synchronisation.  A group is valid while the grid does not grow. */
#define SVR_REDUCE_PUBLISH 0
#define SVR_REDUCE_SUM 1
#define SVR_REDUCE_ADOPT 2
typedef struct svr_peer_export {
    uint8_t grad[64];        /* cudaIpcMemHandle_t of the gradient plane */
    uint8_t active[64];      /* cudaIpcMemHandle_t of the u8 active flags */
    uint8_t ev_done[64];     /* cudaIpcEventHandle_t, phase PUBLISH */
    uint8_t ev_reduced[64];  /* cudaIpcEventHandle_t, phase SUM */
    uint64_t n_blocks;
    int32_t device;
    int32_t reserved;
} svr_peer_export;
typedef struct svr_peer_group svr_peer_group;
int svr_peer_export_get(svr_grid* g, svr_peer_export* out);
int svr_peer_group_open(svr_grid* g, const svr_peer_export* all, uint32_t world, uint32_t rank,
                        svr_peer_group** out);
int svr_peer_reduce_phase(svr_peer_group* pg, int32_t phase);
int svr_peer_group_close(svr_peer_group* pg);

/* ---- fusion + de-noising (SPEC.md:207-233 module "fusion", PAPER Eq. 9-11, sec. 3.4.3) ----
 * The reference declares the state (VoxelBlock::sum_*, grid.hpp:59-68) but ships no code;
 * the contract is the SPEC's:
 *   association  voxel centre v*h -> Camera::project (camera.cpp:7-18) -> nearest pixel
 *                floor(p + 0.5) inside the image; depth > 0 and ScaleField value > 0
 *   distance     d = D(p) * phi(p) - z_v (positive in front of the surface), rejected when
 *                d < -mu, integrated as psi = min(d, mu)
 *   running mean sums in 32.32 fixed point + counts: any frame order gives bit-identical
 *                results; each |rgb|, |semantic| value < 2^19 and every
 *                per-voxel sum < 2^31 in magnitude
 *   finalize     sdf/rgb/logits = sum / count, logits scaled to unit L2 norm (Eq. 11),
 *                weight = count (grid.hpp:57-58), voxels never associated keep their
 *                payload with weight 0 (unobserved)
 * Images: depth [n][H][W] (<= 0 invalid), rgb [n][H][W][3], semantic [n][H][W][C] (the
 * reference ImageF32 interleave, frame.hpp:60-67), all frames one size; optional ScaleField
 * grids scales [n][rows][cols] as in svr_grid_activate_depth. */
#define SVR_FUSE_COLOR 1
#define SVR_FUSE_SEMANTIC 2
typedef struct {
    uint64_t frames;
    uint64_t in_view;    /* voxel-frame pairs projecting on a pixel with depth > 0, scale > 0 */
    uint64_t integrated; /* in_view pairs with d >= -mu */
    uint64_t rejected;   /* in_view pairs with d < -mu: behind the surface beyond the band */
} svr_fuse_report;
/* Open a fusion session (zeroed sums over the current blocks; blocks allocated later join
 * with zero sums).  flags = SVR_FUSE_COLOR | SVR_FUSE_SEMANTIC selects the fused channels;
 * the sdf is always fused.  Re-opening discards an open session. */
int svr_fuse_begin(svr_grid* g, int32_t flags);
/* fuse_frame over n_frames frames (fuse_all = begin + frames + finalize).  rgb / semantic
 * must be given exactly when the session's flags select them.  mu in (0, 2^19). */
int svr_fuse_frames(svr_grid* g, const float* depth, const float* rgb, const float* semantic,
                    const svr_camera* cams, uint32_t n_frames, const double* scales,
                    int32_t sf_rows, int32_t sf_cols, double mu, svr_fuse_report* report);
/* Write the means into the payload and close the session (sums released). */
int svr_fuse_finalize(svr_grid* g);
/* denoise(grid, sigma_vox, radius): every property of every valid voxel
 * (sdf, rgb, logits) becomes the Gaussian-weighted mean over the valid voxels of its
 * (2r+1)^3 neighbourhood, g(d) = exp(-d^2 / (2 sigma^2)) per axis, weights renormalised over
 * the valid set; weights / validity unchanged.  radius in [0, 4], sigma_vox > 0. */
int svr_denoise(svr_grid* g, double sigma_vox, int32_t radius);

/* ---- refinement losses (SPEC.md:286-319 backward_step, PAPER Eq. 12-14 / 23) ----
 * Per-ray upstream gradients for svr_render_backward from the rendered rgb[n][3], depth[n]
 * (distance along the ray), normal[n][3] (world, un-normalised), wsum[n] and the frame
 * targets: tgt_rgb[n][3], prior_depth[n] (<= 0 invalid, may be NULL), prior_normal[n][3]
 * (camera frame, all-zero invalid, may be NULL; needs cam_idx[n] into cams[n_cams]).
 *   participating ray: wsum > 0 (at least one valid sample)
 *   L_c = mean sum_ch |C - C*|                                   (colour L1)
 *   L_d = mean (t - (a D + b))^2, (a, b) = least squares of t on D over the batch (fp64 2x2
 *         normal equations; singular or fewer than 2 rays: a = 1, b = mean(t - D))
 *   L_n = mean |normalize(R^T N) - n*|_1 over rays with |R^T N| > 1e-12
 *   total = L_c + lambda_d L_d + lambda_n L_n (the Eikonal term: svr_eikonal with scale
 *   lambda_eik); d_rgb / d_depth / d_normal = d total / d output (d/d(a,b) = 0 at the LS
 *   optimum).  stats may be NULL (then no host synchronisation is needed). */
typedef struct {
    double L_c, L_d, L_n, total;
    double a, b;          /* depth prior fit */
    uint64_t n_c, n_d, n_n; /* rays in each term */
    int32_t singular;     /* depth fit fell back to a = 1 */
} svr_loss_stats;
int svr_render_losses(svr_grid* g, uint64_t n, const float* rgb, const float* depth, const float* normal,
                      const float* wsum, const float* tgt_rgb, const float* prior_depth,
                      const float* prior_normal, const uint32_t* cam_idx, const svr_camera* cams,
                      uint32_t n_cams, double lambda_d, double lambda_n, float* d_rgb, float* d_depth,
                      float* d_normal, svr_loss_stats* stats);

/* A refinement batch (SPEC.md RenderConfig: images_per_batch x rays_per_image rays) from the
 * frames rgb[F][H][W][3] / prior depth[F][H][W] / prior normal[F][H][W][3] (camera frame;
 * depth / normal may be NULL -> 0 targets; pass device arrays, host ones are staged per
 * call): image slot j takes frame splitmix(seed, j) mod F, ray i pixel splitmix(seed, i)
 * mod W*H; o = camera centre, d = Camera::ray_direction (camera.cpp:27-30, fp64 reference
 * order); targets are the pixel's values; cam_idx = frame, pixel = frame * W * H + y * W + x.
 * Outputs other than o / d may be NULL. */
int svr_sample_frame_rays(svr_grid* g, const svr_camera* cams, uint32_t n_frames, const float* rgb,
                          const float* depth, const float* normal, uint32_t images_per_batch,
                          uint32_t rays_per_image, uint64_t seed, double* o, double* d, float* tgt_rgb,
                          float* prior_depth, float* prior_normal, uint32_t* cam_idx, uint32_t* pixel);
/* sample_eikonal_points part (a): the samples of the last forward with
 * |sdf| < band (the forward's fp32 interpolated sdf; needs records = 1), as points
 * out[cap][3] in (ray, sample) order; *n_out = how many qualify (may exceed cap). */
int svr_band_points(svr_grid* g, double band, uint64_t cap, double* out, uint64_t* n_out);

/* ---- native refine loop (SPEC.md:320-327 refine; paper_2305_13220_b200/refine.py is the same
 * composition in Python, with data parallelism over a process group) ----
 * An svr_refiner owns device copies of the frames (rgb [F][H][W][3], optional depth prior
 * [F][H][W] and camera-frame normal prior [F][H][W][3]) and the per-step buffers; each
 * svr_refiner_step runs: batch sampling -> render_forward -> render_losses -> render_backward
 * -> band + uniform Eikonal points -> svr_eikonal(lambda_eik) -> svr_rmsprop_step(lr_i) with
 * lr_i = lr * gamma^(i / (steps - 1)).  stats (optional) gets the loss breakdown (its total
 * includes lambda_eik * L_eik), eik_loss (optional) the Eikonal mean. */
typedef struct {
    uint32_t rays_per_image, images_per_batch; /* RenderConfig: 1024 x 64 */
    double lambda_d, lambda_n, lambda_eik;     /* 0.1, 0.05, 0.1 */
    double lr, gamma, alpha, eps;              /* 1e-3, 0.1, RMSProp 0.99, 1e-8 */
    uint32_t max_samples, uniform_points, band_cap;
    uint64_t seed;
    double step, beta, mu; /* sample spacing (h/2), Laplace beta (2h), truncation (band mu/2) */
} svr_refine_config;
typedef struct svr_refiner svr_refiner;
void svr_refine_config_default(svr_refine_config* cfg); /* step / beta / mu left 0: set them */
int svr_refiner_create(svr_grid* g, const svr_camera* cams, uint32_t n_frames, const float* rgb,
                       const float* depth, const float* normal, const svr_refine_config* cfg,
                       svr_refiner** out);
int svr_refiner_step(svr_refiner* r, uint32_t i, uint32_t steps, svr_loss_stats* stats, double* eik_loss);
int svr_refiner_destroy(svr_refiner* r);

/* ---- meshing (meshing.hpp:23-28, meshing.cpp:168-273; mesh_io.cpp:30-68) ----
 * marching_cubes(grid, iso): iso surface over every cell whose 8 corners are allocated and
 * observed (cells across block faces included), vertices on cell edges by linear
 * interpolation, deduplicated per edge (first occurrence in (block, z, y, x, triangle)
 * order numbers the vertex), degenerate / zero-area (<= 1e-12) triangles dropped, normal /
 * colour / label from fp64 trilinear queries -- the reference's Mesh word for word.  The
 * mesh stays on the device (handle-owned) until the next call.  Edge keys need the block
 * AABB within 2^18 x 2^18 x 2^17 blocks (SVR_ERR_CONFIG otherwise). */
int svr_marching_cubes(svr_grid* g, double iso, uint64_t* n_vertices, uint64_t* n_triangles);
/* Copy the last mesh out: vertices / normals / colors [nv][3] f64, labels [nv] i32,
 * triangles [nt][3] i32 (host or device pointers; NULL skips). */
int svr_mesh_get(svr_grid* g, double* vertices, double* normals, double* colors, int32_t* labels,
                 int32_t* triangles);
/* export_ply (mesh_io.cpp:30-68) of the last mesh: binary little-endian PLY with float
 * xyz + normals, uchar rgb = lround(clamp(c) * 255), int label, uchar-count int triangles. */
int svr_mesh_save_ply(svr_grid* g, const char* path);
/* export_obj (mesh_io.cpp:155-164) of the last mesh: "v x y z" (9 significant digits) and
 * 1-based "f i j k" lines. */
int svr_mesh_save_obj(svr_grid* g, const char* path);

#ifdef __cplusplus
}
#endif

#endif
