// Host-side internals shared by the C-ABI (svr_grid.cu) and the kernel launchers.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "svr.h"
#include "svr_device.cuh"

namespace svr_internal {

void set_error(const std::string& msg);
// Launchers report CUDA runtime failures by throwing the ABI's status exception
// (SVR_ERR_CUDA, caught by the entry point's guarded() wrapper); defined in svr_grid.cu.
[[noreturn]] void throw_cuda(cudaError_t e, const char* what);
// SM count of the current device (cached per device): persistent / grid-stride grids are
// sized in multiples of it.  Defined in svr_grid.cu.
unsigned sm_count();
// AABB of blocks coords4[0, n) folded into b[6] = {lo xyz, hi xyz} (svr_grads.cu)
void launch_bounds(const int32_t* coords4, uint64_t n, int32_t* b, cudaStream_t s);
#define SVR_LCK(expr)                                                            \
    do {                                                                         \
        const cudaError_t e_ = (expr);                                           \
        if (e_ != cudaSuccess) ::svr_internal::throw_cuda(e_, #expr);            \
    } while (0)

struct Status {
    int code;
    std::string msg;
};

// Launchers (svr_render.cu)
void launch_query(const svr_dev::GridView& g, const double* x, uint64_t n, double* sdf,
                  double* grad, double* rgb, double* logits, uint8_t* valid, cudaStream_t s);
void launch_march(const svr_dev::GridView& g, const double* o, const double* d, uint64_t n,
                  const uint32_t* order, double step, uint32_t max_samples, uint32_t* counts,
                  double* t, double* delta, cudaStream_t s, uint32_t* pkeys = nullptr,
                  uint32_t* pids = nullptr, unsigned long long* valid_counter = nullptr);
void launch_render_forward(const svr_dev::GridView& g, const double* o, const double* d,
                           uint64_t n, const uint32_t* order, const uint32_t* counts,
                           const double* t, uint32_t S, double step, double beta, float* rgb,
                           float* depth, float* normal, float* wsum,
                           unsigned long long* valid_counter, float4* rec, cudaStream_t s,
                           float4* zgrad = nullptr, uint8_t* zactive = nullptr, const uint32_t* zlist = nullptr,
                           const unsigned long long* zcount = nullptr);
// Non-pipelined backward (any max_samples; re-gathers the payload when rec == NULL).
void launch_render_backward(const svr_dev::GridView& g, const double* o, const double* d,
                            uint64_t n, const uint32_t* order, const uint32_t* counts,
                            const double* t, uint32_t S, double step, double beta,
                            const float* d_rgb, const float* d_depth, const float* d_normal,
                            const float4* rec, cudaStream_t s);
// Pipelined backward (records, max_samples <= 64, even); returns false if not applicable.
bool launch_render_backward_pipe(const svr_dev::GridView& g, const double* o, const double* d,
                                 uint64_t n, const uint32_t* order, const uint32_t* counts,
                                 const double* t, uint32_t S, double step, double beta,
                                 const float* d_rgb, const float* d_depth, const float* d_normal,
                                 const float4* rec, cudaStream_t s, int num_sms);
// Sort rays for locality; *sorted_ids points into ids or ids_alt.  post_march: keys / ids
// were written by the march (Morton code of each ray's first-sample block); otherwise the
// keys are computed here from the origin hash + octahedral-direction Morton code.
void launch_ray_order(const double* o, const double* d, uint64_t n, const svr_dev::GridView& g,
                      bool post_march, uint32_t* keys, uint32_t* ids, uint32_t* keys_alt,
                      uint32_t* ids_alt, void* tmp, size_t tmp_bytes, uint32_t** sorted_ids,
                      cudaStream_t s);
size_t ray_order_tmp_bytes(uint64_t n);

// Launchers (svr_activate.cu)
struct KeySet {
    unsigned long long* slots = nullptr;  // open addressing, kEmptyKey = free
    unsigned long long mask = 0;
    unsigned long long* list = nullptr;   // unique keys in insertion order
    unsigned long long cap = 0;           // capacity of `list` (== slots/2)
};
void launch_keyset_clear(KeySet& ks, cudaStream_t s);
// points -> base block keys; flags[0] |= 1 on an unpackable coordinate
void launch_points_to_keys(const double* xyz, uint64_t n, double L, KeySet ks,
                           unsigned long long* count, uint32_t* flags, cudaStream_t s);
void launch_depth_to_keys(const float* depth, const svr_camera* cams, uint32_t n_frames,
                          int32_t W, int32_t H, const double* scales, int32_t rows, int32_t cols,
                          double L, KeySet ks, unsigned long long* count,
                          unsigned long long* pixels, uint32_t* flags, double* tab, cudaStream_t s);
void launch_dilate(const unsigned long long* base, uint64_t nbase, int32_t R, KeySet ks,
                   unsigned long long* count, uint32_t* flags, cudaStream_t s);
void launch_filter_fresh(const svr_dev::GridView& g, const unsigned long long* keys, uint64_t n,
                         unsigned long long* fresh, unsigned long long* nfresh, cudaStream_t s);
size_t sort_keys_tmp_bytes(uint64_t n);
void launch_sort_keys(unsigned long long* keys, uint64_t n, void* tmp,
                      cudaStream_t s);
void launch_hash_insert(svr_dev::HashSlot* slots, unsigned long long mask,
                        const unsigned long long* keys, uint64_t n, uint32_t first_index,
                        int32_t* coords4, cudaStream_t s);
void launch_hash_find(const svr_dev::HashSlot* slots, unsigned long long mask,
                      const int32_t* coords3, uint64_t n, uint32_t* out, cudaStream_t s);

// Launchers (svr_grads.cu)
void launch_payload_in(float4* pay, float* weight, float* logits, uint32_t* vmask,
                       uint32_t* meta, uint32_t first, uint32_t n, int32_t C, const float* sdf,
                       const float* w, const float* rgb, const float* lg, cudaStream_t s);
void launch_payload_out(const float4* pay, const float* weight, const float* logits,
                        uint32_t first, uint32_t n, int32_t C, float* sdf, float* w, float* rgb,
                        float* lg, cudaStream_t s);
void launch_dense_build(const int32_t* coords4, const uint32_t* meta, uint32_t n,
                        const int32_t* lo, const int32_t* dim, uint32_t* dense, uint32_t* occ,
                        cudaStream_t s);
void launch_bdist(const uint32_t* occ, const int32_t* dim, uint8_t* out, uint8_t* tmp, cudaStream_t s);
// hash mode block-distance bricks (svr_grads.cu): superblock info + brick count (synchronises),
// then the bricks' occupancy and three separable distance passes
uint32_t launch_brick_assign(const int32_t* sb_dim, const uint8_t* sbdist, uint32_t* info, uint32_t* brick_sb,
                             uint32_t* counter, cudaStream_t s);
void launch_brick_fill(const int32_t* coords4, uint32_t n, const int32_t* sb_lo, const int32_t* sb_dim,
                       const uint32_t* info, const uint32_t* brick_sb, uint32_t n_bricks, uint8_t* bricks,
                       uint8_t* tmp, cudaStream_t s);
void launch_superblock_occ(const int32_t* coords4, uint32_t n, const int32_t* sb_lo, const int32_t* sb_dim,
                           uint32_t* occ, cudaStream_t s);
void launch_peer_allreduce(float4* const* planes, uint32_t world, uint32_t rank, const uint32_t* rows,
                           uint64_t n_rows, cudaStream_t s);
void launch_nbr_build(const svr_dev::GridView& g, const int32_t* coords4, uint32_t n, uint32_t* nbr,
                      cudaStream_t s);
void launch_grad_out(const float4* grad, uint32_t n, float* g_sdf, float* g_rgb, cudaStream_t s);
void launch_active_list(const uint8_t* active, uint32_t n, uint32_t* list,
                        unsigned long long* count, cudaStream_t s);
void launch_set_active(uint8_t* active, const uint8_t* mask, uint32_t n, cudaStream_t s);
void launch_grad_pack(const float4* grad, const uint32_t* blocks, uint64_t n, float4* out,
                      cudaStream_t s);
void launch_grad_unpack(float4* grad, const uint32_t* blocks, uint64_t n, const float4* in,
                        cudaStream_t s);
void launch_grad_zero_active(float4* grad, uint8_t* active, const uint32_t* list,
                             const unsigned long long* count, uint32_t n_max, cudaStream_t s,
                             unsigned ctas_per_sm = 16);

// Launchers (svr_regularize.cu)
void launch_sample_uniform(const int32_t* coords4, uint32_t A, double L, uint64_t n, uint64_t seed,
                           double* out, cudaStream_t s);
void launch_eikonal_stats(const svr_dev::GridView& g, const double* x, uint64_t n, double* sums,
                          cudaStream_t s);
void launch_eikonal_scatter(const svr_dev::GridView& g, const double* x, uint64_t n, double coef,
                            cudaStream_t s);
void launch_rmsprop(float4* pay, float4* grad, float4* rms, uint8_t* active, const uint32_t* list,
                    const unsigned long long* count, uint32_t n_max, float lr, float alpha, float eps,
                    cudaStream_t s);

// Fusion + de-noising (svr_fusion.cu)
void launch_fuse(const int32_t* coords4, uint32_t n_blocks, const svr_camera* cams, uint32_t n_frames,
                 int32_t W, int32_t H, int32_t C, const float* depth, const float* rgb, const float* sem,
                 const double* scales, int32_t rows, int32_t cols, double h, double mu, long long* fsum,
                 uint32_t* fcount, unsigned long long* counters, cudaStream_t s);
void launch_fuse_finalize(const long long* fsum, const uint32_t* fcount, uint32_t n_blocks, int32_t C,
                          int flags, float4* pay, float* weight, float* logits, uint32_t* vmask,
                          uint32_t* meta, cudaStream_t s);
size_t denoise_smem(int radius);
void launch_denoise(const svr_dev::GridView& g, const int32_t* coords4, float4* pay_out, float* logits_out,
                    int32_t radius, const double* gw, cudaStream_t s);

// Refinement losses (svr_losses.cu); acc = 16 doubles of device scratch (see LossArgs)
void launch_render_losses(uint64_t n, const float* rgb, const float* depth, const float* normal,
                          const float* wsum, const float* tgt, const float* pdepth, const float* pnormal,
                          const uint32_t* cam_idx, const svr_camera* cams, double lambda_d, double lambda_n,
                          float* d_rgb, float* d_depth, float* d_normal, double* acc, cudaStream_t s);

// Refinement batch + Eikonal band points (svr_refine.cu)
void launch_sample_frame_rays(const svr_camera* cams, uint32_t n_frames, int32_t W, int32_t H,
                              uint32_t rays_per_image, uint64_t n, uint64_t seed, const float* rgb_img,
                              const float* depth_img, const float* normal_img, double* o, double* d, float* tgt,
                              float* pdepth, float* pnormal, uint32_t* cam_idx, uint32_t* pixel, cudaStream_t s);
uint64_t band_points(const double* o, const double* d, const uint32_t* counts, const double* t,
                     const float4* rec, uint64_t n, uint32_t S, float band, uint32_t* scratch, void* tmp,
                     size_t tmp_bytes, uint64_t cap, double* pts, cudaStream_t s);
size_t band_points_tmp_bytes(uint64_t n);

// Marching cubes (svr_mesh.cu): the last mesh of a handle, device resident.
struct MeshBufs {
    double* v = nullptr;   // [nv][3] vertices
    double* n = nullptr;   // [nv][3] unit normals
    double* c = nullptr;   // [nv][3] colours in [0, 1]
    int32_t* l = nullptr;  // [nv] argmax labels
    int32_t* t = nullptr;  // [nt][3] triangles
    uint64_t nv = 0, nt = 0, cap_v = 0, cap_t = 0;
    void reserve(uint64_t nv, uint64_t nt);
    void release();
    ~MeshBufs() { release(); }
};
// Needs the lookup structures (dense / hash + neighbour table) of the current grid.
void run_marching_cubes(const svr_dev::GridView& g, const int32_t* coords4, const uint32_t* nbr,
                        const int32_t* lo_block, double iso, MeshBufs& out, cudaStream_t s);

}  // namespace svr_internal
