// svr.hpp -- header-only C++ host mirror of the reference grid / renderer interface over
// the C-ABI in svr.h.  Names, argument meaning and error behaviour follow the reference
// (/root/reference/proj/src/core/grid.hpp:100-223, allocation.hpp:13-29, grid_io.hpp:14-15,
// meshing.hpp:10-28, mesh_io.hpp:12, errors.hpp:8-31; renderer ops per SPEC.md:268-319,
// fusion per SPEC.md:207-233), so code written against
// svr::SparseDenseGrid switches to the B200 build by changing the include and namespace:
//
//     #include "svr.hpp"                       // instead of "core/grid.hpp" + friends
//     svr::b200::SparseDenseGrid grid(0.015, 8, 4);
//     svr::b200::allocate_for_frames(grid, frames, nullptr, 2);
//     grid.render_forward(o, d, n, step, 64, beta, out);  grid.render_backward(dC, dD, dN);
//
// Status codes become the reference's exception types.  Arrays are plain pointers (host or
// device), so there is no Eigen in the interface.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "svr.h"

namespace svr::b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {  // errors.hpp:12-15
    using Error::Error;
};
struct DataError : Error {  // errors.hpp:17-20
    using Error::Error;
};
struct DivergedError : Error {  // errors.hpp:22-25
    using Error::Error;
};
struct CapacityError : Error {  // errors.hpp:27-31
    CapacityError(const std::string& what, std::size_t unallocated)
        : Error(what), unallocated_blocks(unallocated) {}
    std::size_t unallocated_blocks = 0;
};
struct CudaError : Error {
    using Error::Error;
};

inline void check(int status, const svr_alloc_report* rep = nullptr) {
    if (status == SVR_OK) return;
    const std::string msg = svr_last_error();
    switch (status) {
        case SVR_ERR_CONFIG: throw ConfigError(msg);
        case SVR_ERR_DATA: throw DataError(msg);
        case SVR_ERR_DIVERGED: throw DivergedError(msg);
        case SVR_ERR_CAPACITY: throw CapacityError(msg, rep ? rep->unallocated : 0);
        default: throw CudaError(msg);
    }
}

struct BlockCoord {  // grid.hpp:11-14
    std::int32_t x = 0, y = 0, z = 0;
};

using AllocationReport = svr_alloc_report;  // allocation.hpp:13-17
using Camera = svr_camera;                  // camera.hpp:16-29 (row-major R, camera-to-world)

struct RenderOutputs {  // render_ray outputs per ray
    float* rgb = nullptr;     // [n][3]
    float* depth = nullptr;   // [n]
    float* normal = nullptr;  // [n][3], world frame, un-normalised
    float* wsum = nullptr;    // [n]
    std::uint32_t* n_samples = nullptr;
};

class SparseDenseGrid {
public:
    static constexpr std::uint32_t kInvalidBlock = SVR_INVALID_BLOCK;
    static constexpr std::size_t kDefaultCapacity = std::size_t(1) << 21;

    SparseDenseGrid(double voxel_size, int block_res, int label_channels,
                    std::size_t capacity = kDefaultCapacity, int device = 0) {
        check(svr_grid_create(voxel_size, block_res, label_channels, capacity, device, &g_));
    }
    explicit SparseDenseGrid(svr_grid* adopt) : g_(adopt) {}
    SparseDenseGrid(const SparseDenseGrid&) = delete;
    SparseDenseGrid& operator=(const SparseDenseGrid&) = delete;
    SparseDenseGrid(SparseDenseGrid&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}
    ~SparseDenseGrid() {
        if (g_) svr_grid_destroy(g_);
    }

    svr_grid* handle() const { return g_; }
    svr_grid_info info() const {
        svr_grid_info i{};
        check(svr_grid_get_info(g_, &i));
        return i;
    }
    double voxel_size() const { return info().voxel_size; }
    int block_res() const { return info().block_res; }
    int label_channels() const { return info().label_channels; }
    double block_extent() const { return voxel_size() * block_res(); }
    std::size_t capacity() const { return info().capacity; }
    std::size_t block_count() const { return info().block_count; }
    bool empty() const { return block_count() == 0; }

    // find_block / allocate_block (grid.hpp:156-159)
    std::uint32_t find_block(const BlockCoord& c) const {
        std::uint32_t idx = kInvalidBlock;
        check(svr_grid_find(g_, &c.x, 1, &idx));
        return idx;
    }
    std::uint32_t allocate_block(const BlockCoord& c) {
        std::uint32_t idx = kInvalidBlock;
        check(svr_grid_allocate_blocks(g_, &c.x, 1, &idx));
        return idx;
    }
    std::vector<BlockCoord> coords() const {
        std::vector<BlockCoord> out(block_count());
        if (!out.empty()) check(svr_grid_coords(g_, &out[0].x));
        return out;
    }

    // payload in the reference's VoxelBlock layout (grid.hpp:62-66)
    void set_payload(std::uint32_t first, std::uint32_t n, const float* sdf, const float* weight,
                     const float* rgb, const float* logits) {
        check(svr_grid_set_payload(g_, first, n, sdf, weight, rgb, logits));
    }
    void get_payload(std::uint32_t first, std::uint32_t n, float* sdf, float* weight, float* rgb,
                     float* logits) const {
        check(svr_grid_get_payload(g_, first, n, sdf, weight, rgb, logits));
    }

    // query_sdf / query_sdf_with_gradient (grid.hpp:177-179), batched; fp64 like CornerCacheD
    bool query_sdf_with_gradient(const double x[3], double& sdf, double grad[3]) const {
        std::uint8_t valid = 0;
        check(svr_query(g_, x, 1, &sdf, grad, nullptr, nullptr, &valid));
        return valid != 0;
    }
    bool query_sdf(const double x[3], double& sdf) const {
        std::uint8_t valid = 0;
        check(svr_query(g_, x, 1, &sdf, nullptr, nullptr, nullptr, &valid));
        return valid != 0;
    }
    void query(const double* x, std::size_t n, double* sdf, double* grad, double* rgb,
               double* logits, std::uint8_t* valid) const {
        check(svr_query(g_, x, n, sdf, grad, rgb, logits, valid));
    }

    // march_ray (grid.hpp:190-198), batched
    void march(const double* o, const double* d, std::size_t n, double step,
               std::uint32_t max_samples, std::uint32_t* counts, double* t, double* delta) const {
        check(svr_march(g_, o, d, n, step, max_samples, counts, t, delta));
    }

    // renderer
    void render_forward(const double* o, const double* d, std::size_t n, double step,
                        std::uint32_t max_samples, double beta, const RenderOutputs& out) {
        check(svr_render_forward(g_, o, d, n, step, max_samples, beta, out.rgb, out.depth, out.normal,
                                 out.wsum, out.n_samples));
    }
    void render_backward(const float* d_rgb, const float* d_depth, const float* d_normal) {
        check(svr_render_backward(g_, d_rgb, d_depth, d_normal));
    }
    void zero_grad() { check(svr_grad_zero(g_)); }
    void grads(float* g_sdf, float* g_rgb) const { check(svr_grad_get(g_, g_sdf, g_rgb)); }
    std::vector<std::uint32_t> active_blocks() const {
        std::vector<std::uint32_t> list(block_count() ? block_count() : 1);
        std::uint64_t count = 0;
        check(svr_active_blocks(g_, nullptr, list.data(), &count));
        list.resize(count);
        return list;
    }

    void set_stream(void* cuda_stream) { check(svr_grid_set_stream(g_, cuda_stream)); }
    void synchronize() const { check(svr_grid_synchronize(g_)); }
    void join() const { check(svr_grid_join(g_)); }

private:
    svr_grid* g_ = nullptr;
};

// allocate_for_points / allocate_for_frames (allocation.hpp:22-29)
inline AllocationReport allocate_for_points(SparseDenseGrid& grid, const double* xyz, std::size_t n,
                                            int dilation) {
    AllocationReport r{};
    check(svr_grid_activate_points(grid.handle(), xyz, n, dilation, &r), &r);
    return r;
}
inline AllocationReport allocate_for_frames(SparseDenseGrid& grid, const float* depth,
                                            const Camera* cams, std::uint32_t n_frames,
                                            const double* scales, int sf_rows, int sf_cols,
                                            int dilation) {
    AllocationReport r{};
    check(svr_grid_activate_depth(grid.handle(), depth, cams, n_frames, scales, sf_rows, sf_cols,
                                  dilation, &r),
          &r);
    return r;
}

// save_grid / load_grid (grid_io.hpp:14-15)
inline void save_grid(const SparseDenseGrid& grid, const std::string& path) {
    check(svr_grid_save_sdgv(grid.handle(), path.c_str()));
}
inline SparseDenseGrid load_grid(const std::string& path, int device = 0) {
    svr_grid* g = nullptr;
    check(svr_grid_load_sdgv(path.c_str(), device, &g));
    return SparseDenseGrid(g);
}

// fusion module: fuse_all = begin + frames + finalize; images as in svr.h
using FuseReport = svr_fuse_report;
inline FuseReport fuse_all(SparseDenseGrid& grid, const float* depth, const float* rgb, const float* semantic,
                           const Camera* cams, std::uint32_t n_frames, const double* scales, int sf_rows,
                           int sf_cols, double mu) {
    FuseReport r{};
    check(svr_fuse_begin(grid.handle(), (rgb ? SVR_FUSE_COLOR : 0) | (semantic ? SVR_FUSE_SEMANTIC : 0)));
    check(svr_fuse_frames(grid.handle(), depth, rgb, semantic, cams, n_frames, scales, sf_rows, sf_cols, mu, &r));
    check(svr_fuse_finalize(grid.handle()));
    return r;
}
inline void denoise(SparseDenseGrid& grid, double sigma_vox = 1.0, int radius = 1) {
    check(svr_denoise(grid.handle(), sigma_vox, radius));
}

// refinement: loss layer of backward_step, batch sampling, band points
using LossStats = svr_loss_stats;
inline LossStats render_losses(SparseDenseGrid& grid, std::uint64_t n, const RenderOutputs& out,
                               const float* tgt_rgb, const float* prior_depth, const float* prior_normal,
                               const std::uint32_t* cam_idx, const Camera* cams, std::uint32_t n_cams,
                               double lambda_d, double lambda_n, float* d_rgb, float* d_depth, float* d_normal) {
    LossStats st{};
    check(svr_render_losses(grid.handle(), n, out.rgb, out.depth, out.normal, out.wsum, tgt_rgb, prior_depth,
                            prior_normal, cam_idx, cams, n_cams, lambda_d, lambda_n, d_rgb, d_depth, d_normal, &st));
    return st;
}
inline void sample_frame_rays(SparseDenseGrid& grid, const Camera* cams, std::uint32_t n_frames, const float* rgb,
                              const float* depth, const float* normal, std::uint32_t images_per_batch,
                              std::uint32_t rays_per_image, std::uint64_t seed, double* o, double* d,
                              float* tgt_rgb, float* prior_depth, float* prior_normal, std::uint32_t* cam_idx) {
    check(svr_sample_frame_rays(grid.handle(), cams, n_frames, rgb, depth, normal, images_per_batch, rays_per_image,
                                seed, o, d, tgt_rgb, prior_depth, prior_normal, cam_idx, nullptr));
}
inline std::uint64_t band_points(SparseDenseGrid& grid, double band, std::uint64_t cap, double* out) {
    std::uint64_t n = 0;
    check(svr_band_points(grid.handle(), band, cap, out, &n));
    return n;
}

// Mesh + marching_cubes + export_ply (meshing.hpp:10-28, mesh_io.hpp:12): flat arrays in the
// reference's element order (vertices / normals / colors xyz per vertex, triangles ijk).
struct Mesh {
    std::vector<double> vertices, normals, colors;
    std::vector<std::int32_t> labels, triangles;
    std::size_t vertex_count() const { return labels.size(); }
    std::size_t triangle_count() const { return triangles.size() / 3; }
};
inline Mesh marching_cubes(SparseDenseGrid& grid, double iso = 0.0) {
    std::uint64_t nv = 0, nt = 0;
    check(svr_marching_cubes(grid.handle(), iso, &nv, &nt));
    Mesh m;
    m.vertices.resize(3 * nv), m.normals.resize(3 * nv), m.colors.resize(3 * nv);
    m.labels.resize(nv), m.triangles.resize(3 * nt);
    check(svr_mesh_get(grid.handle(), nv ? m.vertices.data() : nullptr, nv ? m.normals.data() : nullptr,
                       nv ? m.colors.data() : nullptr, nv ? m.labels.data() : nullptr,
                       nt ? m.triangles.data() : nullptr));
    return m;
}
// export_ply of the grid's last marching_cubes mesh (written from the device copy)
inline void export_ply(SparseDenseGrid& grid, const std::string& path) {
    check(svr_mesh_save_ply(grid.handle(), path.c_str()));
}

// Multi-GPU: sum the active-block gradients of the replicas (one per device) into every
// replica -- the cross-GPU form of the reference's per-worker accumulation
// (parallel.cpp:35-63).  Stream-ordered, no host synchronisation, when the
// devices reach each other's memory; NCCL otherwise (svr.h svr_reduce_grads_ex).
inline void reduce_grads(const std::vector<SparseDenseGrid*>& replicas, int mode = SVR_REDUCE_AUTO) {
    std::vector<svr_grid*> hs;
    for (SparseDenseGrid* g : replicas) hs.push_back(g->handle());
    check(svr_reduce_grads_ex(hs.data(), static_cast<std::uint32_t>(hs.size()), mode));
}

}  // namespace svr::b200
