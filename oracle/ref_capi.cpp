// TEST INFRASTRUCTURE ONLY -- C wrapper over the REFERENCE's own grid code
// (/root/reference/proj/src/core/*.cpp compiled verbatim, see Makefile) so Python
// tests can (a) validate the restated oracle against the reference and (b) time the
// reference CPU path for bench.py --impl reference.  The reference has no renderer
// (SURVEY.md section 0.2); svrr_render_* below restate SPEC.md:268-319 ON TOP of the
// reference API exactly as the spec prescribes: march_ray -> gather_corners into a
// retained CornerCache (grid.hpp:76-86) -> sdf_at / sdf_gradient_at / color_at ->
// Laplace density -> compositing; backward scatters from the retained caches into the
// reference's grad_sdf / grad_color shadow buffers (grid.hpp:69), rays split with
// svr::parallel_chunks (parallel.cpp:35-63) and float atomics.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "core/allocation.hpp"
#include "core/errors.hpp"
#include "core/grid.hpp"
#include "core/grid_io.hpp"
#include "core/mesh_io.hpp"
#include "core/meshing.hpp"
#include "core/parallel.hpp"
#include "core/scale_field.hpp"

using namespace svr;

namespace {
thread_local std::string g_err;

struct Retained {
    CornerCache cc;
    float s, grad[3], rgb[3];
    double t, delta;
    bool valid;
};
}  // namespace

struct svrr_grid {
    std::unique_ptr<SparseDenseGrid> g;
    // retained forward context for svrr_render_backward
    std::vector<std::vector<Retained>> rays;
    double beta = 0.0;
    // fusion session: 32.32 fixed-point sums [voxel][4 + C] + counts (see svr_oracle.cpp)
    int fuse_flags = -1;
    std::vector<int64_t> fsum;
    std::vector<uint32_t> fcount;
    Mesh mesh;  // last svrr_marching_cubes result
};

typedef struct {
    uint64_t blocks_added, blocks_requested, pixels_used, unallocated;
} svrr_report;
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R[9];
    double t[3];
} svrr_camera;

namespace {
template <typename Fn>
int guarded(Fn&& fn, svrr_report* rep = nullptr) {
    try {
        fn();
        return 0;
    } catch (const CapacityError& e) {
        g_err = e.what();
        if (rep) rep->unallocated = e.unallocated_blocks;
        return 5;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const DataError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

Camera to_camera(const svrr_camera& c) {
    Camera cam;
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.width = c.width;
    cam.height = c.height;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) cam.rotation(i, j) = c.R[3 * i + j];
    cam.translation = Eigen::Vector3d(c.t[0], c.t[1], c.t[2]);
    return cam;
}

inline double density(double s, double beta) {
    const double ib = 1.0 / beta;
    return s > 0.0 ? ib * (0.5 * std::exp(-s / beta)) : ib * (1.0 - 0.5 * std::exp(s / beta));
}
}  // namespace

extern "C" {

const char* svrr_last_error(void) { return g_err.c_str(); }
void svrr_set_threads(int n) { set_worker_count(n); }
int svrr_worker_count(void) { return worker_count(); }

int svrr_grid_create(double h, int B, int C, uint64_t capacity, svrr_grid** out) {
    return guarded([&] {
        auto* w = new svrr_grid();
        w->g = std::make_unique<SparseDenseGrid>(
            h, B, C, capacity ? capacity : SparseDenseGrid::kDefaultCapacity);
        *out = w;
    });
}
void svrr_grid_destroy(svrr_grid* w) { delete w; }
uint64_t svrr_block_count(const svrr_grid* w) { return w->g->block_count(); }
void svrr_coords(const svrr_grid* w, int32_t* out) {
    for (uint32_t i = 0; i < w->g->block_count(); ++i) {
        const BlockCoord& c = w->g->block_coord(i);
        out[3 * i] = c.x, out[3 * i + 1] = c.y, out[3 * i + 2] = c.z;
    }
}
int svrr_bounds(const svrr_grid* w, double* lo3, double* hi3) {
    if (w->g->empty()) return 3;
    const Eigen::AlignedBox3d b = w->g->allocated_bounds();
    for (int a = 0; a < 3; ++a) lo3[a] = b.min()[a], hi3[a] = b.max()[a];
    return 0;
}

int svrr_allocate_blocks(svrr_grid* w, const int32_t* coords, uint64_t n, uint32_t* idx) {
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t v =
                w->g->allocate_block(BlockCoord{coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]});
            if (idx) idx[i] = v;
        }
    });
}

int svrr_allocate_points(svrr_grid* w, const double* xyz, uint64_t n, int dilation,
                         svrr_report* rep) {
    svrr_report r{};
    const int st = guarded(
        [&] {
            std::vector<Eigen::Vector3d> pts(n);
            for (uint64_t i = 0; i < n; ++i)
                pts[i] = Eigen::Vector3d(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
            const AllocationReport a = allocate_for_points(*w->g, pts, dilation);
            r.blocks_added = a.blocks_added;
            r.blocks_requested = a.blocks_requested;
            r.pixels_used = a.pixels_used;
        },
        &r);
    if (rep) *rep = r;
    return st;
}

int svrr_allocate_frames(svrr_grid* w, const float* depth, const svrr_camera* cams,
                         uint32_t n_frames, const double* scales, int rows, int cols,
                         int dilation, svrr_report* rep) {
    svrr_report r{};
    const int st = guarded(
        [&] {
            std::vector<Frame> frames(n_frames);
            std::vector<ScaleField> sfs;
            for (uint32_t f = 0; f < n_frames; ++f) {
                frames[f].id = static_cast<int>(f);
                frames[f].camera = to_camera(cams[f]);
                const int W = cams[f].width, H = cams[f].height;
                frames[f].depth = ImageF32(W, H, 1);
                std::memcpy(frames[f].depth.data.data(), depth + static_cast<size_t>(f) * W * H,
                            static_cast<size_t>(W) * H * 4);
                if (scales) {
                    sfs.emplace_back(rows, cols, W, H);
                    std::memcpy(sfs.back().values().data(),
                                scales + static_cast<size_t>(f) * rows * cols,
                                static_cast<size_t>(rows) * cols * 8);
                }
            }
            const AllocationReport a =
                allocate_for_frames(*w->g, frames, scales ? &sfs : nullptr, dilation);
            r.blocks_added = a.blocks_added;
            r.blocks_requested = a.blocks_requested;
            r.pixels_used = a.pixels_used;
        },
        &r);
    if (rep) *rep = r;
    return st;
}

void svrr_find(const svrr_grid* w, const int32_t* coords, uint64_t n, uint32_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = w->g->find_block(BlockCoord{coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]});
}

int svrr_set_payload(svrr_grid* w, uint32_t first, uint32_t n, const float* sdf,
                     const float* weight, const float* rgb, const float* logits) {
    return guarded([&] {
        if (static_cast<size_t>(first) + n > w->g->block_count())
            throw DataError("payload: block range out of bounds");
        const size_t V = w->g->voxels_per_block(), C = w->g->label_channels();
        for (uint32_t i = 0; i < n; ++i) {
            VoxelBlock& b = w->g->block(first + i);
            if (sdf) std::memcpy(b.sdf.data(), sdf + i * V, V * 4);
            if (weight) std::memcpy(b.weight.data(), weight + i * V, V * 4);
            if (rgb) std::memcpy(b.color.data(), rgb + 3 * i * V, 3 * V * 4);
            if (logits) std::memcpy(b.logits.data(), logits + C * i * V, C * V * 4);
        }
    });
}

void svrr_query(const svrr_grid* w, const double* x, uint64_t n, double* sdf, double* grad,
                double* rgb, uint8_t* valid) {
    parallel_chunks(n, [&](size_t b, size_t e, int) {
        for (size_t i = b; i < e; ++i) {
            const Eigen::Vector3d p(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
            double s = 0.0;
            Eigen::Vector3d gr = Eigen::Vector3d::Zero(), col = Eigen::Vector3d::Zero();
            const bool ok = w->g->query_sdf_with_gradient(p, s, gr);
            if (ok) {
                CornerCacheD cc;
                w->g->gather_corners(p, cc);
                col = w->g->color_at(cc);
            }
            if (sdf) sdf[i] = s;
            for (int a = 0; a < 3; ++a) {
                if (grad) grad[3 * i + a] = gr[a];
                if (rgb) rgb[3 * i + a] = col[a];
            }
            if (valid) valid[i] = ok;
        }
    });
}

void svrr_march(const svrr_grid* w, const double* o, const double* d, uint64_t n, double step,
                uint32_t max_samples, uint32_t* counts, double* t, double* delta) {
    parallel_chunks(n, [&](size_t b, size_t e, int) {
        std::vector<SparseDenseGrid::RaySample> s;
        for (size_t i = b; i < e; ++i) {
            w->g->march_ray(Eigen::Vector3d(o[3 * i], o[3 * i + 1], o[3 * i + 2]),
                            Eigen::Vector3d(d[3 * i], d[3 * i + 1], d[3 * i + 2]), step,
                            max_samples, s);
            counts[i] = static_cast<uint32_t>(s.size());
            for (size_t k = 0; k < s.size(); ++k) {
                if (t) t[i * max_samples + k] = s[k].t;
                if (delta) delta[i * max_samples + k] = s[k].delta;
            }
        }
    });
}

// Forward: per sample gather into a retained float CornerCache (grid.hpp:76-86).
int svrr_render_forward(svrr_grid* w, const double* o, const double* d, uint64_t n, double step,
                        uint32_t max_samples, double beta, float* rgb, float* depth,
                        float* normal, float* wsum, uint32_t* nvalid) {
    return guarded([&] {
        if (!(beta > 0.0)) throw ConfigError("render: beta must be positive");
        w->rays.resize(n);
        w->beta = beta;
        parallel_chunks(n, [&](size_t b, size_t e, int) {
            std::vector<SparseDenseGrid::RaySample> s;
            for (size_t i = b; i < e; ++i) {
                const Eigen::Vector3d ro(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
                const Eigen::Vector3d rd(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
                w->g->march_ray(ro, rd, step, max_samples, s);
                std::vector<Retained>& rec = w->rays[i];
                rec.resize(s.size());
                double T = 1.0, C[3] = {0, 0, 0}, D = 0, N[3] = {0, 0, 0}, W = 0;
                uint32_t nv = 0;
                for (size_t k = 0; k < s.size(); ++k) {
                    Retained& r = rec[k];
                    r.t = s[k].t;
                    r.delta = s[k].delta;
                    r.valid = w->g->gather_corners(ro + s[k].t * rd, r.cc);
                    if (!r.valid) continue;
                    ++nv;
                    r.s = w->g->sdf_at(r.cc);
                    const Eigen::Vector3f gr = w->g->sdf_gradient_at(r.cc);
                    const Eigen::Vector3f col = w->g->color_at(r.cc);
                    for (int a = 0; a < 3; ++a) r.grad[a] = gr[a], r.rgb[a] = col[a];
                    const double tau = density(r.s, beta) * r.delta;
                    const double wk = T * (1.0 - std::exp(-tau));
                    for (int a = 0; a < 3; ++a) C[a] += wk * r.rgb[a], N[a] += wk * r.grad[a];
                    D += wk * r.t;
                    W += wk;
                    T *= std::exp(-tau);
                }
                for (int a = 0; a < 3; ++a) {
                    if (rgb) rgb[3 * i + a] = static_cast<float>(C[a]);
                    if (normal) normal[3 * i + a] = static_cast<float>(N[a]);
                }
                if (depth) depth[i] = static_cast<float>(D);
                if (wsum) wsum[i] = static_cast<float>(W);
                if (nvalid) nvalid[i] = nv;
            }
        });
    });
}

// Backward from the retained caches into VoxelBlock::grad_sdf / grad_color.
int svrr_render_backward(svrr_grid* w, const float* d_rgb, const float* d_depth,
                         const float* d_normal) {
    return guarded([&] {
        const size_t V = w->g->voxels_per_block();
        for (uint32_t i = 0; i < w->g->block_count(); ++i) {
            VoxelBlock& b = w->g->block(i);
            if (b.grad_sdf.size() != V) b.grad_sdf.assign(V, 0.0f);
            if (b.grad_color.size() != 3 * V) b.grad_color.assign(3 * V, 0.0f);
        }
        const double beta = w->beta;
        parallel_chunks(w->rays.size(), [&](size_t b, size_t e, int) {
            std::vector<double> wk, Tn, vk;
            for (size_t i = b; i < e; ++i) {
                const std::vector<Retained>& rec = w->rays[i];
                const float* dC = d_rgb + 3 * i;
                const float* dN = d_normal + 3 * i;
                const double dD = d_depth[i];
                wk.assign(rec.size(), 0.0);
                Tn.assign(rec.size(), 0.0);
                vk.assign(rec.size(), 0.0);
                double T = 1.0;
                for (size_t k = 0; k < rec.size(); ++k) {
                    const Retained& r = rec[k];
                    if (!r.valid) {
                        Tn[k] = T;
                        continue;
                    }
                    const double tau = density(r.s, beta) * r.delta;
                    wk[k] = T * (1.0 - std::exp(-tau));
                    T *= std::exp(-tau);
                    Tn[k] = T;
                    vk[k] = dC[0] * r.rgb[0] + dC[1] * r.rgb[1] + dC[2] * r.rgb[2] + dD * r.t +
                            dN[0] * r.grad[0] + dN[1] * r.grad[1] + dN[2] * r.grad[2];
                }
                double S = 0.0;
                for (size_t k = rec.size(); k-- > 0;) {
                    const Retained& r = rec[k];
                    if (!r.valid) continue;
                    const double sig = density(r.s, beta);
                    const double dsig = r.s > 0.0 ? -sig / beta : -(1.0 / beta - sig) / beta;
                    const double ds = r.delta * dsig * (Tn[k] * vk[k] - S);
                    for (int c = 0; c < 8; ++c) {
                        VoxelBlock& blk = w->g->block(r.cc.block[c]);
                        const uint32_t v = r.cc.voxel[c];
                        const double gs = r.cc.w[c] * ds + wk[k] * (r.cc.dw[c][0] * dN[0] +
                                                                    r.cc.dw[c][1] * dN[1] +
                                                                    r.cc.dw[c][2] * dN[2]);
                        std::atomic_ref<float>(blk.grad_sdf[v]).fetch_add(
                            static_cast<float>(gs), std::memory_order_relaxed);
                        const double wc = r.cc.w[c] * wk[k];
                        for (int a = 0; a < 3; ++a)
                            std::atomic_ref<float>(blk.grad_color[3 * v + a])
                                .fetch_add(static_cast<float>(wc * dC[a]),
                                           std::memory_order_relaxed);
                    }
                    S += wk[k] * vk[k];
                }
            }
        });
    });
}

int svrr_grad_get(const svrr_grid* w, float* g_sdf, float* g_rgb) {
    const size_t V = w->g->voxels_per_block();
    for (uint32_t i = 0; i < w->g->block_count(); ++i) {
        const VoxelBlock& b = w->g->block(i);
        if (b.grad_sdf.size() == V) {
            if (g_sdf) std::memcpy(g_sdf + i * V, b.grad_sdf.data(), V * 4);
            if (g_rgb) std::memcpy(g_rgb + 3 * i * V, b.grad_color.data(), 3 * V * 4);
        } else {
            if (g_sdf) std::memset(g_sdf + i * V, 0, V * 4);
            if (g_rgb) std::memset(g_rgb + 3 * i * V, 0, 3 * V * 4);
        }
    }
    return 0;
}

int svrr_save_sdgv(const svrr_grid* w, const char* path) {
    return guarded([&] { save_grid(*w->g, path); });
}
int svrr_load_sdgv(const char* path, svrr_grid** out) {
    return guarded([&] {
        auto* w = new svrr_grid();
        w->g = std::make_unique<SparseDenseGrid>(load_grid(path));
        *out = w;
    });
}

}  // extern "C"

// Fusion restated ON the reference's own primitives: voxel_to_world
// (grid.hpp:124), Camera::project + pixel_in_frame (camera.cpp:7-18), ScaleField::value
// (scale_field.cpp:56-60).  Same association / fixed-point rules as svr_oracle.cpp, so a
// bit-exact match pins the oracle's projection arithmetic to the reference's.
extern "C" {

int svrr_fuse_begin(svrr_grid* w, int flags) {
    return guarded([&] {
        const size_t V = w->g->voxels_per_block(), nb = w->g->block_count();
        w->fuse_flags = flags;
        w->fsum.assign(nb * V * (4 + w->g->label_channels()), 0);
        w->fcount.assign(nb * V, 0);
    });
}

int svrr_fuse_frames(svrr_grid* w, const float* depth, const float* rgb, const float* sem,
                     const svrr_camera* cams, uint32_t n_frames, const double* scales, int rows,
                     int cols, double mu) {
    return guarded([&] {
        const SparseDenseGrid& g = *w->g;
        const int B = g.block_res(), C = g.label_channels();
        const size_t V = g.voxels_per_block(), K = 4 + C, nb = g.block_count();
        w->fsum.resize(nb * V * K, 0);
        w->fcount.resize(nb * V, 0);
        for (uint32_t f = 0; f < n_frames; ++f) {
            const Camera cam = to_camera(cams[f]);
            const int W = cam.width, H = cam.height;
            std::unique_ptr<ScaleField> sf;
            if (scales) {
                sf = std::make_unique<ScaleField>(rows, cols, W, H);
                std::memcpy(sf->values().data(), scales + static_cast<size_t>(f) * rows * cols,
                            static_cast<size_t>(rows) * cols * 8);
            }
            parallel_chunks(nb, [&](std::size_t b0, std::size_t b1, int) {
                for (std::size_t b = b0; b < b1; ++b) {
                    const BlockCoord bc = g.block_coord(static_cast<uint32_t>(b));
                    for (size_t v = 0; v < V; ++v) {
                        const Eigen::Vector3i vox(bc.x * B + static_cast<int>(v % B),
                                                  bc.y * B + static_cast<int>((v / B) % B),
                                                  bc.z * B + static_cast<int>(v / (B * B)));
                        const Projection pr = cam.project(g.voxel_to_world(vox));
                        if (pr.behind || !pr.in_frame) continue;
                        const int ix = static_cast<int>(std::floor(pr.pixel.x() + 0.5));
                        const int iy = static_cast<int>(std::floor(pr.pixel.y() + 0.5));
                        const size_t pix = (static_cast<size_t>(f) * H + iy) * W + ix;
                        const float D = depth[pix];
                        if (!(D > 0.0f)) continue;
                        const double phi = sf ? sf->value(ix, iy) : 1.0;
                        if (!(phi > 0.0)) continue;
                        const double d = static_cast<double>(D) * phi - pr.depth;
                        if (d < -mu) continue;
                        const size_t i = b * V + v;
                        int64_t* s = &w->fsum[i * K];
                        auto fix = [](double x) {
                            return static_cast<int64_t>(std::nearbyint(x * 4294967296.0));
                        };
                        s[0] += fix(std::min(d, mu));
                        if (rgb)
                            for (int c = 0; c < 3; ++c) s[1 + c] += fix(rgb[3 * pix + c]);
                        if (sem)
                            for (int k = 0; k < C; ++k) s[4 + k] += fix(sem[C * pix + k]);
                        ++w->fcount[i];
                    }
                }
            });
        }
    });
}

int svrr_fuse_finalize(svrr_grid* w) {
    return guarded([&] {
        SparseDenseGrid& g = *w->g;
        const size_t V = g.voxels_per_block(), C = g.label_channels(), K = 4 + C;
        for (uint32_t b = 0; b < g.block_count(); ++b) {
            VoxelBlock& blk = g.block(b);
            for (size_t v = 0; v < V; ++v) {
                const size_t i = b * V + v;
                const uint32_t n = i < w->fcount.size() ? w->fcount[i] : 0;
                blk.weight[v] = static_cast<float>(n);
                if (!n) continue;
                const double dn = n;
                const int64_t* s = &w->fsum[i * K];
                blk.sdf[v] = static_cast<float>(static_cast<double>(s[0]) * 0x1p-32 / dn);
                if (w->fuse_flags & 1)
                    for (int c = 0; c < 3; ++c)
                        blk.color[3 * v + c] = static_cast<float>(static_cast<double>(s[1 + c]) * 0x1p-32 / dn);
                if (w->fuse_flags & 2) {
                    std::vector<double> mm(C);
                    double n2 = 0.0;
                    for (size_t k = 0; k < C; ++k) {
                        mm[k] = static_cast<double>(s[4 + k]) * 0x1p-32 / dn;
                        n2 = n2 + mm[k] * mm[k];
                    }
                    const double nrm = std::sqrt(n2);
                    for (size_t k = 0; k < C; ++k)
                        blk.logits[C * v + k] = nrm > 0.0 ? static_cast<float>(mm[k] / nrm) : 0.0f;
                }
            }
        }
        w->fuse_flags = -1;
    });
}

int svrr_get_payload(const svrr_grid* w, uint32_t first, uint32_t n, float* sdf, float* weight,
                     float* rgb, float* logits) {
    const size_t V = w->g->voxels_per_block(), C = w->g->label_channels();
    for (uint32_t i = 0; i < n; ++i) {
        const VoxelBlock& b = w->g->block(first + i);
        if (sdf) std::memcpy(sdf + i * V, b.sdf.data(), V * 4);
        if (weight) std::memcpy(weight + i * V, b.weight.data(), V * 4);
        if (rgb) std::memcpy(rgb + 3 * i * V, b.color.data(), 3 * V * 4);
        if (logits) std::memcpy(logits + C * i * V, b.logits.data(), C * V * 4);
    }
    return 0;
}

}  // extern "C"

// marching_cubes (meshing.cpp:168-273) and export_ply (mesh_io.cpp:30-68), the reference's
// own code.
extern "C" {

int svrr_marching_cubes(svrr_grid* w, double iso, uint64_t* nv, uint64_t* nt) {
    return guarded([&] {
        w->mesh = marching_cubes(*w->g, iso);
        *nv = w->mesh.vertices.size();
        *nt = w->mesh.triangles.size();
    });
}

int svrr_mesh_get(const svrr_grid* w, double* v, double* n, double* c, int32_t* labels, int32_t* tris) {
    const Mesh& m = w->mesh;
    for (size_t i = 0; i < m.vertices.size(); ++i)
        for (int a = 0; a < 3; ++a) {
            if (v) v[3 * i + a] = m.vertices[i][a];
            if (n) n[3 * i + a] = m.normals[i][a];
            if (c) c[3 * i + a] = m.colors[i][a];
        }
    if (labels)
        for (size_t i = 0; i < m.labels.size(); ++i) labels[i] = m.labels[i];
    if (tris)
        for (size_t i = 0; i < m.triangles.size(); ++i)
            for (int k = 0; k < 3; ++k) tris[3 * i + k] = m.triangles[i][k];
    return 0;
}

int svrr_mesh_export_ply(const svrr_grid* w, const char* path) {
    return guarded([&] { export_ply(w->mesh, path); });
}

double svrr_mesh_area(const svrr_grid* w) { return w->mesh.area(); }

int svrr_mesh_export_obj(const svrr_grid* w, const char* path) {
    return guarded([&] { export_obj(w->mesh, path); });
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// The REFERENCE's synthetic generator (proj/src/core/synthetic.cpp, compiled verbatim; the
// file-writing helpers it calls only from generate_synthetic are stubbed in
// shim/io_stubs.cpp) behind the same C interface as fixtures/libsvr_fixture.so, so the
// --impl reference bench arm builds its inputs with reference code only, and the fixture
// restatement is pinned to it bit for bit (tests/test_synthetic.py).
//
// The recipes around the scene are the harness's: GT depth = the z-depth
// raycast per integer pixel as generate_synthetic renders it (synthetic.cpp:318-340),
// payload = clamp(sdf(v h), -mu, mu) with colour / one-hot logits of the nearest surface's
// class, rays through mt19937_64-drawn pixels with Camera::ray_direction (camera.cpp:27-30).
// ---------------------------------------------------------------------------------------
#include <random>
#include <thread>

#include "core/synthetic.hpp"

namespace {
// Layout mirror of SyntheticScene's private state (synthetic.hpp:61-71), used only to read the
// object list for the nearest-surface class of a payload voxel (the reference exposes sdf()
// but not which surface attains it).  Checked against the real object at construction.
struct SceneMirror {
    struct Object {
        bool is_sphere = true;
        Eigen::Vector3d center{0, 0, 0};
        Eigen::Vector3d half{0.1, 0.1, 0.1};
        int label = 2;
    };
    SceneSpec spec_;
    Eigen::Vector3d room_half_;
    std::vector<Object> objects_;
};
static_assert(sizeof(SceneMirror) == sizeof(SyntheticScene), "SyntheticScene layout changed");

double mirror_box_sdf(const Eigen::Vector3d& p, const Eigen::Vector3d& half) {  // synthetic.cpp:33-38
    const Eigen::Vector3d q = p.cwiseAbs() - half;
    const Eigen::Vector3d outside = q.cwiseMax(0.0);
    const double inside = std::min(q.maxCoeff(), 0.0);
    return outside.norm() + inside;
}

template <typename F>
void for_range(uint64_t n, int threads, F&& fn) {
    int w = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    w = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(w), std::max<uint64_t>(n, 1)));
    if (w <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    const uint64_t chunk = (n + w - 1) / w;
    std::vector<std::thread> pool;
    for (int i = 0; i < w; ++i) {
        const uint64_t b = i * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}
}  // namespace

typedef struct {
    double room_w, room_d, room_h;
    int32_t n_objects, n_frames, width, height;
    double fov_deg;
    int32_t label_channels;
    double texture_amplitude, texture_frequency;
    uint64_t seed;
} svrr_scene_spec;

struct svrr_scene {
    std::unique_ptr<SyntheticScene> s;
    const SceneMirror* m = nullptr;
    // class of the surface nearest to x: walls / floor from the room box, else the nearest object
    int label(const Eigen::Vector3d& x) const {
        const Eigen::Vector3d dw = m->room_half_ - x.cwiseAbs();
        int axis = 0;
        for (int a = 1; a < 3; ++a)
            if (dw[a] < dw[axis]) axis = a;
        double best = dw[axis];
        int lab = (axis == 2 && x.z() < 0.0) ? 1 : 0;
        for (const auto& o : m->objects_) {
            const double od = o.is_sphere ? (x - o.center).norm() - o.half.x() : mirror_box_sdf(x - o.center, o.half);
            if (od < best) {
                best = od;
                lab = o.label;
            }
        }
        return lab;
    }
};

namespace {
svrr_camera from_camera(const Camera& c) {
    svrr_camera o{};
    o.fx = c.fx, o.fy = c.fy, o.cx = c.cx, o.cy = c.cy;
    o.width = c.width, o.height = c.height;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.R[3 * i + j] = c.rotation(i, j);
    for (int i = 0; i < 3; ++i) o.t[i] = c.translation[i];
    return o;
}
}  // namespace

extern "C" {

int svrr_scene_create(const svrr_scene_spec* in, svrr_scene** out) {
    return guarded([&] {
        SceneSpec sp;  // synthetic.hpp:13-30 (the fields the fixture sets; the rest default)
        sp.room_w = in->room_w, sp.room_d = in->room_d, sp.room_h = in->room_h;
        sp.n_objects = in->n_objects, sp.n_frames = in->n_frames;
        sp.width = in->width, sp.height = in->height, sp.fov_deg = in->fov_deg;
        sp.label_channels = in->label_channels;
        sp.texture_amplitude = in->texture_amplitude, sp.texture_frequency = in->texture_frequency;
        sp.seed = in->seed;
        auto w = std::make_unique<svrr_scene>();
        w->s = std::make_unique<SyntheticScene>(sp);
        w->m = reinterpret_cast<const SceneMirror*>(w->s.get());
        // the mirror must reproduce the reference's own sdf (synthetic.cpp:71-80)
        std::mt19937_64 rng(12345);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (int i = 0; i < 64; ++i) {
            const Eigen::Vector3d x(u(rng) * sp.room_w / 2, u(rng) * sp.room_d / 2, u(rng) * sp.room_h / 2);
            double d = (w->m->room_half_ - x.cwiseAbs()).minCoeff();
            for (const auto& o : w->m->objects_)
                d = std::min(d, o.is_sphere ? (x - o.center).norm() - o.half.x() : mirror_box_sdf(x - o.center, o.half));
            if (d != w->s->sdf(x)) throw DataError("scene mirror disagrees with SyntheticScene::sdf");
        }
        *out = w.release();
    });
}

void svrr_scene_destroy(svrr_scene* s) { delete s; }

int svrr_scene_camera(const svrr_scene* s, int32_t frame, svrr_camera* out) {
    return guarded([&] { *out = from_camera(s->s->camera_for_frame(frame)); });
}

// depth / rgb / semantic / camera-frame normal per integer pixel, as generate_synthetic
// renders its frames (synthetic.cpp:318-340); any output may be NULL
int svrr_scene_frames(const svrr_scene* s, const svrr_camera* cams, uint32_t n, float* depth, float* rgb,
                      float* sem, int32_t C, float* normal, int32_t threads) {
    if (!n) return 0;
    std::atomic<bool> escaped{false};
    const int W = cams[0].width, H = cams[0].height;
    std::vector<Camera> cs(n);
    for (uint32_t f = 0; f < n; ++f) cs[f] = to_camera(cams[f]);
    for_range(static_cast<uint64_t>(n) * H, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t r = b; r < e; ++r) {
            const uint32_t f = static_cast<uint32_t>(r / H);
            const int y = static_cast<int>(r % H);
            for (int x = 0; x < W; ++x) {
                SyntheticScene::Hit hit;
                if (!s->s->raycast(cs[f], x, y, hit)) {
                    escaped = true;
                    continue;
                }
                const uint64_t px = r * W + x;
                if (depth) depth[px] = static_cast<float>(hit.depth);
                if (normal) {
                    const Eigen::Vector3d n_cam = cs[f].rotation.transpose() * hit.normal;
                    for (int c = 0; c < 3; ++c) normal[3 * px + c] = static_cast<float>(n_cam[c]);
                }
                if (sem)
                    for (int k = 0; k < C; ++k) sem[C * px + k] = k == hit.label ? 1.0f : 0.0f;
                if (rgb) {
                    const Eigen::Vector3d c = s->s->color(hit.point, hit.label);
                    for (int k = 0; k < 3; ++k) rgb[3 * px + k] = static_cast<float>(c[k]);
                }
            }
        }
    });
    if (escaped) {
        g_err = "synthetic: ray escaped the room";
        return 3;
    }
    return 0;
}

int svrr_scene_sdf(const svrr_scene* s, const double* x, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = s->s->sdf(Eigen::Vector3d(x[3 * i], x[3 * i + 1], x[3 * i + 2]));
    return 0;
}

int svrr_scene_fill_payload(const svrr_scene* s, double h, int32_t B, int32_t C, double trunc,
                            const int32_t* coords, uint64_t nblocks, float* sdf, float* weight, float* rgb,
                            float* logits, int32_t threads) {
    const uint64_t V = static_cast<uint64_t>(B) * B * B;
    for_range(nblocks, threads, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
            for (uint64_t v = 0; v < V; ++v) {
                const int lx = static_cast<int>(v % B), ly = static_cast<int>((v / B) % B),
                          lz = static_cast<int>(v / (B * B));
                // voxel_to_world (grid.hpp:124-126)
                const Eigen::Vector3d x = Eigen::Vector3i(coords[3 * i] * B + lx, coords[3 * i + 1] * B + ly,
                                                          coords[3 * i + 2] * B + lz)
                                              .cast<double>() *
                                          h;
                const uint64_t o = i * V + v;
                if (sdf) sdf[o] = static_cast<float>(std::clamp(s->s->sdf(x), -trunc, trunc));
                if (weight) weight[o] = 1.0f;
                if (rgb || logits) {
                    const int lab = s->label(x);
                    if (rgb) {
                        const Eigen::Vector3d c = s->s->color(x, lab);
                        for (int k = 0; k < 3; ++k) rgb[3 * o + k] = static_cast<float>(c[k]);
                    }
                    if (logits)
                        for (int k = 0; k < C; ++k) logits[C * o + k] = k == lab ? 1.0f : 0.0f;
                }
            }
    });
    return 0;
}

int svrr_scene_rays(const svrr_scene* s, uint32_t n_poses, uint32_t rays_per_pose, uint64_t seed, double* o,
                    double* d) {
    const SceneSpec& sp = s->s->spec();
    std::mt19937_64 rng(seed);
    const uint64_t npix = static_cast<uint64_t>(sp.width) * sp.height;
    std::uniform_int_distribution<uint64_t> pick(0, npix - 1);
    uint64_t i = 0;
    for (uint32_t p = 0; p < n_poses; ++p) {
        const Camera cam = s->s->camera_for_frame(static_cast<int>(p));
        for (uint32_t r = 0; r < rays_per_pose; ++r, ++i) {
            const uint64_t px = pick(rng);
            const Eigen::Vector3d dir = cam.ray_direction(
                Eigen::Vector2d(static_cast<double>(px % sp.width), static_cast<double>(px / sp.width)));
            for (int a = 0; a < 3; ++a) o[3 * i + a] = cam.translation[a], d[3 * i + a] = dir[a];
        }
    }
    return 0;
}

int svrr_scene_image_rays(const svrr_scene* s, int32_t frame, double* o, double* d) {
    const SceneSpec& sp = s->s->spec();
    const Camera cam = s->s->camera_for_frame(frame);
    uint64_t i = 0;
    for (int y = 0; y < sp.height; ++y)
        for (int x = 0; x < sp.width; ++x, ++i) {
            const Eigen::Vector3d dir = cam.ray_direction(Eigen::Vector2d(x, y));
            for (int a = 0; a < 3; ++a) o[3 * i + a] = cam.translation[a], d[3 * i + a] = dir[a];
        }
    return 0;
}

int svrr_uniform_floats(uint64_t n, uint64_t seed, float lo, float hi, float* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> u(lo, hi);
    for (uint64_t i = 0; i < n; ++i) out[i] = u(rng);
    return 0;
}

}  // extern "C"
