// TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the sparse-dense SDF rendering
// path.  See svr_oracle.h for the contract.  Every function cites the reference
// file:line it restates (paths relative to /root/reference/).  Nothing here is on the
// product path: paper_2305_13220_b200 never links or loads this library.
#include "svr_oracle.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

thread_local std::string g_err;
int g_threads = 1;

struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
constexpr int kConfig = 2, kData = 3, kCapacity = 5;

// ---------------------------------------------------------------------------
// Block coordinates and the hash map (proj/src/core/grid.hpp:11-55,
// proj/src/core/grid.cpp:11-67).
// ---------------------------------------------------------------------------
struct BlockCoord {
    int32_t x = 0, y = 0, z = 0;
    bool operator==(const BlockCoord& o) const { return x == o.x && y == o.y && z == o.z; }
};

// grid.hpp:16-26
uint64_t hash_block_coord(const BlockCoord& c) {
    uint64_t h = static_cast<uint32_t>(c.x) * 0x9E3779B185EBCA87ull;
    h ^= static_cast<uint32_t>(c.y) * 0xC2B2AE3D27D4EB4Full;
    h += static_cast<uint32_t>(c.z) * 0x165667B19E3779F9ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    return h;
}

// grid.cpp:14-24: the slot-array size table.
constexpr size_t kPrimes[] = {97,       193,      389,      769,       1543,      3079,
                              6151,     12289,    24593,    49157,     98317,     196613,
                              393241,   786433,   1572869,  3145739,   6291469,   12582917,
                              25165843, 50331653, 100663319, 201326611};

size_t next_prime_size(size_t at_least) {
    for (size_t p : kPrimes)
        if (p >= at_least) return p;
    return kPrimes[std::size(kPrimes) - 1];
}

constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // grid.hpp:33

// Exact-key open addressing, linear probing over a prime-sized array, grows at
// load > 0.75 (grid.cpp:28-67).
class BlockMap {
public:
    BlockMap() : slots_(kPrimes[0]) {}
    uint32_t find(const BlockCoord& k) const {  // grid.cpp:30-38
        size_t i = hash_block_coord(k) % slots_.size();
        for (;;) {
            const Slot& s = slots_[i];
            if (s.value == kInvalid) return kInvalid;
            if (s.key == k) return s.value;
            if (++i == slots_.size()) i = 0;
        }
    }
    uint32_t insert(const BlockCoord& k, uint32_t v) {  // grid.cpp:40-54
        if ((count_ + 1) * 4 > slots_.size() * 3) grow();
        size_t i = hash_block_coord(k) % slots_.size();
        for (;;) {
            Slot& s = slots_[i];
            if (s.value == kInvalid) {
                s.key = k;
                s.value = v;
                ++count_;
                return v;
            }
            if (s.key == k) return s.value;
            if (++i == slots_.size()) i = 0;
        }
    }

private:
    struct Slot {
        BlockCoord key;
        uint32_t value = kInvalid;
    };
    void grow() {  // grid.cpp:56-67
        std::vector<Slot> old;
        old.swap(slots_);
        slots_.assign(next_prime_size(old.size() * 2), Slot{});
        for (const Slot& s : old) {
            if (s.value == kInvalid) continue;
            size_t i = hash_block_coord(s.key) % slots_.size();
            while (slots_[i].value != kInvalid)
                if (++i == slots_.size()) i = 0;
            slots_[i] = s;
        }
    }
    std::vector<Slot> slots_;
    size_t count_ = 0;
};

// floor_div (grid.hpp:207-210)
int32_t floor_div(int32_t a, int32_t b) {
    int32_t q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// Packed 64-bit key, 21 bits/axis biased by 2^20.  Defines the deterministic
// allocation order this build uses in place of libstdc++ unordered_set iteration
// order (allocation.cpp:31).
constexpr int32_t kCoordLim = 1 << 20;
bool packable(const BlockCoord& c) {
    return c.x >= -kCoordLim && c.x < kCoordLim && c.y >= -kCoordLim && c.y < kCoordLim &&
           c.z >= -kCoordLim && c.z < kCoordLim;
}
uint64_t pack_key(const BlockCoord& c) {
    return (static_cast<uint64_t>(c.z + kCoordLim) << 42) |
           (static_cast<uint64_t>(c.y + kCoordLim) << 21) |
           static_cast<uint64_t>(c.x + kCoordLim);
}
BlockCoord unpack_key(uint64_t k) {
    const uint64_t m = (1ull << 21) - 1;
    return BlockCoord{static_cast<int32_t>(k & m) - kCoordLim,
                      static_cast<int32_t>((k >> 21) & m) - kCoordLim,
                      static_cast<int32_t>((k >> 42) & m) - kCoordLim};
}

struct KeyHash {
    size_t operator()(uint64_t k) const { return static_cast<size_t>(k * 0x9E3779B97F4A7C15ull); }
};

}  // namespace

// ---------------------------------------------------------------------------
// The grid (grid.hpp:100-223).  Payload kept as flat arrays in the reference's
// per-block layout (sdf[V], weight[V], color[3V] interleaved, logits[CV]
// interleaved; grid.hpp:62-66, grid.cpp:69-75).
// ---------------------------------------------------------------------------
struct svro_grid {
    double h;
    int B;
    int C;
    size_t capacity;
    int V;  // B^3
    BlockMap map;
    std::vector<BlockCoord> coords;
    std::vector<float> sdf, weight, rgb, logits;
    // fusion session: fixed-point running sums + counts, see svro_fuse_begin
    int fuse_flags = -1;           // -1 = no session open
    std::vector<int64_t> fsum;     // [voxel][4 + C]: sdf, r, g, b, logits
    std::vector<uint32_t> fcount;  // [voxel]
    // last marching_cubes result (svro_mesh_get)
    std::vector<double> mv, mn, mc;  // vertices / normals / colors, 3 per vertex
    std::vector<int32_t> ml, mt;     // labels, triangles (3 per)
    BlockCoord lo{0, 0, 0}, hi{0, 0, 0};

    double L() const { return h * B; }  // grid.hpp:112

    // grid.hpp:132-135
    BlockCoord block_of_voxel(int vx, int vy, int vz) const {
        return BlockCoord{floor_div(vx, B), floor_div(vy, B), floor_div(vz, B)};
    }
    // grid.hpp:136-141: floor(x / L), a true division (not x * (1/L)).
    BlockCoord block_of_point(const double* x) const {
        const double Lx = L();
        return BlockCoord{static_cast<int32_t>(std::floor(x[0] / Lx)),
                          static_cast<int32_t>(std::floor(x[1] / Lx)),
                          static_cast<int32_t>(std::floor(x[2] / Lx))};
    }
    // grid.hpp:142-147
    uint32_t local_index(int vx, int vy, int vz, const BlockCoord& b) const {
        const int lx = vx - b.x * B, ly = vy - b.y * B, lz = vz - b.z * B;
        return static_cast<uint32_t>(lx + B * (ly + B * lz));
    }

    // grid.cpp:88-108 (allocate_block), payload zero-init grid.cpp:69-75.
    uint32_t allocate_block(const BlockCoord& c) {
        const uint32_t existing = map.find(c);
        if (existing != kInvalid) return existing;
        if (coords.size() >= capacity) throw Status(kCapacity, "grid: block capacity exceeded");
        if (!packable(c)) throw Status(kConfig, "grid: block coordinate outside +-2^20");
        const uint32_t idx = static_cast<uint32_t>(coords.size());
        map.insert(c, idx);
        coords.push_back(c);
        sdf.resize(sdf.size() + V, 0.0f);
        weight.resize(weight.size() + V, 0.0f);
        rgb.resize(rgb.size() + 3 * V, 0.0f);
        logits.resize(logits.size() + static_cast<size_t>(C) * V, 0.0f);
        if (coords.size() == 1) {
            lo = hi = c;
        } else {
            lo.x = std::min(lo.x, c.x);
            lo.y = std::min(lo.y, c.y);
            lo.z = std::min(lo.z, c.z);
            hi.x = std::max(hi.x, c.x);
            hi.y = std::max(hi.y, c.y);
            hi.z = std::max(hi.z, c.z);
        }
        return idx;
    }
};

namespace {

// CornerCacheD (grid.hpp:90-96)
struct Corners {
    uint32_t block[8];
    uint32_t voxel[8];
    double w[8];
    double dw[8][3];
};

// gather_impl (grid.cpp:112-155): g = x * (1/h) (multiply by the reciprocal),
// base = floor(g), corner c takes bit a of c on axis a, re-find only when the
// corner's block differs from the previous corner's, any missing block or
// weight <= 0 invalidates the query.
bool gather(const svro_grid& g, const double* x, Corners& cc) {
    const double inv_h = 1.0 / g.h;
    double fx[3];
    int base[3];
    for (int a = 0; a < 3; ++a) {
        const double gg = x[a] * inv_h;
        const double fl = std::floor(gg);
        base[a] = static_cast<int>(fl);
        fx[a] = gg - fl;
    }
    const double w0[3] = {1.0 - fx[0], 1.0 - fx[1], 1.0 - fx[2]};
    BlockCoord last{std::numeric_limits<int32_t>::min(), 0, 0};
    uint32_t last_idx = kInvalid;
    for (int c = 0; c < 8; ++c) {
        const int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
        const int vx = base[0] + bx, vy = base[1] + by, vz = base[2] + bz;
        const BlockCoord bc = g.block_of_voxel(vx, vy, vz);
        if (!(bc == last)) {
            last = bc;
            last_idx = g.map.find(bc);
        }
        if (last_idx == kInvalid) return false;
        const uint32_t vox = g.local_index(vx, vy, vz, bc);
        if (!(g.weight[static_cast<size_t>(last_idx) * g.V + vox] > 0.0f)) return false;
        cc.block[c] = last_idx;
        cc.voxel[c] = vox;
        const double wx = bx ? fx[0] : w0[0];
        const double wy = by ? fx[1] : w0[1];
        const double wz = bz ? fx[2] : w0[2];
        cc.w[c] = wx * wy * wz;
        cc.dw[c][0] = (bx ? 1.0 : -1.0) * inv_h * wy * wz;
        cc.dw[c][1] = (by ? 1.0 : -1.0) * inv_h * wx * wz;
        cc.dw[c][2] = (bz ? 1.0 : -1.0) * inv_h * wx * wy;
    }
    return true;
}

// sdf_impl / sdf_gradient_impl / color_impl (grid.cpp:157-188), double accumulation.
struct Interp {
    double s, grad[3], rgb[3];
};
void interpolate(const svro_grid& g, const Corners& cc, Interp& o) {
    o.s = 0.0;
    o.grad[0] = o.grad[1] = o.grad[2] = 0.0;
    o.rgb[0] = o.rgb[1] = o.rgb[2] = 0.0;
    for (int i = 0; i < 8; ++i) {
        const size_t v = static_cast<size_t>(cc.block[i]) * g.V + cc.voxel[i];
        o.s += cc.w[i] * g.sdf[v];
    }
    for (int i = 0; i < 8; ++i) {
        const double s = g.sdf[static_cast<size_t>(cc.block[i]) * g.V + cc.voxel[i]];
        o.grad[0] += cc.dw[i][0] * s;
        o.grad[1] += cc.dw[i][1] * s;
        o.grad[2] += cc.dw[i][2] * s;
    }
    for (int i = 0; i < 8; ++i) {
        const float* col = &g.rgb[3 * (static_cast<size_t>(cc.block[i]) * g.V + cc.voxel[i])];
        const double w = cc.w[i];
        o.rgb[0] += w * col[0];
        o.rgb[1] += w * col[1];
        o.rgb[2] += w * col[2];
    }
}

struct Sample {
    double t, delta;
};

// march_intervals + march_ray (grid.cpp:263-353), fused: samples are emitted per
// allocated block while the DDA walks, with the same cursor rule (phase kept across
// contiguous blocks, reset to t0 + step/2 after a gap, cursor += step by repeated
// addition) and stopping once max_samples are produced.  Emitting while
// cursor < t_exit(block) is identical to the reference's two-pass form because
// t_exit is non-decreasing along the walk and the merged interval's end equals the
// t_exit of its last block (grid.cpp:316-335).
void march_ray(const svro_grid& g, const double* o, const double* d, double step,
               size_t max_samples, std::vector<Sample>& out) {
    out.clear();
    if (g.coords.empty() || max_samples == 0) return;
    const double L = g.L();
    const double box_lo[3] = {g.lo.x * L, g.lo.y * L, g.lo.z * L};
    const double box_hi[3] = {(g.hi.x + 1) * L, (g.hi.y + 1) * L, (g.hi.z + 1) * L};
    double t0 = 0.0, t1 = std::numeric_limits<double>::max();
    for (int a = 0; a < 3; ++a) {  // grid.cpp:270-285
        if (d[a] == 0.0) {
            if (o[a] < box_lo[a] || o[a] >= box_hi[a]) return;
            continue;
        }
        const double ta = (box_lo[a] - o[a]) / d[a];
        const double tb = (box_hi[a] - o[a]) / d[a];
        t0 = std::max(t0, std::min(ta, tb));
        t1 = std::min(t1, std::max(ta, tb));
    }
    if (!(t0 < t1)) return;
    const double t_eps = 1e-12 * std::max(1.0, std::abs(t0));  // grid.cpp:289-296
    const double ts = t0 + t_eps;
    int32_t b[3];
    const int32_t lo[3] = {g.lo.x, g.lo.y, g.lo.z};
    const int32_t hi[3] = {g.hi.x, g.hi.y, g.hi.z};
    for (int a = 0; a < 3; ++a) {
        const double start = o[a] + ts * d[a];
        b[a] = static_cast<int32_t>(std::floor(start / L));
        b[a] = std::clamp(b[a], lo[a], hi[a]);
    }
    auto crossing = [&](int a) {  // grid.cpp:298-302
        if (d[a] == 0.0) return std::numeric_limits<double>::infinity();
        const double plane = (b[a] + (d[a] > 0.0 ? 1 : 0)) * L;
        return (plane - o[a]) / d[a];
    };
    double t = t0;
    bool open = false;
    double cursor = -std::numeric_limits<double>::infinity();
    while (t < t1) {  // grid.cpp:306-333
        double t_exit = t1;
        int axis = -1;
        for (int a = 0; a < 3; ++a) {
            const double c = crossing(a);
            if (c < t_exit) {
                t_exit = c;
                axis = a;
            }
        }
        const bool allocated = g.map.find(BlockCoord{b[0], b[1], b[2]}) != kInvalid;
        if (allocated && !open) {
            open = true;
            if (cursor < t) cursor = t + 0.5 * step;  // grid.cpp:345 with iv.t0 = t
        } else if (!allocated && open) {
            open = false;
        }
        if (allocated) {
            while (cursor < t_exit && out.size() < max_samples) {  // grid.cpp:346-349
                out.push_back({cursor, step});
                cursor += step;
            }
            if (out.size() >= max_samples) break;
        }
        if (axis < 0) {
            t = t1;
            break;
        }
        b[axis] += d[axis] > 0.0 ? 1 : -1;
        t = t_exit;
        if (b[axis] < lo[axis] || b[axis] > hi[axis]) break;
    }
    for (size_t k = 0; k + 1 < out.size(); ++k) out[k].delta = out[k + 1].t - out[k].t;  // :352
}

// Camera::unproject (camera.cpp:20-25) with R x evaluated row-wise left to right.
void unproject(const svro_camera& cam, double px, double py, double depth, double* out) {
    const double xc[3] = {(px - cam.cx) / cam.fx * depth, (py - cam.cy) / cam.fy * depth, depth};
    for (int i = 0; i < 3; ++i) {
        double acc = cam.R[3 * i + 0] * xc[0];
        acc = acc + cam.R[3 * i + 1] * xc[1];
        acc = acc + cam.R[3 * i + 2] * xc[2];
        out[i] = acc + cam.t[i];
    }
}

// ScaleField::lookup + value (scale_field.cpp:15-60).
double scale_value(const double* grid, int rows, int cols, int iw, int ih, double px, double py) {
    const double sx = static_cast<double>(cols - 1) / (iw - 1);
    const double sy = static_cast<double>(rows - 1) / (ih - 1);
    const double gx = std::clamp(px * sx, 0.0, static_cast<double>(cols - 1));
    const double gy = std::clamp(py * sy, 0.0, static_cast<double>(rows - 1));
    const int c0 = std::min(static_cast<int>(gx), cols - 2);
    const int r0 = std::min(static_cast<int>(gy), rows - 2);
    const double fx = gx - c0, fy = gy - r0;
    const int base = r0 * cols + c0;
    const int idx[4] = {base, base + 1, base + cols, base + cols + 1};
    const double w[4] = {(1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy};
    double v = 0.0;
    for (int i = 0; i < 4; ++i) v += w[i] * grid[idx[i]];
    return v;
}

// commit (allocation.cpp:19-43) with new blocks allocated in ascending packed-key
// order (deterministic; the reference's unordered_set order is a libstdc++ artefact).
void commit(svro_grid& g, const std::unordered_set<uint64_t, KeyHash>& base, int dilation,
            svro_report& rep) {
    std::unordered_set<uint64_t, KeyHash> wanted;
    wanted.reserve(base.size() * (dilation > 0 ? 8 : 1));
    for (uint64_t k : base) {
        const BlockCoord c = unpack_key(k);
        for (int dz = -dilation; dz <= dilation; ++dz)
            for (int dy = -dilation; dy <= dilation; ++dy)
                for (int dx = -dilation; dx <= dilation; ++dx) {
                    const BlockCoord n{c.x + dx, c.y + dy, c.z + dz};
                    if (!packable(n)) throw Status(kConfig, "allocate: block outside +-2^20");
                    wanted.insert(pack_key(n));
                }
    }
    rep.blocks_requested = wanted.size();
    std::vector<uint64_t> fresh;
    for (uint64_t k : wanted)
        if (g.map.find(unpack_key(k)) == kInvalid) fresh.push_back(k);
    std::sort(fresh.begin(), fresh.end());
    uint64_t unallocated = 0;
    for (uint64_t k : fresh) {
        if (g.coords.size() >= g.capacity) {
            ++unallocated;
            continue;
        }
        g.allocate_block(unpack_key(k));
        ++rep.blocks_added;
    }
    rep.unallocated = unallocated;
    if (unallocated > 0) throw Status(kCapacity, "allocate: grid capacity exceeded");
}

// Laplace density.
inline double density(double s, double beta) {
    const double ib = 1.0 / beta;
    return s > 0.0 ? ib * (0.5 * std::exp(-s / beta)) : ib * (1.0 - 0.5 * std::exp(s / beta));
}
inline double density_ds(double s, double sigma, double beta) {
    return s > 0.0 ? -sigma / beta : -(1.0 / beta - sigma) / beta;
}

template <typename F>
void parallel_chunks(size_t n, F&& fn) {  // proj/src/core/parallel.cpp:35-63
    const int workers = static_cast<int>(std::min<size_t>(std::max(1, g_threads), n));
    if (workers <= 1) {
        if (n) fn(size_t(0), n);
        return;
    }
    const size_t chunk = (n + workers - 1) / workers;
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w) {
        const size_t b = static_cast<size_t>(w) * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Status& s) {
        g_err = s.what();
        return s.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kData;
    }
}

}  // namespace

extern "C" {

const char* svro_last_error(void) { return g_err.c_str(); }
void svro_set_threads(int n) { g_threads = n > 0 ? n : 1; }

int svro_grid_create(double voxel_size, int block_res, int label_channels, uint64_t capacity,
                     svro_grid** out) {
    return guarded([&] {
        // grid.cpp:83-85
        if (!(voxel_size > 0.0)) throw Status(kConfig, "grid: voxel_size must be positive");
        if (block_res < 2) throw Status(kConfig, "grid: block_res must be >= 2");
        if (label_channels < 1) throw Status(kConfig, "grid: label_channels must be >= 1");
        auto* g = new svro_grid();
        g->h = voxel_size;
        g->B = block_res;
        g->C = label_channels;
        g->capacity = capacity ? capacity : (1u << 21);  // grid.hpp:107
        g->V = block_res * block_res * block_res;
        *out = g;
    });
}
void svro_grid_destroy(svro_grid* g) { delete g; }
uint64_t svro_block_count(const svro_grid* g) { return g->coords.size(); }
uint64_t svro_capacity(const svro_grid* g) { return g->capacity; }
void svro_coords(const svro_grid* g, int32_t* out) {
    for (size_t i = 0; i < g->coords.size(); ++i) {
        out[3 * i] = g->coords[i].x;
        out[3 * i + 1] = g->coords[i].y;
        out[3 * i + 2] = g->coords[i].z;
    }
}
int svro_bounds(const svro_grid* g, int32_t* lo3, int32_t* hi3) {
    lo3[0] = g->lo.x, lo3[1] = g->lo.y, lo3[2] = g->lo.z;
    hi3[0] = g->hi.x, hi3[1] = g->hi.y, hi3[2] = g->hi.z;
    return g->coords.empty() ? kData : 0;
}

int svro_allocate_blocks(svro_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out) {
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t idx =
                g->allocate_block(BlockCoord{coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]});
            if (idx_out) idx_out[i] = idx;
        }
    });
}

// allocate_for_points (allocation.cpp:45-54)
int svro_allocate_points(svro_grid* g, const double* xyz, uint64_t n, int dilation,
                         svro_report* rep) {
    svro_report r{};
    const int st = guarded([&] {
        if (dilation < 0) throw Status(kConfig, "allocate: dilation must be >= 0");
        std::unordered_set<uint64_t, KeyHash> base;
        base.reserve(n);
        for (uint64_t i = 0; i < n; ++i) {
            const BlockCoord c = g->block_of_point(xyz + 3 * i);
            if (!packable(c)) throw Status(kConfig, "allocate: block outside +-2^20");
            base.insert(pack_key(c));
        }
        r.pixels_used = n;
        commit(*g, base, dilation, r);
    });
    if (rep) *rep = r;
    return st;
}

// allocate_for_frames (allocation.cpp:56-83)
int svro_allocate_frames(svro_grid* g, const float* depth, const svro_camera* cams,
                         uint32_t n_frames, const double* scales, int sf_rows, int sf_cols,
                         int dilation, svro_report* rep) {
    svro_report r{};
    const int st = guarded([&] {
        if (dilation < 0) throw Status(kConfig, "allocate: dilation must be >= 0");
        if (n_frames == 0) {
            std::unordered_set<uint64_t, KeyHash> none;
            commit(*g, none, dilation, r);
            return;
        }
        const int W = cams[0].width, H = cams[0].height;
        for (uint32_t f = 0; f < n_frames; ++f)
            if (cams[f].width != W || cams[f].height != H)
                throw Status(kConfig, "allocate: all frames must share one size");
        if (scales && (sf_rows < 2 || sf_cols < 2))
            throw Status(kConfig, "scale field needs at least a 2x2 grid");
        std::unordered_set<uint64_t, KeyHash> base;
        uint64_t pixels = 0;
        for (uint32_t f = 0; f < n_frames; ++f) {
            const float* dm = depth + static_cast<size_t>(f) * W * H;
            const double* sf = scales ? scales + static_cast<size_t>(f) * sf_rows * sf_cols : nullptr;
            for (int y = 0; y < H; ++y)
                for (int x = 0; x < W; ++x) {
                    const float d = dm[static_cast<size_t>(y) * W + x];
                    if (!(d > 0.0f)) continue;
                    const double scale =
                        sf ? scale_value(sf, sf_rows, sf_cols, W, H, x, y) : 1.0;
                    if (!(scale > 0.0)) continue;
                    double p[3];
                    unproject(cams[f], static_cast<double>(x), static_cast<double>(y), d * scale, p);
                    const BlockCoord c = g->block_of_point(p);
                    if (!packable(c)) throw Status(kConfig, "allocate: block outside +-2^20");
                    base.insert(pack_key(c));
                    ++pixels;
                }
        }
        r.pixels_used = pixels;
        commit(*g, base, dilation, r);
    });
    if (rep) *rep = r;
    return st;
}

void svro_find(const svro_grid* g, const int32_t* coords, uint64_t n, uint32_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = g->map.find(BlockCoord{coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]});
}

int svro_set_payload(svro_grid* g, uint32_t first, uint32_t n, const float* sdf,
                     const float* weight, const float* rgb, const float* logits) {
    return guarded([&] {
        if (static_cast<size_t>(first) + n > g->coords.size())
            throw Status(kData, "payload: block range out of bounds");
        const size_t V = g->V, o = static_cast<size_t>(first) * V, m = static_cast<size_t>(n) * V;
        if (sdf) std::memcpy(&g->sdf[o], sdf, m * 4);
        if (weight) std::memcpy(&g->weight[o], weight, m * 4);
        if (rgb) std::memcpy(&g->rgb[3 * o], rgb, 3 * m * 4);
        if (logits) std::memcpy(&g->logits[g->C * o], logits, g->C * m * 4);
    });
}
int svro_get_payload(const svro_grid* g, uint32_t first, uint32_t n, float* sdf, float* weight,
                     float* rgb, float* logits) {
    return guarded([&] {
        if (static_cast<size_t>(first) + n > g->coords.size())
            throw Status(kData, "payload: block range out of bounds");
        const size_t V = g->V, o = static_cast<size_t>(first) * V, m = static_cast<size_t>(n) * V;
        if (sdf) std::memcpy(sdf, &g->sdf[o], m * 4);
        if (weight) std::memcpy(weight, &g->weight[o], m * 4);
        if (rgb) std::memcpy(rgb, &g->rgb[3 * o], 3 * m * 4);
        if (logits) std::memcpy(logits, &g->logits[g->C * o], g->C * m * 4);
    });
}

// query_sdf_with_gradient + color_at + logits_at over CornerCacheD
// (grid.cpp:157-261): invalid -> zeros and valid = 0.
void svro_query(const svro_grid* g, const double* x, uint64_t n, double* sdf, double* grad,
                double* rgb, double* logits, uint8_t* valid) {
    parallel_chunks(n, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            Corners cc;
            const bool ok = !g->coords.empty() && gather(*g, x + 3 * i, cc);
            Interp it{};
            if (ok) interpolate(*g, cc, it);
            if (sdf) sdf[i] = ok ? it.s : 0.0;
            for (int a = 0; a < 3; ++a) {
                if (grad) grad[3 * i + a] = ok ? it.grad[a] : 0.0;
                if (rgb) rgb[3 * i + a] = ok ? it.rgb[a] : 0.0;
            }
            if (logits) {  // logits_at(CornerCacheD) grid.cpp:230-238
                double* out = logits + static_cast<size_t>(g->C) * i;
                for (int k = 0; k < g->C; ++k) out[k] = 0.0;
                if (ok)
                    for (int j = 0; j < 8; ++j) {
                        const float* l =
                            &g->logits[static_cast<size_t>(g->C) *
                                       (static_cast<size_t>(cc.block[j]) * g->V + cc.voxel[j])];
                        for (int k = 0; k < g->C; ++k) out[k] += cc.w[j] * l[k];
                    }
            }
            if (valid) valid[i] = ok ? 1 : 0;
        }
    });
}

void svro_march(const svro_grid* g, const double* o, const double* d, uint64_t n, double step,
                uint32_t max_samples, uint32_t* counts, double* t, double* delta) {
    parallel_chunks(n, [&](size_t b, size_t e) {
        std::vector<Sample> s;
        for (size_t i = b; i < e; ++i) {
            march_ray(*g, o + 3 * i, d + 3 * i, step, max_samples, s);
            counts[i] = static_cast<uint32_t>(s.size());
            for (size_t k = 0; k < s.size(); ++k) {
                if (t) t[i * max_samples + k] = s[k].t;
                if (delta) delta[i * max_samples + k] = s[k].delta;
            }
        }
    });
}

double svro_sdf_to_density(double s, double beta) { return density(s, beta); }

// render_ray forward:
//   x_k = o + t_k d; invalid samples contribute tau = 0 (builder decision, SPEC.md:281
//   leaves them undefined); w_k = T_k (1 - exp(-sigma_k delta_k)), T_{k+1} = T_k exp(-tau_k);
//   C = sum w c, D = sum w t, N = sum w grad(sdf) (world, un-normalised), W = sum w.
int svro_render_forward(const svro_grid* g, const double* o, const double* d, uint64_t n,
                        double step, uint32_t max_samples, double beta, double* rgb,
                        double* depth, double* normal, double* wsum, uint32_t* nsamples,
                        uint32_t* nvalid) {
    return guarded([&] {
        if (!(beta > 0.0)) throw Status(kConfig, "render: beta must be positive");
        if (!(step > 0.0)) throw Status(kConfig, "render: step must be positive");
        parallel_chunks(n, [&](size_t b, size_t e) {
            std::vector<Sample> s;
            for (size_t i = b; i < e; ++i) {
                march_ray(*g, o + 3 * i, d + 3 * i, step, max_samples, s);
                double T = 1.0, C[3] = {0, 0, 0}, D = 0, N[3] = {0, 0, 0}, W = 0;
                uint32_t nv = 0;
                for (const Sample& sm : s) {
                    double x[3];
                    for (int a = 0; a < 3; ++a) x[a] = o[3 * i + a] + sm.t * d[3 * i + a];
                    Corners cc;
                    if (!gather(*g, x, cc)) continue;
                    ++nv;
                    Interp it;
                    interpolate(*g, cc, it);
                    const double tau = density(it.s, beta) * sm.delta;
                    const double w = T * (1.0 - std::exp(-tau));
                    for (int a = 0; a < 3; ++a) {
                        C[a] += w * it.rgb[a];
                        N[a] += w * it.grad[a];
                    }
                    D += w * sm.t;
                    W += w;
                    T *= std::exp(-tau);
                }
                for (int a = 0; a < 3; ++a) {
                    if (rgb) rgb[3 * i + a] = C[a];
                    if (normal) normal[3 * i + a] = N[a];
                }
                if (depth) depth[i] = D;
                if (wsum) wsum[i] = W;
                if (nsamples) nsamples[i] = static_cast<uint32_t>(s.size());
                if (nvalid) nvalid[i] = nv;
            }
        });
    });
}

// backward_step, render part: with v_k = dC.c_k + dD t_k + dN.n_k
// and S_k = sum_{m>k} w_m v_m:  dL/dtau_k = T_{k+1} v_k - S_k,
// dL/ds_k = delta_k sigma'(s_k) dL/dtau_k, and per corner c of sample k
//   g_sdf[c] += w_c dL/ds_k + dw_c . (w_k dN),   g_rgb[c] += w_c w_k dC.
// Accumulates into grad_sdf[A*V] / grad_rgb[A*V*3] (caller zeroes); `active[A]`
// (optional) gets 1 for every block owning a corner of a valid sample.
int svro_render_backward(const svro_grid* g, const double* o, const double* d, uint64_t n,
                         double step, uint32_t max_samples, double beta, const double* d_rgb,
                         const double* d_depth, const double* d_normal, double* grad_sdf,
                         double* grad_rgb, uint8_t* active) {
    return guarded([&] {
        if (!(beta > 0.0)) throw Status(kConfig, "render: beta must be positive");
        if (!(step > 0.0)) throw Status(kConfig, "render: step must be positive");
        const bool atomic = g_threads > 1;
        auto add = [atomic](double& dst, double v) {
            if (atomic)
                std::atomic_ref<double>(dst).fetch_add(v, std::memory_order_relaxed);
            else
                dst += v;
        };
        parallel_chunks(n, [&](size_t b, size_t e) {
            std::vector<Sample> s;
            struct Rec {
                Corners cc;
                Interp it;
                double t, delta, w, Tn, v;
                bool valid;
            };
            std::vector<Rec> rec;
            for (size_t i = b; i < e; ++i) {
                march_ray(*g, o + 3 * i, d + 3 * i, step, max_samples, s);
                rec.resize(s.size());
                const double* dC = d_rgb + 3 * i;
                const double dD = d_depth[i];
                const double* dN = d_normal + 3 * i;
                double T = 1.0;
                for (size_t k = 0; k < s.size(); ++k) {
                    Rec& r = rec[k];
                    r.t = s[k].t;
                    r.delta = s[k].delta;
                    double x[3];
                    for (int a = 0; a < 3; ++a) x[a] = o[3 * i + a] + r.t * d[3 * i + a];
                    r.valid = gather(*g, x, r.cc);
                    if (!r.valid) {
                        r.w = 0.0;
                        r.Tn = T;
                        r.v = 0.0;
                        continue;
                    }
                    interpolate(*g, r.cc, r.it);
                    const double tau = density(r.it.s, beta) * r.delta;
                    r.w = T * (1.0 - std::exp(-tau));
                    T *= std::exp(-tau);
                    r.Tn = T;
                    r.v = dC[0] * r.it.rgb[0] + dC[1] * r.it.rgb[1] + dC[2] * r.it.rgb[2] +
                          dD * r.t + dN[0] * r.it.grad[0] + dN[1] * r.it.grad[1] +
                          dN[2] * r.it.grad[2];
                }
                double S = 0.0;
                for (size_t kk = s.size(); kk-- > 0;) {
                    const Rec& r = rec[kk];
                    if (!r.valid) continue;
                    const double sigma = density(r.it.s, beta);
                    const double dtau = r.Tn * r.v - S;
                    const double ds = r.delta * density_ds(r.it.s, sigma, beta) * dtau;
                    const double wn[3] = {r.w * dN[0], r.w * dN[1], r.w * dN[2]};
                    for (int c = 0; c < 8; ++c) {
                        const size_t vx = static_cast<size_t>(r.cc.block[c]) * g->V + r.cc.voxel[c];
                        const double gs = r.cc.w[c] * ds + (r.cc.dw[c][0] * wn[0] +
                                                            r.cc.dw[c][1] * wn[1] +
                                                            r.cc.dw[c][2] * wn[2]);
                        add(grad_sdf[vx], gs);
                        const double wc = r.cc.w[c] * r.w;
                        for (int a = 0; a < 3; ++a) add(grad_rgb[3 * vx + a], wc * dC[a]);
                        if (active)
                            std::atomic_ref<uint8_t>(active[r.cc.block[c]])
                                .store(1, std::memory_order_relaxed);
                    }
                    S += r.w * r.v;
                }
            }
        });
    });
}

// eikonal_loss (Eq. 16/18): mean over valid points of
// (|grad f(x)| - 1)^2, gradient (2 scale / N) (1 - 1/|g|) (g . dw_c) into grad_sdf.
int svro_eikonal(const svro_grid* g, const double* x, uint64_t n, double scale, double* grad_sdf,
                 uint8_t* active, double* loss, uint64_t* n_valid) {
    return guarded([&] {
        struct P {
            Corners cc;
            double gr[3];
            bool ok;
        };
        std::vector<P> pts(n);
        double sum = 0.0;
        uint64_t cnt = 0;
        for (uint64_t i = 0; i < n; ++i) {
            P& p = pts[i];
            p.ok = !g->coords.empty() && gather(*g, x + 3 * i, p.cc);
            if (!p.ok) continue;
            Interp it;
            interpolate(*g, p.cc, it);
            for (int a = 0; a < 3; ++a) p.gr[a] = it.grad[a];
            const double nrm = std::sqrt(p.gr[0] * p.gr[0] + p.gr[1] * p.gr[1] + p.gr[2] * p.gr[2]);
            sum += (nrm - 1.0) * (nrm - 1.0);
            ++cnt;
        }
        if (loss) *loss = cnt ? sum / static_cast<double>(cnt) : 0.0;
        if (n_valid) *n_valid = cnt;
        if (!cnt || !grad_sdf) return;
        const double coef = 2.0 * scale / static_cast<double>(cnt);
        for (uint64_t i = 0; i < n; ++i) {
            const P& p = pts[i];
            if (!p.ok) continue;
            const double nrm = std::sqrt(p.gr[0] * p.gr[0] + p.gr[1] * p.gr[1] + p.gr[2] * p.gr[2]);
            if (!(nrm > 0.0)) continue;
            const double k = coef * (1.0 - 1.0 / nrm);
            for (int c = 0; c < 8; ++c) {
                grad_sdf[static_cast<size_t>(p.cc.block[c]) * g->V + p.cc.voxel[c]] +=
                    k * (p.gr[0] * p.cc.dw[c][0] + p.gr[1] * p.cc.dw[c][1] + p.gr[2] * p.cc.dw[c][2]);
                if (active) active[p.cc.block[c]] = 1;
            }
        }
    });
}

// RMSProp over the active blocks, fp32 like the device:
//   v = alpha v + (1 - alpha) g^2,  theta -= lr g / (sqrt(v) + eps)   for sdf and rgb.
// rms_state is [A][V][4] (sdf, r, g, b), caller-owned.
int svro_rmsprop(svro_grid* g, const double* grad_sdf, const double* grad_rgb, const uint8_t* active,
                 float lr, float alpha, float eps, float* rms_state) {
    return guarded([&] {
        const size_t V = g->V;
        const float beta = 1.f - alpha;
        for (size_t b = 0; b < g->coords.size(); ++b) {
            if (!active[b]) continue;
            for (size_t v = 0; v < V; ++v) {
                const size_t i = b * V + v;
                float* r = rms_state + 4 * i;
                const float gv[4] = {static_cast<float>(grad_sdf[i]), static_cast<float>(grad_rgb[3 * i]),
                                     static_cast<float>(grad_rgb[3 * i + 1]),
                                     static_cast<float>(grad_rgb[3 * i + 2])};
                float* th[4] = {&g->sdf[i], &g->rgb[3 * i], &g->rgb[3 * i + 1], &g->rgb[3 * i + 2]};
                for (int k = 0; k < 4; ++k) {
                    r[k] = alpha * r[k] + beta * gv[k] * gv[k];
                    *th[k] -= lr * gv[k] / (std::sqrt(r[k]) + eps);
                }
            }
        }
    });
}

// save_grid / load_grid (grid_io.cpp:37-97), SDGV v1 little-endian.
int svro_save_sdgv(const svro_grid* g, const char* path) {
    return guarded([&] {
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Status(kData, std::string("save_grid: cannot open ") + path);
        const uint32_t ver = 1, B = g->B, C = g->C;
        const uint64_t n = g->coords.size();
        os.write("SDGV", 4);
        os.write(reinterpret_cast<const char*>(&ver), 4);
        os.write(reinterpret_cast<const char*>(&g->h), 8);
        os.write(reinterpret_cast<const char*>(&B), 4);
        os.write(reinterpret_cast<const char*>(&n), 8);
        os.write(reinterpret_cast<const char*>(&C), 4);
        const size_t V = g->V;
        for (size_t i = 0; i < n; ++i) {
            os.write(reinterpret_cast<const char*>(&g->coords[i]), 12);
            os.write(reinterpret_cast<const char*>(&g->sdf[i * V]), V * 4);
            os.write(reinterpret_cast<const char*>(&g->weight[i * V]), V * 4);
            os.write(reinterpret_cast<const char*>(&g->rgb[3 * i * V]), 3 * V * 4);
            os.write(reinterpret_cast<const char*>(&g->logits[g->C * i * V]), g->C * V * 4);
        }
        if (!os) throw Status(kData, std::string("save_grid: write failed for ") + path);
    });
}

int svro_load_sdgv(const char* path, svro_grid** out) {
    return guarded([&] {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw Status(kData, std::string("load_grid: cannot open ") + path);
        char magic[4];
        is.read(magic, 4);
        if (!is || std::memcmp(magic, "SDGV", 4) != 0) throw Status(kData, "load_grid: bad magic");
        uint32_t ver = 0, B = 0, C = 0;
        double h = 0;
        uint64_t n = 0;
        is.read(reinterpret_cast<char*>(&ver), 4);
        if (ver != 1) throw Status(kData, "load_grid: unsupported version");
        is.read(reinterpret_cast<char*>(&h), 8);
        is.read(reinterpret_cast<char*>(&B), 4);
        is.read(reinterpret_cast<char*>(&n), 8);
        is.read(reinterpret_cast<char*>(&C), 4);
        if (!is) throw Status(kData, "load_grid: truncated header");
        svro_grid* g = nullptr;
        const int st = svro_grid_create(h, static_cast<int>(B), static_cast<int>(C),
                                        std::max<uint64_t>(1u << 21, n), &g);
        if (st) throw Status(st, g_err);
        std::unique_ptr<svro_grid> hold(g);
        const size_t V = g->V;
        for (uint64_t i = 0; i < n; ++i) {
            BlockCoord c;
            is.read(reinterpret_cast<char*>(&c), 12);
            const uint32_t idx = g->allocate_block(c);
            is.read(reinterpret_cast<char*>(&g->sdf[idx * V]), V * 4);
            is.read(reinterpret_cast<char*>(&g->weight[idx * V]), V * 4);
            is.read(reinterpret_cast<char*>(&g->rgb[3 * idx * V]), 3 * V * 4);
            is.read(reinterpret_cast<char*>(&g->logits[g->C * idx * V]), g->C * V * 4);
            if (!is) throw Status(kData, "load_grid: truncated block data");
        }
        *out = hold.release();
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Fusion + de-noising (Eq. 9-11).  The reference ships
// no code for this module; this is the restatement of the SPEC's contract with the
// decisions the product shares:
//   * association: voxel centre v*h (grid.hpp:124) -> Camera::project (camera.cpp:7-18,
//     R^T (x - t) accumulated left to right, z <= 1e-6 = behind, pixel_in_frame margin 0)
//     -> nearest pixel floor(p + 0.5); depth <= 0 or ScaleField value <= 0 -> no association
//   * d = D(p) phi(p) - z_v  (positive in front of the surface, the grid's SDF sign; the
//     SPEC examples fix the sign: d = -0.5 "behind surface" is rejected), reject d < -mu,
//     integrate psi = min(d, mu)
//   * running sums in 32.32 fixed point (int64): integer addition is associative, so any
//     frame order gives bit-identical sums/counts (SPEC.md:227 order-independence)
//   * finalize: mean = sum * 2^-32 / count; logits scaled to unit L2 norm (Eq. 11);
//     weight = count (grid.hpp:57-58: weight doubles as the observation count)
//   * denoise: num/den of a separable Gaussian over the (2r+1)^3 neighbourhood restricted
//     to valid voxels, accumulated x, then y, then z in fp64; invalid voxels unchanged.
// ---------------------------------------------------------------------------
namespace {
constexpr double kFix = 4294967296.0;          // 2^32
constexpr double kInvFix = 1.0 / 4294967296.0;  // 2^-32 (exact)

inline int64_t to_fix(double v) { return static_cast<int64_t>(std::nearbyint(v * kFix)); }

// Camera::project + pixel_in_frame (camera.cpp:7-18, camera.hpp:23-25,39-42).
bool project_px(const svro_camera& c, const double x[3], double& px, double& py, double& z) {
    const double d[3] = {x[0] - c.t[0], x[1] - c.t[1], x[2] - c.t[2]};
    double xc[3];
    for (int r = 0; r < 3; ++r) {  // (R^T)(r, k) = R(k, r)
        double acc = c.R[r] * d[0];
        acc = acc + c.R[3 + r] * d[1];
        acc = acc + c.R[6 + r] * d[2];
        xc[r] = acc;
    }
    if (xc[2] <= 1e-6) return false;
    z = xc[2];
    px = c.fx * xc[0] / xc[2] + c.cx;
    py = c.fy * xc[1] / xc[2] + c.cy;
    return px >= 0.0 && px <= c.width - 1 - 0.0 && py >= 0.0 && py <= c.height - 1 - 0.0;
}
}  // namespace

extern "C" {

int svro_fuse_begin(svro_grid* g, int flags) {
    return guarded([&] {
        if (flags & ~3) throw Status(kConfig, "fuse_begin: unknown flags");
        g->fuse_flags = flags;
        g->fsum.assign(g->coords.size() * g->V * (4 + g->C), 0);
        g->fcount.assign(g->coords.size() * g->V, 0);
    });
}

int svro_fuse_frames(svro_grid* g, const float* depth, const float* rgb, const float* sem,
                     const svro_camera* cams, uint32_t n_frames, const double* scales, int sf_rows,
                     int sf_cols, double mu, svro_fuse_report* rep) {
    svro_fuse_report r{};
    const int st = guarded([&] {
        if (g->fuse_flags < 0) throw Status(kConfig, "fuse: no session (fuse_begin)");
        if (!(mu > 0.0) || !(mu < 524288.0)) throw Status(kConfig, "fuse: mu must be in (0, 2^19)");
        if (((g->fuse_flags & 1) != 0) != (rgb != nullptr) || ((g->fuse_flags & 2) != 0) != (sem != nullptr))
            throw Status(kConfig, "fuse: channels differ from the session's flags");
        if (scales && (sf_rows < 2 || sf_cols < 2)) throw Status(kConfig, "scale field needs at least a 2x2 grid");
        if (n_frames == 0) return;
        const int W = cams[0].width, H = cams[0].height;
        for (uint32_t f = 0; f < n_frames; ++f)
            if (cams[f].width != W || cams[f].height != H)
                throw Status(kConfig, "fuse: all frames must share one size");
        if (scales && (W < 2 || H < 2)) throw Status(kConfig, "scale field image size too small");
        const size_t V = g->V, K = 4 + g->C, nb = g->coords.size();
        g->fsum.resize(nb * V * K, 0);  // blocks allocated since fuse_begin start empty
        g->fcount.resize(nb * V, 0);
        const int B = g->B, C = g->C;
        std::atomic<uint64_t> a_in{0}, a_rej{0};
        parallel_chunks(nb, [&](size_t b0, size_t b1) {
            uint64_t in = 0, rej = 0;
            for (size_t b = b0; b < b1; ++b)
                for (size_t v = 0; v < V; ++v) {
                    const int lx = static_cast<int>(v % B), ly = static_cast<int>((v / B) % B),
                              lz = static_cast<int>(v / (B * B));
                    const BlockCoord& bc = g->coords[b];
                    const double x[3] = {static_cast<double>(bc.x * B + lx) * g->h,
                                         static_cast<double>(bc.y * B + ly) * g->h,
                                         static_cast<double>(bc.z * B + lz) * g->h};
                    const size_t i = b * V + v;
                    for (uint32_t f = 0; f < n_frames; ++f) {
                        double px, py, z;
                        if (!project_px(cams[f], x, px, py, z)) continue;
                        const int ix = static_cast<int>(std::floor(px + 0.5));
                        const int iy = static_cast<int>(std::floor(py + 0.5));
                        const size_t pix = static_cast<size_t>(f) * W * H + static_cast<size_t>(iy) * W + ix;
                        const float D = depth[pix];
                        if (!(D > 0.0f)) continue;
                        const double phi = scales ? scale_value(scales + static_cast<size_t>(f) * sf_rows * sf_cols,
                                                                sf_rows, sf_cols, W, H, ix, iy)
                                                  : 1.0;
                        if (!(phi > 0.0)) continue;
                        ++in;
                        const double d = static_cast<double>(D) * phi - z;
                        if (d < -mu) {
                            ++rej;
                            continue;
                        }
                        int64_t* s = &g->fsum[i * K];
                        s[0] += to_fix(std::min(d, mu));
                        if (rgb)
                            for (int c = 0; c < 3; ++c) s[1 + c] += to_fix(static_cast<double>(rgb[3 * pix + c]));
                        if (sem)
                            for (int k = 0; k < C; ++k)
                                s[4 + k] += to_fix(static_cast<double>(sem[static_cast<size_t>(C) * pix + k]));
                        ++g->fcount[i];
                    }
                }
            a_in += in;
            a_rej += rej;
        });
        r.frames = n_frames;
        r.in_view = a_in;
        r.rejected = a_rej;
        r.integrated = r.in_view - r.rejected;
    });
    if (rep) *rep = r;
    return st;
}

int svro_fuse_finalize(svro_grid* g) {
    return guarded([&] {
        if (g->fuse_flags < 0) throw Status(kConfig, "fuse: no session (fuse_begin)");
        const size_t V = g->V, K = 4 + g->C, C = g->C, nb = g->coords.size();
        g->fsum.resize(nb * V * K, 0);
        g->fcount.resize(nb * V, 0);
        for (size_t i = 0; i < nb * V; ++i) {
            const uint32_t n = g->fcount[i];
            g->weight[i] = static_cast<float>(n);
            if (!n) continue;
            const double dn = static_cast<double>(n);
            const int64_t* s = &g->fsum[i * K];
            g->sdf[i] = static_cast<float>(static_cast<double>(s[0]) * kInvFix / dn);
            if (g->fuse_flags & 1)
                for (int c = 0; c < 3; ++c)
                    g->rgb[3 * i + c] = static_cast<float>(static_cast<double>(s[1 + c]) * kInvFix / dn);
            if (g->fuse_flags & 2) {
                double m[64];
                double nrm2 = 0.0;
                for (size_t k = 0; k < C; ++k) {
                    m[k] = static_cast<double>(s[4 + k]) * kInvFix / dn;
                    nrm2 = nrm2 + m[k] * m[k];
                }
                const double nrm = std::sqrt(nrm2);
                for (size_t k = 0; k < C; ++k)
                    g->logits[C * i + k] = nrm > 0.0 ? static_cast<float>(m[k] / nrm) : 0.0f;
            }
        }
        g->fuse_flags = -1;
        std::vector<int64_t>().swap(g->fsum);
        std::vector<uint32_t>().swap(g->fcount);
    });
}

int svro_denoise(svro_grid* g, double sigma_vox, int radius) {
    return guarded([&] {
        if (!(sigma_vox > 0.0)) throw Status(kConfig, "denoise: sigma must be positive");
        if (radius < 0 || radius > 4) throw Status(kConfig, "denoise: radius must be in [0, 4]");
        if (g->C > 64) throw Status(kConfig, "denoise: at most 64 label channels");
        double gw[9];
        for (int d = -radius; d <= radius; ++d)
            gw[d + radius] = std::exp(-static_cast<double>(d * d) / (2.0 * sigma_vox * sigma_vox));
        const int B = g->B, C = g->C, K = 4 + C;
        const size_t V = g->V, nb = g->coords.size();
        const std::vector<float> sdf0 = g->sdf, rgb0 = g->rgb, lg0 = g->logits;
        // valid neighbour voxel -> flat index, else -1
        auto locate = [&](int vx, int vy, int vz) -> int64_t {
            const BlockCoord bc = g->block_of_voxel(vx, vy, vz);
            const uint32_t bi = g->map.find(bc);
            if (bi == kInvalid) return -1;
            const size_t i = static_cast<size_t>(bi) * V + g->local_index(vx, vy, vz, bc);
            return g->weight[i] > 0.0f ? static_cast<int64_t>(i) : -1;
        };
        auto prop = [&](size_t i, int k) -> double {
            if (k == 0) return sdf0[i];
            if (k < 4) return rgb0[3 * i + k - 1];
            return lg0[static_cast<size_t>(C) * i + k - 4];
        };
        parallel_chunks(nb, [&](size_t b0, size_t b1) {
            std::vector<double> num(K);
            for (size_t b = b0; b < b1; ++b)
                for (size_t v = 0; v < V; ++v) {
                    const size_t i = b * V + v;
                    if (!(g->weight[i] > 0.0f)) continue;
                    const BlockCoord& bc = g->coords[b];
                    const int cx = bc.x * B + static_cast<int>(v % B);
                    const int cy = bc.y * B + static_cast<int>((v / B) % B);
                    const int cz = bc.z * B + static_cast<int>(v / (B * B));
                    std::fill(num.begin(), num.end(), 0.0);
                    double den = 0.0;
                    for (int dz = -radius; dz <= radius; ++dz) {
                        std::vector<double> ny(K, 0.0);
                        double dy_den = 0.0;
                        for (int dy = -radius; dy <= radius; ++dy) {
                            std::vector<double> nx(K, 0.0);
                            double dx_den = 0.0;
                            for (int dx = -radius; dx <= radius; ++dx) {
                                const int64_t j = locate(cx + dx, cy + dy, cz + dz);
                                const double w = gw[dx + radius];
                                for (int k = 0; k < K; ++k) nx[k] = nx[k] + w * (j >= 0 ? prop(j, k) : 0.0);
                                dx_den = dx_den + w * (j >= 0 ? 1.0 : 0.0);
                            }
                            const double w = gw[dy + radius];
                            for (int k = 0; k < K; ++k) ny[k] = ny[k] + w * nx[k];
                            dy_den = dy_den + w * dx_den;
                        }
                        const double w = gw[dz + radius];
                        for (int k = 0; k < K; ++k) num[k] = num[k] + w * ny[k];
                        den = den + w * dy_den;
                    }
                    g->sdf[i] = static_cast<float>(num[0] / den);
                    for (int c = 0; c < 3; ++c) g->rgb[3 * i + c] = static_cast<float>(num[1 + c] / den);
                    for (int k = 0; k < C; ++k) g->logits[static_cast<size_t>(C) * i + k] = static_cast<float>(num[4 + k] / den);
                }
        });
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Marching cubes (meshing.cpp:168-273) + the 256-case table it builds (meshing.cpp:56-150),
// restated.  Table rules: edges are the corner pairs differing in one bit, numbered
// axis * 4 + rank of the lower corner among the corners with that bit clear; faces are
// cyclic quads (base, base+u, base+u+v, base+v) with (u, v) the other two axes in
// increasing order, x faces then y then z, side 0 before side 1.  On a face, 2 sign
// changes pair up; 4 (alternating) pair so that each inside corner is cut off by the two
// edges next to it.  Segments chain into loops, walked from the lowest edge; a loop whose
// midpoint polygon normal points from the outside corners to the inside ones is reversed;
// loops are fan-triangulated from their first edge.
// ---------------------------------------------------------------------------
namespace {
struct McTable {
    int edge_a[12], edge_b[12], edge_axis[12];
    std::vector<std::array<int, 3>> tris[256];
};

const McTable& mc_table() {
    static const McTable T = [] {
        McTable t{};
        for (int a = 0; a < 3; ++a) {
            int slot = 0;
            for (int c = 0; c < 8; ++c)
                if (!((c >> a) & 1)) {
                    t.edge_a[a * 4 + slot] = c;
                    t.edge_b[a * 4 + slot] = c | (1 << a);
                    t.edge_axis[a * 4 + slot] = a;
                    ++slot;
                }
        }
        auto edge_of = [&](int p, int q) {
            for (int e = 0; e < 12; ++e)
                if ((t.edge_a[e] == p && t.edge_b[e] == q) || (t.edge_a[e] == q && t.edge_b[e] == p)) return e;
            return -1;
        };
        int faces[6][4];
        for (int a = 0, f = 0; a < 3; ++a) {
            const int u = a == 0 ? 1 : 0, v = a == 2 ? 1 : 2;
            for (int side = 0; side < 2; ++side, ++f) {
                const int b = side << a;
                faces[f][0] = b;
                faces[f][1] = b | (1 << u);
                faces[f][2] = b | (1 << u) | (1 << v);
                faces[f][3] = b | (1 << v);
            }
        }
        for (int cfg = 0; cfg < 256; ++cfg) {
            auto in = [&](int c) { return (cfg >> c) & 1; };
            int nbr[12][2], deg[12] = {0};
            auto join = [&](int e, int f) {
                nbr[e][deg[e]++] = f;
                nbr[f][deg[f]++] = e;
            };
            for (const auto& q : faces) {
                int cut[4], n = 0;
                for (int i = 0; i < 4; ++i)
                    if (in(q[i]) != in(q[(i + 1) & 3])) cut[n++] = edge_of(q[i], q[(i + 1) & 3]);
                if (n == 2) join(cut[0], cut[1]);
                if (n == 4)
                    for (int k = 0; k < 4; ++k)  // each inside corner: its two incident edges
                        if (in(q[k])) join(edge_of(q[(k + 3) & 3], q[k]), edge_of(q[k], q[(k + 1) & 3]));
            }
            bool seen[12] = {false};
            for (int e0 = 0; e0 < 12; ++e0) {
                if (deg[e0] != 2 || seen[e0]) continue;
                std::vector<int> loop;
                int cur = e0, prev = -1;
                do {
                    loop.push_back(cur);
                    seen[cur] = true;
                    const int nx = nbr[cur][0] == prev ? nbr[cur][1] : nbr[cur][0];
                    prev = cur;
                    cur = nx;
                } while (cur != e0);
                if (loop.size() < 3) continue;
                // orientation: sum of mid_i x mid_{i+1} vs (mean outside corner - mean inside corner)
                auto mid = [&](int e, int a) {
                    return 0.5 * (((t.edge_a[e] >> a) & 1) + ((t.edge_b[e] >> a) & 1));
                };
                double nrm[3] = {0, 0, 0};
                for (size_t i = 0; i < loop.size(); ++i) {
                    const int e = loop[i], f = loop[(i + 1) % loop.size()];
                    nrm[0] += mid(e, 1) * mid(f, 2) - mid(e, 2) * mid(f, 1);
                    nrm[1] += mid(e, 2) * mid(f, 0) - mid(e, 0) * mid(f, 2);
                    nrm[2] += mid(e, 0) * mid(f, 1) - mid(e, 1) * mid(f, 0);
                }
                double mi[3] = {0, 0, 0}, mo[3] = {0, 0, 0};
                int ni = 0, no = 0;
                for (int c = 0; c < 8; ++c) {
                    double* m = in(c) ? mi : mo;
                    (in(c) ? ni : no) += 1;
                    for (int a = 0; a < 3; ++a) m[a] += (c >> a) & 1;
                }
                double dot = 0.0;
                for (int a = 0; a < 3; ++a)
                    dot += nrm[a] * (mo[a] / std::max(no, 1) - mi[a] / std::max(ni, 1));
                if (dot < 0.0) std::reverse(loop.begin(), loop.end());
                for (size_t i = 1; i + 1 < loop.size(); ++i) t.tris[cfg].push_back({loop[0], loop[i], loop[i + 1]});
            }
        }
        return t;
    }();
    return T;
}
}  // namespace

extern "C" {

int svro_mc_table(int32_t* counts, int32_t* tris) {  // counts[256], tris[256][16][3] (-1 pad)
    const McTable& t = mc_table();
    for (int c = 0; c < 256; ++c) {
        counts[c] = static_cast<int32_t>(t.tris[c].size());
        for (int i = 0; i < 16; ++i)
            for (int k = 0; k < 3; ++k)
                tris[(c * 16 + i) * 3 + k] = i < static_cast<int>(t.tris[c].size()) ? t.tris[c][i][k] : -1;
    }
    return 0;
}

int svro_marching_cubes(svro_grid* g, double iso, uint64_t* n_vertices, uint64_t* n_triangles) {
    return guarded([&] {
        const McTable& T = mc_table();
        const int B = g->B;
        const size_t V = g->V, nb = g->coords.size();
        // corner value: allocated and observed (meshing.cpp:175-184)
        auto corner = [&](int vx, int vy, int vz, double& sdf) {
            const BlockCoord bc = g->block_of_voxel(vx, vy, vz);
            const uint32_t bi = g->map.find(bc);
            if (bi == kInvalid) return false;
            const size_t i = static_cast<size_t>(bi) * V + g->local_index(vx, vy, vz, bc);
            if (!(g->weight[i] > 0.0f)) return false;
            sdf = g->sdf[i];
            return true;
        };
        struct Raw {
            int64_t key[3][4];
            double p[3][3];
        };
        std::vector<std::vector<Raw>> per(nb);
        parallel_chunks(nb, [&](size_t b0, size_t b1) {
            for (size_t b = b0; b < b1; ++b) {
                const BlockCoord& bc = g->coords[b];
                for (int lz = 0; lz < B; ++lz)
                    for (int ly = 0; ly < B; ++ly)
                        for (int lx = 0; lx < B; ++lx) {
                            const int ax = bc.x * B + lx, ay = bc.y * B + ly, az = bc.z * B + lz;
                            double s[8];
                            bool ok = true;
                            for (int c = 0; c < 8 && ok; ++c)
                                ok = corner(ax + (c & 1), ay + ((c >> 1) & 1), az + ((c >> 2) & 1), s[c]);
                            if (!ok) continue;
                            int cfg = 0;
                            for (int c = 0; c < 8; ++c)
                                if (s[c] < iso) cfg |= 1 << c;
                            for (const auto& tri : T.tris[cfg]) {
                                Raw r;
                                for (int k = 0; k < 3; ++k) {
                                    const int e = tri[k], ca = T.edge_a[e], cb = T.edge_b[e], axis = T.edge_axis[e];
                                    const int va[3] = {ax + (ca & 1), ay + ((ca >> 1) & 1), az + ((ca >> 2) & 1)};
                                    const double tt = (iso - s[ca]) / (s[cb] - s[ca]);
                                    for (int a = 0; a < 3; ++a) r.p[k][a] = static_cast<double>(va[a]) * g->h;
                                    r.p[k][axis] += tt * g->h;
                                    r.key[k][0] = va[0], r.key[k][1] = va[1], r.key[k][2] = va[2], r.key[k][3] = axis;
                                }
                                per[b].push_back(r);
                            }
                        }
            }
        });
        // first-occurrence vertex numbering + degenerate / zero-area filter (meshing.cpp:233-251)
        struct KeyH {
            size_t operator()(const std::array<int64_t, 4>& k) const {
                uint64_t h = static_cast<uint64_t>(k[0]) * 0x9E3779B97F4A7C15ull;
                h ^= static_cast<uint64_t>(k[1]) * 0xBF58476D1CE4E5B9ull + (h >> 31);
                h ^= static_cast<uint64_t>(k[2]) * 0x94D049BB133111EBull + (h >> 29);
                return static_cast<size_t>(h ^ static_cast<uint64_t>(k[3]));
            }
        };
        std::unordered_map<std::array<int64_t, 4>, int32_t, KeyH> vid;
        g->mv.clear(), g->mt.clear();
        for (const auto& list : per)
            for (const Raw& r : list) {
                int32_t idx[3];
                for (int k = 0; k < 3; ++k) {
                    const std::array<int64_t, 4> key{r.key[k][0], r.key[k][1], r.key[k][2], r.key[k][3]};
                    auto it = vid.find(key);
                    if (it == vid.end()) {
                        it = vid.emplace(key, static_cast<int32_t>(g->mv.size() / 3)).first;
                        g->mv.insert(g->mv.end(), r.p[k], r.p[k] + 3);
                    }
                    idx[k] = it->second;
                }
                if (idx[0] == idx[1] || idx[1] == idx[2] || idx[0] == idx[2]) continue;
                const double* v0 = &g->mv[3 * idx[0]];
                const double* v1 = &g->mv[3 * idx[1]];
                const double* v2 = &g->mv[3 * idx[2]];
                const double e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
                const double e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
                const double c[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                                     e1[0] * e2[1] - e1[1] * e2[0]};
                if (0.5 * std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]) <= 1e-12) continue;
                g->mt.insert(g->mt.end(), idx, idx + 3);
            }
        // vertex attributes from fp64 trilinear queries (meshing.cpp:254-270)
        const size_t nv = g->mv.size() / 3;
        g->mn.assign(3 * nv, 0.0);
        g->mc.assign(3 * nv, 0.0);
        g->ml.assign(nv, 0);
        parallel_chunks(nv, [&](size_t i0, size_t i1) {
            std::vector<double> lg(g->C);
            for (size_t i = i0; i < i1; ++i) {
                g->mn[3 * i + 2] = 1.0;  // UnitZ default
                Corners cc;
                if (!gather(*g, &g->mv[3 * i], cc)) continue;
                Interp it{};
                interpolate(*g, cc, it);
                const double n2 = it.grad[0] * it.grad[0] + it.grad[1] * it.grad[1] + it.grad[2] * it.grad[2];
                if (std::sqrt(n2) > 1e-12) {
                    const double n = std::sqrt(n2);  // normalized(): v / sqrt(squaredNorm)
                    for (int a = 0; a < 3; ++a) g->mn[3 * i + a] = it.grad[a] / n;
                }
                for (int a = 0; a < 3; ++a) g->mc[3 * i + a] = std::min(std::max(it.rgb[a], 0.0), 1.0);
                std::fill(lg.begin(), lg.end(), 0.0);
                for (int j = 0; j < 8; ++j) {
                    const float* l = &g->logits[static_cast<size_t>(g->C) *
                                                (static_cast<size_t>(cc.block[j]) * g->V + cc.voxel[j])];
                    for (int k = 0; k < g->C; ++k) lg[k] += cc.w[j] * l[k];
                }
                g->ml[i] = static_cast<int32_t>(std::max_element(lg.begin(), lg.end()) - lg.begin());
            }
        });
        *n_vertices = nv;
        *n_triangles = g->mt.size() / 3;
    });
}

int svro_mesh_get(const svro_grid* g, double* v, double* n, double* c, int32_t* labels, int32_t* tris) {
    if (v) std::memcpy(v, g->mv.data(), g->mv.size() * 8);
    if (n) std::memcpy(n, g->mn.data(), g->mn.size() * 8);
    if (c) std::memcpy(c, g->mc.data(), g->mc.size() * 8);
    if (labels) std::memcpy(labels, g->ml.data(), g->ml.size() * 4);
    if (tris) std::memcpy(tris, g->mt.data(), g->mt.size() * 4);
    return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Refinement losses (SPEC.md:286-319 backward_step, PAPER Eq. 12-14, 23): the per-ray
// upstream gradients render_backward consumes.  Restatement with the SPEC's decisions:
//   participating ray: rendered wsum > 0 (>= 1 valid sample; degenerate rays excluded)
//   L_c = mean_rays sum_ch |C - C*|                      (colour L1)
//   L_d = mean_rays (t - (a D + b))^2, D > 0; (a, b) = least squares of t on D over the batch
//         (2x2 normal equations in fp64; singular or < 2 rays: a = 1, b = mean(t - D))
//   L_n = mean_rays |normalize(R^T N) - n*|_1, |n*| > 0, |R^T N| > 1e-12
//   total = L_c + lambda_d L_d + lambda_n L_n;  d/d(a, b) = 0 at the optimum (envelope)
// ---------------------------------------------------------------------------
namespace {
inline double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// (a, b) of the depth prior; *singular set when the fallback was used
void depth_fit(const double* S, double& a, double& b, bool& singular) {
    // S = {n, sum D, sum D^2, sum t, sum D t}
    const double det = S[0] * S[2] - S[1] * S[1];
    singular = !(S[0] >= 2.0) || !(det > 1e-12 * S[0] * S[2]);
    if (singular) {
        a = 1.0;
        b = S[0] > 0.0 ? (S[3] - S[1]) / S[0] : 0.0;
    } else {
        a = (S[0] * S[4] - S[1] * S[3]) / det;
        b = (S[3] - a * S[1]) / S[0];
    }
}
}  // namespace

extern "C" {

int svro_fit_depth_affine(const double* t, const double* D, uint64_t n, double* a, double* b) {
    double S[5] = {0, 0, 0, 0, 0};
    for (uint64_t i = 0; i < n; ++i) {
        S[0] += 1.0;
        S[1] += D[i];
        S[2] += D[i] * D[i];
        S[3] += t[i];
        S[4] += D[i] * t[i];
    }
    bool singular = false;
    depth_fit(S, *a, *b, singular);
    return singular ? 1 : 0;
}

int svro_render_losses(uint64_t n, const double* rgb, const double* depth, const double* normal,
                       const double* wsum, const float* tgt_rgb, const float* prior_depth,
                       const float* prior_normal, const uint32_t* cam_idx, const svro_camera* cams,
                       double lambda_d, double lambda_n, double* d_rgb, double* d_depth, double* d_normal,
                       double* stats) {
    return guarded([&] {
        double S[5] = {0, 0, 0, 0, 0};
        uint64_t nc = 0, nn = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (!(wsum[i] > 0.0)) continue;
            ++nc;
            if (prior_depth && prior_depth[i] > 0.0f) {
                const double D = prior_depth[i], t = depth[i];
                S[0] += 1.0, S[1] += D, S[2] += D * D, S[3] += t, S[4] += D * t;
            }
        }
        double a = 1.0, b = 0.0;
        bool singular = false;
        depth_fit(S, a, b, singular);
        const double nd = S[0];
        // normal term participation needs the camera-frame normal
        std::vector<double> ncam(3 * n, 0.0), len(n, 0.0);
        if (prior_normal)
            for (uint64_t i = 0; i < n; ++i) {
                if (!(wsum[i] > 0.0)) continue;
                const float* ps = prior_normal + 3 * i;
                if (!(ps[0] != 0.0f || ps[1] != 0.0f || ps[2] != 0.0f)) continue;
                const double* R = cams[cam_idx[i]].R;
                double* c = &ncam[3 * i];
                for (int r = 0; r < 3; ++r)  // R^T N
                    c[r] = R[r] * normal[3 * i] + R[3 + r] * normal[3 * i + 1] + R[6 + r] * normal[3 * i + 2];
                len[i] = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
                if (len[i] > 1e-12) ++nn;
            }
        double Lc = 0.0, Ld = 0.0, Ln = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            double* gc = d_rgb + 3 * i;
            double* gn = d_normal + 3 * i;
            gc[0] = gc[1] = gc[2] = 0.0;
            gn[0] = gn[1] = gn[2] = 0.0;
            d_depth[i] = 0.0;
            if (!(wsum[i] > 0.0)) continue;
            for (int k = 0; k < 3; ++k) {
                const double e = rgb[3 * i + k] - tgt_rgb[3 * i + k];
                Lc += std::fabs(e);
                gc[k] = sgn(e) / nc;
            }
            if (prior_depth && prior_depth[i] > 0.0f) {
                const double r = depth[i] - (a * prior_depth[i] + b);
                Ld += r * r;
                d_depth[i] = lambda_d * 2.0 * r / nd;
            }
            if (len[i] > 1e-12) {
                const double* c = &ncam[3 * i];
                const double nh[3] = {c[0] / len[i], c[1] / len[i], c[2] / len[i]};
                const float* ps = prior_normal + 3 * i;
                double sg[3];
                for (int k = 0; k < 3; ++k) {
                    const double e = nh[k] - ps[k];
                    Ln += std::fabs(e);
                    sg[k] = sgn(e);
                }
                const double dot = nh[0] * sg[0] + nh[1] * sg[1] + nh[2] * sg[2];
                double gcam[3];
                for (int k = 0; k < 3; ++k) gcam[k] = (sg[k] - nh[k] * dot) / len[i] * (lambda_n / nn);
                const double* R = cams[cam_idx[i]].R;
                for (int r = 0; r < 3; ++r)  // R gcam
                    gn[r] = R[3 * r] * gcam[0] + R[3 * r + 1] * gcam[1] + R[3 * r + 2] * gcam[2];
            }
        }
        Lc = nc ? Lc / nc : 0.0;
        Ld = nd > 0.0 ? Ld / nd : 0.0;
        Ln = nn ? Ln / nn : 0.0;
        stats[0] = Lc, stats[1] = Ld, stats[2] = Ln;
        stats[3] = Lc + lambda_d * Ld + lambda_n * Ln;
        stats[4] = a, stats[5] = b;
        stats[6] = static_cast<double>(nc), stats[7] = nd, stats[8] = static_cast<double>(nn);
        stats[9] = singular ? 1.0 : 0.0;
    });
}

}  // extern "C"
