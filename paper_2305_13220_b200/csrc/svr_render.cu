// sm_100a kernels of the rendering hot path:
//   K2 k_query     -- fp64 trilinear query, bit-exact with grid.cpp:112-261
//   K4 k_march     -- ray-block DDA + fixed-step sampling, bit-exact with grid.cpp:263-353
//   K5 k_forward   -- fused gather/interpolate/Laplace density/compositing, warp per ray
//   K6 k_backward  -- compositing adjoint (warp suffix scan) + trilinear adjoint +
//                     red.global.add.v4.f32 scatter into the float4 gradient planes
// Discrete decisions (which block/cell, sample t) use fp64 with explicit _rn
// intrinsics so nvcc cannot contract them into FMA (the reference's x86-64 Release
// build has no FMA, proj/CMakeLists.txt:9-11).  Continuous interpolation and
// compositing run in fp32 (tolerance in tests/test_gpu_render.py).
#include <cfloat>
#include <cstdint>

#include <cub/device/device_radix_sort.cuh>

#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// K2: query_sdf_with_gradient + color_at + logits_at (grid.cpp:112-261), fp64 with the
// reference's association order.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_query(GridView g, const double* __restrict__ x,
                                               uint64_t n, double* sdf, double* grad,
                                               double* rgb, double* logits, uint8_t* valid) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double xp[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    uint32_t gidx[8];
    double w[8], dw[8][3];
    const bool ok = gather_fp64(g, xp, gidx, w, dw);
    if (!ok) {
        if (sdf) sdf[i] = 0.0;
        for (int a = 0; a < 3; ++a) {
            if (grad) grad[3 * i + a] = 0.0;
            if (rgb) rgb[3 * i + a] = 0.0;
        }
        if (logits)
            for (int k = 0; k < g.C; ++k) logits[static_cast<uint64_t>(g.C) * i + k] = 0.0;
        if (valid) valid[i] = 0;
        return;
    }
    float4 p[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) p[c] = __ldg(g.pay + gidx[c]);
    double s = 0.0, gr[3] = {0.0, 0.0, 0.0}, col[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 8; ++c) s = __dadd_rn(s, __dmul_rn(w[c], static_cast<double>(p[c].x)));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double v = p[c].x;
        gr[0] = __dadd_rn(gr[0], __dmul_rn(dw[c][0], v));
        gr[1] = __dadd_rn(gr[1], __dmul_rn(dw[c][1], v));
        gr[2] = __dadd_rn(gr[2], __dmul_rn(dw[c][2], v));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        col[0] = __dadd_rn(col[0], __dmul_rn(w[c], static_cast<double>(p[c].y)));
        col[1] = __dadd_rn(col[1], __dmul_rn(w[c], static_cast<double>(p[c].z)));
        col[2] = __dadd_rn(col[2], __dmul_rn(w[c], static_cast<double>(p[c].w)));
    }
    if (sdf) sdf[i] = s;
    for (int a = 0; a < 3; ++a) {
        if (grad) grad[3 * i + a] = gr[a];
        if (rgb) rgb[3 * i + a] = col[a];
    }
    if (logits) {  // logits_at(CornerCacheD) grid.cpp:230-238
        for (int k = 0; k < g.C; ++k) {
            double acc = 0.0;
            for (int c = 0; c < 8; ++c)
                acc = __dadd_rn(acc, __dmul_rn(w[c], static_cast<double>(__ldg(
                                                         g.logits + static_cast<size_t>(gidx[c]) * g.C + k))));
            logits[static_cast<uint64_t>(g.C) * i + k] = acc;
        }
    }
    if (valid) valid[i] = 1;
}

// ---------------------------------------------------------------------------
// K4: march_intervals + march_ray (grid.cpp:263-353) fused into one DDA walk that
// emits samples per allocated block (equivalence argued in oracle/svr_oracle.cpp).
// Crossing times are recomputed from plane equations exactly as the reference does;
// only the stepped axis' crossing changes per step, so the other two are cached.
// ---------------------------------------------------------------------------
// o / d: anything indexable as o[a] (registers, or a strided shared-memory view)
template <typename V, typename Emit>
__device__ __forceinline__ uint32_t march_dev(const GridView& g, const V& o, const V& d, double step, uint32_t S,
                                              Emit&& emit) {
    if (g.n_blocks == 0 || S == 0) return 0;
    const double L = g.L;
    double t0 = 0.0, t1 = DBL_MAX;
#pragma unroll
    for (int a = 0; a < 3; ++a) {  // grid.cpp:270-285
        const double box_lo = __dmul_rn(static_cast<double>(g.lo[a]), L);
        const double box_hi = __dmul_rn(static_cast<double>(g.hi[a] + 1), L);
        if (d[a] == 0.0) {
            if (o[a] < box_lo || o[a] >= box_hi) return 0;
            continue;
        }
        const double ta = __ddiv_rn(__dsub_rn(box_lo, o[a]), d[a]);
        const double tb = __ddiv_rn(__dsub_rn(box_hi, o[a]), d[a]);
        t0 = smax(t0, smin(ta, tb));
        t1 = smin(t1, smax(ta, tb));
    }
    if (!(t0 < t1)) return 0;
    const double t_eps = __dmul_rn(1e-12, smax(1.0, fabs(t0)));  // grid.cpp:289-296
    const double ts = __dadd_rn(t0, t_eps);
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    // Scalar per-axis state (no local-memory arrays): block coordinate, step, crossing.
    int32_t b0, b1, b2;
    double c0, c1, c2;
    auto start_block = [&](int a) {
        const double st = __dadd_rn(o[a], __dmul_rn(ts, d[a]));
        int32_t v = static_cast<int32_t>(floor(__ddiv_rn(st, L)));
        return v < g.lo[a] ? g.lo[a] : (g.hi[a] < v ? g.hi[a] : v);  // std::clamp
    };
    auto crossing = [&](int a, int32_t bv) {  // grid.cpp:298-302, recomputed exactly
        if (d[a] == 0.0) return kInf;
        return __ddiv_rn(__dsub_rn(__dmul_rn(static_cast<double>(bv + (d[a] > 0.0 ? 1 : 0)), L), o[a]),
                         d[a]);
    };
    b0 = start_block(0), b1 = start_block(1), b2 = start_block(2);
    c0 = crossing(0, b0), c1 = crossing(1, b1), c2 = crossing(2, b2);
    const int32_t s0 = d[0] > 0.0 ? 1 : -1, s1 = d[1] > 0.0 ? 1 : -1, s2 = d[2] > 0.0 ? 1 : -1;

    const int32_t p0 = d[0] > 0.0 ? 1 : 0, p1 = d[1] > 0.0 ? 1 : 0, p2 = d[2] > 0.0 ? 1 : 0;
    // dense mode: occupancy bit index of (b0,b1,b2), updated incrementally per step
    // (the dense index is only built when the AABB has <= 2^28 cells)
    const int32_t st0 = s0, st1 = s1 * g.dim[0], st2 = s2 * g.dim[0] * g.dim[1];
    int32_t cell = ((b2 - g.lo[2]) * g.dim[1] + (b1 - g.lo[1])) * g.dim[0] + (b0 - g.lo[0]);
    const double half_step = __dmul_rn(0.5, step);
    double t = t0, cursor = -kInf;
    bool open = false;
    uint32_t cnt = 0;
    // The walk only records the allocated runs [a, b) (contiguous allocated blocks merge,
    // as march_intervals merges them); the samples are generated afterwards by the exact
    // repeated-addition cursor, so the emission loop is not nested in -- and divergent
    // with -- the DDA steps.  The walk stops once a conservative estimate of the samples
    // covered exceeds S by more than one per run (the exact count per run differs from
    // the estimate by at most one).
    constexpr int kRuns = 4;
    double ra[kRuns], rb[kRuns];
    int nr = 0;
    double est_cursor = -kInf;
    double est = 0.0;
    const double inv_step = 1.0 / step;
    auto flush = [&]() {  // exact samples of the recorded runs (grid.cpp:337-353)
        for (int i = 0; i < nr; ++i) {
            const double a = ra[i], b = rb[i];
            if (cursor < a) cursor = __dadd_rn(a, half_step);  // grid.cpp:345
            while (cursor < b && cnt < S) {                    // grid.cpp:346-349
                emit(cnt, cursor);
                ++cnt;
                cursor = __dadd_rn(cursor, step);
            }
        }
        nr = 0;
    };
    // Empty-space jump (dense mode): every block within Chebyshev distance dist - 1 of an
    // empty block is empty, so the walk may resume at the DDA state of a time t* that stays
    // inside that cube (one block of margin).  The state at t* is exact: per axis the
    // crossings before t* are counted with the same exactly-rounded crossing formula the
    // walk uses (crossings of one axis are monotone), so the blocks / crossings after the
    // jump are those the step-by-step walk reaches, and no sample is skipped (the cube is
    // empty).
    const double inv_md = 1.0 / fmax(fabs(d[0]), fmax(fabs(d[1]), fabs(d[2])));
    while (t < t1) {  // grid.cpp:306-333
        double t_exit = t1;
        int axis = -1;
        if (c0 < t_exit) t_exit = c0, axis = 0;
        if (c1 < t_exit) t_exit = c1, axis = 1;
        if (c2 < t_exit) t_exit = c2, axis = 2;
        int dist = 0;
        bool alloc;
        if (g.bdist) {
            dist = __ldg(g.bdist + static_cast<uint32_t>(cell));
            alloc = dist == 0;
        } else {
            alloc = g.use_dense
                        ? ((__ldg(g.occ + (static_cast<uint32_t>(cell) >> 5)) >> (cell & 31)) & 1u) != 0
                        : hash_find(g, pack_key(b0, b1, b2)) != kInvalid;
        }
        if (dist >= 3) {
            open = false;
            const double ts = t + (dist - 2) * L * inv_md;
            if (ts >= t1) break;  // the ray leaves the AABB inside empty space
            int32_t nbv[3] = {b0, b1, b2};
            double nc[3] = {c0, c1, c2};
            const int32_t sv[3] = {s0, s1, s2};
            bool out = false;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (d[a] == 0.0) continue;
                const int32_t b = nbv[a];
                const int32_t bx = static_cast<int32_t>(floor((o[a] + ts * d[a]) / L));
                int32_t m = (bx - b) * sv[a];
                m = m < 0 ? 0 : m;
                while (m > 0 && !(crossing(a, b + (m - 1) * sv[a]) < ts)) --m;
                double cm = crossing(a, b + m * sv[a]);
                while (cm < ts) {
                    ++m;
                    cm = crossing(a, b + m * sv[a]);
                }
                nbv[a] = b + m * sv[a];
                nc[a] = cm;
                if (nbv[a] < g.lo[a] || nbv[a] > g.hi[a]) out = true;
            }
            if (out) break;
            b0 = nbv[0], b1 = nbv[1], b2 = nbv[2];
            c0 = nc[0], c1 = nc[1], c2 = nc[2];
            cell = ((b2 - g.lo[2]) * g.dim[1] + (b1 - g.lo[1])) * g.dim[0] + (b0 - g.lo[0]);
            t = ts;
            continue;
        }
        if (alloc) {
            if (!open) {
                open = true;
                if (nr == kRuns) flush();
                ra[nr] = t;
                ++nr;
                if (est_cursor < t) est_cursor = t + half_step;
            }
            rb[nr - 1] = t_exit;
            if (est_cursor < t_exit) {  // estimate of the samples in [est_cursor, t_exit)
                const double k = ceil((t_exit - est_cursor) * inv_step);
                est += k;
                est_cursor += k * step;
            }
            if (est >= static_cast<double>(S) + nr + 1) break;
        } else {
            open = false;
        }
        if (axis < 0) break;
        t = t_exit;
        // step the chosen axis; one exactly-rounded division for its next crossing
        const bool a0 = axis == 0, a1 = axis == 1;
        const int32_t nb = (a0 ? b0 : (a1 ? b1 : b2)) + (a0 ? s0 : (a1 ? s1 : s2));
        const int32_t lo_a = a0 ? g.lo[0] : (a1 ? g.lo[1] : g.lo[2]);
        const int32_t hi_a = a0 ? g.hi[0] : (a1 ? g.hi[1] : g.hi[2]);
        if (nb < lo_a || nb > hi_a) break;
        cell += a0 ? st0 : (a1 ? st1 : st2);
        const double oa = a0 ? o[0] : (a1 ? o[1] : o[2]);
        const double da = a0 ? d[0] : (a1 ? d[1] : d[2]);
        const int32_t pa = a0 ? p0 : (a1 ? p1 : p2);
        const double c = __ddiv_rn(__dsub_rn(__dmul_rn(static_cast<double>(nb + pa), L), oa), da);
        if (a0) b0 = nb, c0 = c;
        else if (a1) b1 = nb, c1 = c;
        else b2 = nb, c2 = c;
    }
    flush();
    return cnt;
}

// per-thread o / d kept in shared memory (SoA, stride = CTA size) instead of 12 registers
struct StridedVec {
    const double* base;
    int stride;
    __device__ __forceinline__ double operator[](int a) const { return base[a * stride]; }
};

__device__ __forceinline__ uint32_t spread3(uint32_t v);
// Morton code of the block holding a ray's first sample (k_ray_keys mode 0), computed by the
// march from the t it has just emitted; rays without samples sort last.
template <typename V>
__device__ __forceinline__ uint32_t first_sample_key(const GridView& g, const V& o, const V& d, uint32_t cnt,
                                                     double t) {
    if (!cnt) return 0xFFFFFFFFu;
    uint32_t b[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = o[a] + t * d[a];
        int32_t v = static_cast<int32_t>(floor(x / g.L)) - g.lo[a];
        v = v < 0 ? 0 : (v > 1023 ? 1023 : v);
        b[a] = static_cast<uint32_t>(v);
    }
    return spread3(b[0]) | (spread3(b[1]) << 1) | (spread3(b[2]) << 2);
}

template <int kMinBlocks, bool kSmem, int kThreads = 128>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_march(GridView g, const double* __restrict__ O,
                                               const double* __restrict__ D, uint64_t n,
                                               const uint32_t* __restrict__ order, double step,
                                               uint32_t S, uint32_t* counts, double* T, double* delta,
                                               uint32_t* pkeys = nullptr, uint32_t* pids = nullptr) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t r = order ? order[i] : i;
    double* tr = T + r * S;
    uint32_t cnt, key = 0xFFFFFFFFu;
    double t_first = 0.0;
    if (kSmem) {
        __shared__ double s_od[6][kThreads];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s_od[a][threadIdx.x] = O[3 * r + a];
            s_od[3 + a][threadIdx.x] = D[3 * r + a];
        }
        const StridedVec o{&s_od[0][threadIdx.x], kThreads}, d{&s_od[3][threadIdx.x], kThreads};
        cnt = march_dev(g, o, d, step, S, [&](uint32_t k, double t) {
            tr[k] = t;
            if (k == 0) t_first = t;
        });
        if (pkeys) key = first_sample_key(g, o, d, cnt, t_first);
    } else {
        const double o[3] = {O[3 * r], O[3 * r + 1], O[3 * r + 2]};
        const double d[3] = {D[3 * r], D[3 * r + 1], D[3 * r + 2]};
        cnt = march_dev(g, o, d, step, S, [&](uint32_t k, double t) {
            tr[k] = t;
            if (k == 0) t_first = t;
        });
        if (pkeys) key = first_sample_key(g, o, d, cnt, t_first);
    }
    counts[r] = cnt;
    if (pkeys) {  // the post-march sort key (k_ray_keys mode 0) without re-reading the t row
        pkeys[r] = key;
        pids[r] = static_cast<uint32_t>(r);
    }
    if (delta) {
        double* dr = delta + r * S;
        for (uint32_t k = 0; k < cnt; ++k)
            dr[k] = (k + 1 < cnt) ? __dsub_rn(tr[k + 1], tr[k]) : step;  // grid.cpp:352
    }
}

// ---------------------------------------------------------------------------
// Per-sample gather + interpolation (fp32 payload math, fp64 cell decision).
// Corner c of the cell at base voxel v lies in block (v + bits(c)) >> 3; only axes with
// local coordinate 7 cross a face (smask), and those corners take their block entry from
// the per-block neighbour table -- no extra hash / dense-index lookups.
// ---------------------------------------------------------------------------
struct SampleVal {
    uint32_t gidx[8];
    float fx, fy, fz;
    float s, gx, gy, gz, r, gc, b;
    uint32_t smask;
    uint32_t e0;  // block entry of the base voxel (kInvalid: invalid sample)
};

__device__ __forceinline__ void zero_sample(SampleVal& v) {
    v.s = v.gx = v.gy = v.gz = v.r = v.gc = v.b = 0.f;
    v.fx = v.fy = v.fz = 0.f;
    v.smask = 0;
    v.e0 = kInvalid;
}

// fp64 cell decision: x = o + t d, g = x * (1/h), base = floor(g) (grid.cpp:116-121).
__device__ __forceinline__ void cell_geom(const GridView& g, const double o[3], const double d[3],
                                          double t, int base[3], SampleVal& v) {
    float fr[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = __dadd_rn(o[a], __dmul_rn(t, d[a]));
        const double gg = __dmul_rn(x, g.inv_h);
        const double fl = floor(gg);
        base[a] = static_cast<int>(fl);
        fr[a] = static_cast<float>(__dsub_rn(gg, fl));
    }
    v.fx = fr[0], v.fy = fr[1], v.fz = fr[2];
    const uint32_t lx = base[0] & 7, ly = base[1] & 7, lz = base[2] & 7;
    v.smask = (lx == 7 ? 1u : 0u) | (ly == 7 ? 2u : 0u) | (lz == 7 ? 4u : 0u);
}

// Corner c of the cell lies in block (base + bits(c)) >> 3; only axes with local
// coordinate 7 cross a face (smask), and those corners take their block entry from the
// per-block neighbour table.  kCheck: verify presence + validity (weight > 0).
template <bool kCheck>
__device__ __forceinline__ bool corner_addrs(const GridView& g, const int base[3], uint32_t e0,
                                             SampleVal& v) {
    const uint32_t lx = base[0] & 7, ly = base[1] & 7, lz = base[2] & 7;
    bool ok = e0 != kInvalid;
    const uint32_t blk0 = e0 & ~kFullBit;
    const uint32_t X[2] = {lx, (lx + 1) & 7}, Y[2] = {ly * 8, ((ly + 1) & 7) * 8},
                   Z[2] = {lz * 64, ((lz + 1) & 7) * 64};
    uint32_t full = e0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t k = static_cast<uint32_t>(c) & v.smask;
        uint32_t ec = e0;
        if (k && ok) ec = __ldg(g.nbr + static_cast<size_t>(blk0) * 8 + k);
        if (kCheck) ok = ok && ec != kInvalid;
        full &= ec;
        v.gidx[c] = (ec & ~kFullBit) * kVox + (X[c & 1] + Y[(c >> 1) & 1] + Z[c >> 2]);
    }
    if (kCheck && ok && !(full & kFullBit)) {  // some corner block is partially observed
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t gi = v.gidx[c];
            ok = ok && ((__ldg(g.vmask + (gi >> 5)) >> (gi & 31)) & 1u);
        }
    }
    return ok;
}

// Full gather + trilinear interpolation of sdf, grad(sdf) and rgb (fp32 payload math).
// kDiag (diagnostic builds of k_forward only; results are wrong): 1 = no payload loads,
// 2 = no block lookup (base block assumed to be block 0 and fully valid)
template <int kDiag = 0>
__device__ __forceinline__ bool eval_sample(const GridView& g, const double o[3], const double d[3],
                                            double t, SampleVal& v) {
    int base[3];
    cell_geom(g, o, d, t, base, v);
    const uint32_t e0 = kDiag == 2 ? kFullBit : lookup_block(g, base[0] >> 3, base[1] >> 3, base[2] >> 3);
    const bool ok = corner_addrs<true>(g, base, e0, v);
    if (!ok) {
        v.s = v.gx = v.gy = v.gz = v.r = v.gc = v.b = 0.f;
        v.e0 = kInvalid;
        return false;
    }
    v.e0 = e0;
    float4 p[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (kDiag == 1) {
            const float q = static_cast<float>(v.gidx[c] & 1023) * 1e-4f;
            p[c] = make_float4(q, q, q, q);
        } else {
            p[c] = __ldg(g.pay + v.gidx[c]);
        }
    }
    const float x1 = v.fx, x0 = 1.f - x1, y1 = v.fy, y0 = 1.f - y1, z1 = v.fz, z0 = 1.f - z1;
    const float w[8] = {x0 * y0 * z0, x1 * y0 * z0, x0 * y1 * z0, x1 * y1 * z0,
                        x0 * y0 * z1, x1 * y0 * z1, x0 * y1 * z1, x1 * y1 * z1};
    float s = 0.f, r = 0.f, gc = 0.f, b = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        s = fmaf(w[c], p[c].x, s);
        r = fmaf(w[c], p[c].y, r);
        gc = fmaf(w[c], p[c].z, gc);
        b = fmaf(w[c], p[c].w, b);
    }
    const float ih = static_cast<float>(g.inv_h);
    v.s = s, v.r = r, v.gc = gc, v.b = b;
    v.gx = ih * ((y0 * z0) * (p[1].x - p[0].x) + (y1 * z0) * (p[3].x - p[2].x) +
                 (y0 * z1) * (p[5].x - p[4].x) + (y1 * z1) * (p[7].x - p[6].x));
    v.gy = ih * ((x0 * z0) * (p[2].x - p[0].x) + (x1 * z0) * (p[3].x - p[1].x) +
                 (x0 * z1) * (p[6].x - p[4].x) + (x1 * z1) * (p[7].x - p[5].x));
    v.gz = ih * ((x0 * y0) * (p[4].x - p[0].x) + (x1 * y0) * (p[5].x - p[1].x) +
                 (x0 * y1) * (p[6].x - p[2].x) + (x1 * y1) * (p[7].x - p[3].x));
    return true;
}

// A lane slot past the ray's sample count: well-defined zeros (accumulated with w = 0).
template <int kDiag = 0>
__device__ __forceinline__ bool eval_slot(const GridView& g, const double o[3], const double d[3],
                                          bool in, double t, SampleVal& v) {
    if (in) return eval_sample<kDiag>(g, o, d, t, v);
    zero_sample(v);
    return false;
}

// Per-sample record the forward leaves for the backward (32 B, two float4):
//   {sdf, r, g, b}, {d sdf/dx, d sdf/dy, d sdf/dz, bits(block entry of the base voxel)}.
// The backward re-derives the cell geometry from t (fp64, identical decision) and the
// corner addresses from the entry + neighbour table: no dense-index lookup, no payload.
__device__ __forceinline__ void store_record(float4* rec, const SampleVal& v) {
    rec[0] = make_float4(v.s, v.r, v.gc, v.b);
    rec[1] = make_float4(v.gx, v.gy, v.gz, __uint_as_float(v.e0));
}

// `rec` may point to global memory (k_backward) or shared memory (k_backward_pipe):
// generic loads only.
__device__ __forceinline__ bool eval_from_record(const GridView& g, const double o[3],
                                                 const double d[3], bool in, double t,
                                                 const float4* rec, SampleVal& v) {
    if (!in) {
        zero_sample(v);
        return false;
    }
    const float4 a = rec[0], b = rec[1];
    const uint32_t e0 = __float_as_uint(b.w);
    if (e0 == kInvalid) {
        zero_sample(v);
        return false;
    }
    int base[3];
    cell_geom(g, o, d, t, base, v);
    corner_addrs<false>(g, base, e0, v);
    v.e0 = e0;
    v.s = a.x, v.r = a.y, v.gc = a.z, v.b = a.w;
    v.gx = b.x, v.gy = b.y, v.gz = b.z;
    return true;
}

// Laplace density and its derivative.
__device__ __forceinline__ float density(float s, float ib) {
    return s > 0.f ? ib * (0.5f * expf(-s * ib)) : ib * (1.f - 0.5f * expf(s * ib));
}
__device__ __forceinline__ float density_ds(float s, float sigma, float ib) {
    return s > 0.f ? -sigma * ib : -(ib - sigma) * ib;
}

__device__ __forceinline__ float warp_incl_scan(float v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float n = __shfl_up_sync(kFull, v, off);
        if (lane >= off) v += n;
    }
    return v;
}
__device__ __forceinline__ float warp_incl_suffix(float v, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float n = __shfl_down_sync(kFull, v, off);
        if (lane + off < 32) v += n;
    }
    return v;
}

// Reduce 8 per-lane values over the warp with 9 shuffles (reduce-scatter then butterfly):
// afterwards lane 4 v (v = 0..7) holds the warp total of value v; returns this lane's.
__device__ __forceinline__ float warp_sum8(const float a[8], int lane) {
    const bool hi4 = lane & 16, hi3 = lane & 8, hi2 = lane & 4;
    float b[4], c[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = hi4 ? a[k] : a[k + 4];
        b[k] = (hi4 ? a[k + 4] : a[k]) + __shfl_xor_sync(kFull, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = hi3 ? b[k] : b[k + 2];
        c[k] = (hi3 ? b[k + 2] : b[k]) + __shfl_xor_sync(kFull, send, 8);
    }
    float v = (hi2 ? c[1] : c[0]) + __shfl_xor_sync(kFull, hi2 ? c[0] : c[1], 4);
    v += __shfl_xor_sync(kFull, v, 2);
    v += __shfl_xor_sync(kFull, v, 1);
    return v;
}

// Ray outputs from warp_sum8's layout: lane 4v writes value v (C.rgb, D, N.xyz, W).
__device__ __forceinline__ void write_ray_outputs(float v, int lane, uint64_t r, float* rgb, float* depth,
                                                  float* normal, float* wsum) {
    if (lane & 3) return;
    const int k = lane >> 2;
    if (k < 3) {
        if (rgb) rgb[3 * r + k] = v;
    } else if (k == 3) {
        if (depth) depth[r] = v;
    } else if (k < 7) {
        if (normal) normal[3 * r + (k - 4)] = v;
    } else {
        if (wsum) wsum[r] = v;
    }
}

// Sample k's t and delta (delta_k = t_{k+1} - t_k, last = step: grid.cpp:352) for the
// lane's two consecutive samples k0 = base + 2 lane, k1 = k0 + 1.
struct PairT {
    double t0, t1;
    float d0, d1;
    bool in0, in1;
};
__device__ __forceinline__ PairT load_pair(const double* tr, uint32_t cnt, uint32_t base, int lane,
                                           double step) {
    PairT p;
    const uint32_t k0 = base + 2 * lane, k1 = k0 + 1;
    p.in0 = k0 < cnt;
    p.in1 = k1 < cnt;
    p.t0 = p.in0 ? tr[k0] : 0.0;
    p.t1 = p.in1 ? tr[k1] : 0.0;
    double tn = __shfl_down_sync(kFull, p.t0, 1);
    if (lane == 31 && k1 + 1 < cnt) tn = tr[k1 + 1];
    p.d0 = p.in1 ? static_cast<float>(__dsub_rn(p.t1, p.t0)) : static_cast<float>(step);
    p.d1 = (k1 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn, p.t1)) : static_cast<float>(step);
    return p;
}

// ---------------------------------------------------------------------------
// Ray ordering for L2 locality: key = Morton code of the block holding the ray's first
// sample (10 bits per axis, relative to the AABB); rays without samples sort last.
// The forward / backward warps then visit rays in key order, so concurrently resident
// warps touch the same blocks and the same gradient lines.  Outputs stay in caller order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3FF;
    v = (v | (v << 16)) & 0x030000FF;
    v = (v | (v << 8)) & 0x0300F00F;
    v = (v | (v << 4)) & 0x030C30C3;
    v = (v | (v << 2)) & 0x09249249;
    return v;
}

__global__ void __launch_bounds__(256) k_ray_keys(GridView g, const double* __restrict__ O,
                                                  const double* __restrict__ D, uint64_t n,
                                                  const uint32_t* __restrict__ counts,
                                                  const double* __restrict__ T, uint32_t S,
                                                  uint32_t* keys, uint32_t* ids, int mode) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    uint32_t key = 0xFFFFFFFFu;
    if (counts[r]) {
        // mode 0: block of the first sample; 1: block of the middle sample; 2: first sample at
        // half-block resolution
        const double t = T[r * S + (mode == 1 ? counts[r] / 2 : 0)];
        const double cell = mode == 2 ? 0.5 * g.L : g.L;
        const int scale = mode == 2 ? 2 : 1;
        uint32_t b[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double x = O[3 * r + a] + t * D[3 * r + a];
            int32_t v = static_cast<int32_t>(floor(x / cell)) - scale * g.lo[a];
            v = v < 0 ? 0 : (v > 1023 ? 1023 : v);
            b[a] = static_cast<uint32_t>(v);
        }
        key = spread3(b[0]) | (spread3(b[1]) << 1) | (spread3(b[2]) << 2);
    }
    keys[r] = key;
    ids[r] = static_cast<uint32_t>(r);
}

// Pre-march ordering: 8-bit hash of the origin (1 mm cells) above a 16-bit Morton code of
// the octahedral direction, so rays from one camera with nearby pixels march together.
__global__ void __launch_bounds__(256) k_ray_keys_dir(const double* __restrict__ O,
                                                      const double* __restrict__ D, uint64_t n,
                                                      uint32_t* keys, uint32_t* ids) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double dx = D[3 * r], dy = D[3 * r + 1], dz = D[3 * r + 2];
    const double l1 = fabs(dx) + fabs(dy) + fabs(dz);
    double u = dx / l1, v = dy / l1;
    if (dz < 0.0) {
        const double uu = (1.0 - fabs(v)) * (u >= 0.0 ? 1.0 : -1.0);
        const double vv = (1.0 - fabs(u)) * (v >= 0.0 ? 1.0 : -1.0);
        u = uu, v = vv;
    }
    // 8-bit origin hash above a 16-bit Morton code of the direction (256 x 256 octahedral
    // bins): 24-bit keys, three radix passes
    const uint32_t qu = min(255u, static_cast<uint32_t>((u * 0.5 + 0.5) * 256.0));
    const uint32_t qv = min(255u, static_cast<uint32_t>((v * 0.5 + 0.5) * 256.0));
    uint32_t m = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) m |= (((qu >> b) & 1u) << (2 * b)) | (((qv >> b) & 1u) << (2 * b + 1));
    unsigned long long h = 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int a = 0; a < 3; ++a)
        h = mix64(h ^ static_cast<unsigned long long>(llrint(O[3 * r + a] * 1000.0)));
    keys[r] = (static_cast<uint32_t>(h >> 56) << 16) | m;
    ids[r] = static_cast<uint32_t>(r);
}

// ---------------------------------------------------------------------------
// K5: forward.  One warp per ray, lane l owns samples 2l and 2l+1 of each 64-sample
// chunk; exclusive prefix of tau by a warp scan gives T_k = exp(-sum_{j<k} tau_j).
// ---------------------------------------------------------------------------
template <int kThreads, int kMinBlocks, int kDiag = 0>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_forward(GridView g, const double* __restrict__ O,
                                                    const double* __restrict__ D, uint64_t n,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ counts,
                                                    const double* __restrict__ T, uint32_t S,
                                                    double step, float ib, float* rgb, float* depth,
                                                    float* normal, float* wsum,
                                                    unsigned long long* valid_counter, float4* rec) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const uint64_t r = order ? order[w] : w;
    const double o[3] = {O[3 * r], O[3 * r + 1], O[3 * r + 2]};
    const double d[3] = {D[3 * r], D[3 * r + 1], D[3 * r + 2]};
    const uint32_t cnt = counts[r];
    const double* tr = T + r * S;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // C, D, N, W
    float tau_base = 0.f;
    uint32_t nvalid = 0;
    for (uint32_t base = 0; base < cnt; base += 64) {
        const PairT p = load_pair(tr, cnt, base, lane, step);
        SampleVal v0, v1;
        const bool ok0 = eval_slot<kDiag == 3 ? 0 : kDiag>(g, o, d, p.in0, p.t0, v0);
        const bool ok1 = eval_slot<kDiag == 3 ? 0 : kDiag>(g, o, d, p.in1, p.t1, v1);
        if (rec && kDiag != 3) {  // per-sample record for the backward (coalesced: 64 B per lane)
            float4* rr = rec + (r * S + base + 2 * lane) * 2;
            if (p.in0) store_record(rr, v0);
            if (p.in1) store_record(rr + 2, v1);
        }
        const float tau0 = ok0 ? density(v0.s, ib) * p.d0 : 0.f;
        const float tau1 = ok1 ? density(v1.s, ib) * p.d1 : 0.f;
        const float incl = warp_incl_scan(tau0 + tau1, lane);
        float excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = 0.f;
        // T0 = exp(-P0); w0 = T0 (1 - e^-tau0); T1 = T0 e^-tau0 = T0 - w0 (one exp per pair)
        const float T0 = expf(-(tau_base + excl));
        const float w0 = -T0 * expm1f(-tau0);
        const float T1 = T0 - w0;
        const float w1 = ok1 ? -T1 * expm1f(-tau1) : 0.f;
        acc[0] += w0 * v0.r + w1 * v1.r;
        acc[1] += w0 * v0.gc + w1 * v1.gc;
        acc[2] += w0 * v0.b + w1 * v1.b;
        acc[3] += w0 * static_cast<float>(p.t0) + w1 * static_cast<float>(p.t1);
        acc[4] += w0 * v0.gx + w1 * v1.gx;
        acc[5] += w0 * v0.gy + w1 * v1.gy;
        acc[6] += w0 * v0.gz + w1 * v1.gz;
        acc[7] += w0 + w1;
        if (valid_counter) nvalid += __popc(__ballot_sync(kFull, ok0)) + __popc(__ballot_sync(kFull, ok1));
        tau_base += __shfl_sync(kFull, incl, 31);
    }
    write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
    if (lane == 0 && valid_counter && nvalid)
        atomicAdd(valid_counter, static_cast<unsigned long long>(nvalid));
}

// K5 with the split lane layout: lane l owns samples base + l and base + 32 + l, so the
// 32 lanes of one gather instruction walk 32 consecutive samples (neighbouring lanes share
// cells and cache lines).
template <int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_forward_split(GridView g, const double* __restrict__ O,
                                                    const double* __restrict__ D, uint64_t n,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ counts,
                                                    const double* __restrict__ T, uint32_t S,
                                                    double step, float ib, float* rgb, float* depth,
                                                    float* normal, float* wsum,
                                                    unsigned long long* valid_counter, float4* rec) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const uint64_t r = order ? order[w] : w;
    const double o[3] = {O[3 * r], O[3 * r + 1], O[3 * r + 2]};
    const double d[3] = {D[3 * r], D[3 * r + 1], D[3 * r + 2]};
    const uint32_t cnt = counts[r];
    const double* tr = T + r * S;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // C, D, N, W
    float tau_base = 0.f;
    uint32_t nvalid = 0;
    for (uint32_t base = 0; base < cnt; base += 64) {
        const uint32_t k0 = base + lane, k1 = base + 32 + lane;
        const bool in0 = k0 < cnt, in1 = k1 < cnt;
        const double t0 = in0 ? tr[k0] : 0.0, t1 = in1 ? tr[k1] : 0.0;
        double tn0 = __shfl_down_sync(kFull, t0, 1);
        const double t1_l0 = __shfl_sync(kFull, t1, 0);
        double tn1 = __shfl_down_sync(kFull, t1, 1);
        if (lane == 31) {
            tn0 = t1_l0;
            if (k1 + 1 < cnt) tn1 = tr[k1 + 1];
        }
        const float d0 = (k0 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn0, t0)) : static_cast<float>(step);
        const float d1 = (k1 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn1, t1)) : static_cast<float>(step);
        SampleVal v0, v1;
        const bool ok0 = eval_slot(g, o, d, in0, t0, v0);
        const bool ok1 = eval_slot(g, o, d, in1, t1, v1);
        if (rec) {
            if (in0) store_record(rec + (r * S + k0) * 2, v0);
            if (in1) store_record(rec + (r * S + k1) * 2, v1);
        }
        const float tau0 = ok0 ? density(v0.s, ib) * d0 : 0.f;
        const float tau1 = ok1 ? density(v1.s, ib) * d1 : 0.f;
        const float inc0 = warp_incl_scan(tau0, lane);
        const float inc1 = warp_incl_scan(tau1, lane);
        const float tot0 = __shfl_sync(kFull, inc0, 31);
        const float w0 = -expf(-(tau_base + inc0 - tau0)) * expm1f(-tau0);
        const float w1 = -expf(-(tau_base + tot0 + inc1 - tau1)) * expm1f(-tau1);
        acc[0] += w0 * v0.r + w1 * v1.r;
        acc[1] += w0 * v0.gc + w1 * v1.gc;
        acc[2] += w0 * v0.b + w1 * v1.b;
        acc[3] += w0 * static_cast<float>(t0) + w1 * static_cast<float>(t1);
        acc[4] += w0 * v0.gx + w1 * v1.gx;
        acc[5] += w0 * v0.gy + w1 * v1.gy;
        acc[6] += w0 * v0.gz + w1 * v1.gz;
        acc[7] += w0 + w1;
        if (valid_counter) nvalid += __popc(__ballot_sync(kFull, ok0)) + __popc(__ballot_sync(kFull, ok1));
        tau_base += tot0 + __shfl_sync(kFull, inc1, 31);
    }
    write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
    if (lane == 0 && valid_counter && nvalid)
        atomicAdd(valid_counter, static_cast<unsigned long long>(nvalid));
}

// K5, sequential halves: one sample per lane per pass (samples base + 32 h + l), so only
// one sample's state is live -- fewer registers, more resident warps.
template <int kThreads, int kMinBlocks, bool kOdSmem = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_forward_seq(GridView g, const double* __restrict__ O,
                                                    const double* __restrict__ D, uint64_t n,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ counts,
                                                    const double* __restrict__ T, uint32_t S,
                                                    double step, float ib, float* rgb, float* depth,
                                                    float* normal, float* wsum,
                                                    unsigned long long* valid_counter, float4* rec) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const uint64_t r = order ? order[w] : w;
    // the ray's origin / direction: registers, or (kOdSmem) a per-warp shared slot read at
    // each use, which frees 12 registers
    __shared__ double s_od[kThreads / 32][6];
    double o_r[3], d_r[3];
    const double* o = o_r;
    const double* d = d_r;
    if (kOdSmem) {
        const int wib = threadIdx.x >> 5;
        if (lane < 6) s_od[wib][lane] = lane < 3 ? O[3 * r + lane] : D[3 * r + lane - 3];
        __syncwarp();
        o = s_od[wib];
        d = s_od[wib] + 3;
    } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) o_r[a] = O[3 * r + a], d_r[a] = D[3 * r + a];
    }
    const uint32_t cnt = counts[r];
    const double* tr = T + r * S;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // C, D, N, W
    float tau_base = 0.f;
    uint32_t nvalid = 0;
    for (uint32_t base = 0; base < cnt; base += 32) {
        const uint32_t k0 = base + lane;
        const bool in0 = k0 < cnt;
        const double t0 = in0 ? tr[k0] : 0.0;
        double tn0 = __shfl_down_sync(kFull, t0, 1);
        if (lane == 31 && k0 + 1 < cnt) tn0 = tr[k0 + 1];
        const float d0 = (k0 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn0, t0)) : static_cast<float>(step);
        SampleVal v0;
        const bool ok0 = eval_slot(g, o, d, in0, t0, v0);
        if (rec && in0) store_record(rec + (r * S + k0) * 2, v0);
        const float tau0 = ok0 ? density(v0.s, ib) * d0 : 0.f;
        const float inc0 = warp_incl_scan(tau0, lane);
        const float w0 = -expf(-(tau_base + inc0 - tau0)) * expm1f(-tau0);
        acc[0] += w0 * v0.r;
        acc[1] += w0 * v0.gc;
        acc[2] += w0 * v0.b;
        acc[3] += w0 * static_cast<float>(t0);
        acc[4] += w0 * v0.gx;
        acc[5] += w0 * v0.gy;
        acc[6] += w0 * v0.gz;
        acc[7] += w0;
        if (valid_counter) nvalid += __popc(__ballot_sync(kFull, ok0));
        tau_base += __shfl_sync(kFull, inc0, 31);
    }
    write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
    if (lane == 0 && valid_counter && nvalid)
        atomicAdd(valid_counter, static_cast<unsigned long long>(nvalid));
}

// K5, sequential halves over K consecutive (sorted) rays per warp with the per-ray set-up
// taken off the critical path: one load of the K ray ids, then the K origins / directions
// (to shared memory) and sample counts in one parallel round trip, and every t value one
// pass ahead (the next pass of this ray, or the first pass of the next ray) -- the chain
// order -> o/d -> count -> t -> lookup -> payload of k_forward_seq shrinks to
// lookup -> payload per pass.  Same arithmetic per sample as k_forward_seq.
template <int kThreads, int kMinBlocks, int K, bool kHdr>
__global__ void __launch_bounds__(kThreads, kMinBlocks) k_forward_multi(GridView g, const double* __restrict__ O,
                                                    const double* __restrict__ D, uint64_t n,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ counts,
                                                    const double* __restrict__ T, uint32_t S,
                                                    double step, float ib, float* rgb, float* depth,
                                                    float* normal, float* wsum,
                                                    unsigned long long* valid_counter, float4* rec,
                                                    const uint2* __restrict__ hdr) {
    static_assert(6 * K <= 32, "one lane per origin / direction component");
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t w0 = ((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * K;
    if (w0 >= n) return;
    const int nr = n - w0 < static_cast<uint64_t>(K) ? static_cast<int>(n - w0) : K;
    __shared__ double s_od[kThreads / 32][K][6];
    uint32_t my_r = 0, my_cnt = 0;  // lane j < nr: ray j's id and sample count
    if (lane < nr) {
        if (kHdr) {  // {id, count} in sorted order: one load level less
            const uint2 h = hdr[w0 + lane];
            my_r = h.x, my_cnt = h.y;
        } else {
            my_r = order ? order[w0 + lane] : static_cast<uint32_t>(w0 + lane);
        }
    }
    {
        const int j = lane / 6, a = lane - 6 * (lane / 6);
        const uint32_t rj = __shfl_sync(kFull, my_r, j < K ? j : 0);
        if (j < nr) s_od[wib][j][a] = a < 3 ? O[3ull * rj + a] : D[3ull * rj + a - 3];
        if (lane < nr && !kHdr) my_cnt = counts[my_r];
    }
    __syncwarp();
    uint32_t nvalid = 0;
    // t of the lane's sample in the upcoming pass
    uint32_t r = __shfl_sync(kFull, my_r, 0), cnt = __shfl_sync(kFull, my_cnt, 0);
    double t_cur = static_cast<uint32_t>(lane) < cnt ? T[static_cast<uint64_t>(r) * S + lane] : 0.0;
    for (int j = 0; j < nr; ++j) {
        const double* o = s_od[wib][j];
        const double* d = o + 3;
        const double* tr = T + static_cast<uint64_t>(r) * S;
        const uint32_t r1 = __shfl_sync(kFull, my_r, j + 1 < K ? j + 1 : 0);
        const uint32_t cnt1 = j + 1 < nr ? __shfl_sync(kFull, my_cnt, j + 1 < K ? j + 1 : 0) : 0u;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // C, D, N, W
        float tau_base = 0.f;
        for (uint32_t base = 0; base < cnt; base += 32) {
            const uint32_t k0 = base + lane;
            const bool in0 = k0 < cnt;
            const double t0 = in0 ? t_cur : 0.0;
            // one pass ahead: this ray's next pass, else the next ray's first pass
            t_cur = base + 32 < cnt ? (k0 + 32 < cnt ? tr[k0 + 32] : 0.0)
                                    : (static_cast<uint32_t>(lane) < cnt1 ? T[static_cast<uint64_t>(r1) * S + lane] : 0.0);
            double tn0 = __shfl_down_sync(kFull, t0, 1);
            const double tl0 = __shfl_sync(kFull, t_cur, 0);
            if (lane == 31) tn0 = tl0;
            const float d0 = (k0 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn0, t0)) : static_cast<float>(step);
            SampleVal v0;
            const bool ok0 = eval_slot(g, o, d, in0, t0, v0);
            if (rec && in0) store_record(rec + (static_cast<uint64_t>(r) * S + k0) * 2, v0);
            const float tau0 = ok0 ? density(v0.s, ib) * d0 : 0.f;
            const float inc0 = warp_incl_scan(tau0, lane);
            const float w = -expf(-(tau_base + inc0 - tau0)) * expm1f(-tau0);
            acc[0] += w * v0.r;
            acc[1] += w * v0.gc;
            acc[2] += w * v0.b;
            acc[3] += w * static_cast<float>(t0);
            acc[4] += w * v0.gx;
            acc[5] += w * v0.gy;
            acc[6] += w * v0.gz;
            acc[7] += w;
            if (valid_counter) nvalid += __popc(__ballot_sync(kFull, ok0));
            tau_base += __shfl_sync(kFull, inc0, 31);
        }
        if (cnt == 0)  // no pass ran: the next ray's first pass is still to be fetched
            t_cur = static_cast<uint32_t>(lane) < cnt1 ? T[static_cast<uint64_t>(r1) * S + lane] : 0.0;
        write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
        r = r1;
        cnt = cnt1;
    }
    if (lane == 0 && valid_counter && nvalid)
        atomicAdd(valid_counter, static_cast<unsigned long long>(nvalid));
}

// Gradient of corner c of one sample: (g_sdf, g_r, g_g, g_b) with
//   g_sdf = w_c dL/ds + dw_c . (w_k dN),  g_rgb = w_c w_k dC.
struct CornerCoef {
    float x0, x1, y0, y1, z0, z1, ds, wn0, wn1, wn2, wc0, wc1, wc2;
};
__device__ __forceinline__ CornerCoef make_coef(const SampleVal& v, float ds, float wk,
                                                const float dC[3], const float dN[3], float ih) {
    CornerCoef k;
    k.x1 = v.fx, k.x0 = 1.f - v.fx, k.y1 = v.fy, k.y0 = 1.f - v.fy, k.z1 = v.fz, k.z0 = 1.f - v.fz;
    k.ds = ds;
    k.wn0 = wk * dN[0] * ih, k.wn1 = wk * dN[1] * ih, k.wn2 = wk * dN[2] * ih;
    k.wc0 = wk * dC[0], k.wc1 = wk * dC[1], k.wc2 = wk * dC[2];
    return k;
}
template <int c>
__device__ __forceinline__ float4 corner_grad(const CornerCoef& k) {
    const float wx = (c & 1) ? k.x1 : k.x0, wy = (c & 2) ? k.y1 : k.y0, wz = (c & 4) ? k.z1 : k.z0;
    const float sx = (c & 1) ? 1.f : -1.f, sy = (c & 2) ? 1.f : -1.f, sz = (c & 4) ? 1.f : -1.f;
    const float w = wx * wy * wz;
    const float gs = w * k.ds + sx * (wy * wz) * k.wn0 + sy * (wx * wz) * k.wn1 + sz * (wx * wy) * k.wn2;
    return make_float4(gs, w * k.wc0, w * k.wc1, w * k.wc2);
}

__device__ __forceinline__ void mark_block(const GridView& g, uint32_t blk) {
    if (!g.active[blk]) g.active[blk] = 1;
}
__device__ __forceinline__ void mark_blocks(const GridView& g, const SampleVal& v) {
    mark_block(g, v.gidx[0] >> 9);
    if (v.smask) {  // corners in neighbour blocks: every other corner slot may differ
#pragma unroll
        for (int c = 1; c < 8; ++c)
            if (c & v.smask) mark_block(g, v.gidx[c] >> 9);
    }
}

template <int c, int kMode = 0>
__device__ __forceinline__ void scatter_corner(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                               const CornerCoef& k0, const CornerCoef& k1, bool ok0,
                                               bool ok1, bool same) {
    if (kMode == 1) {  // diagnostic: same arithmetic, plain stores instead of atomics
        if (ok0) grad[v0.gidx[c]] = corner_grad<c>(k0);
        if (ok1) grad[v1.gidx[c]] = corner_grad<c>(k1);
        return;
    }
    if (kMode == 2) {  // diagnostic: arithmetic only, no memory traffic
        const float4 a = corner_grad<c>(k0), b = corner_grad<c>(k1);
        if (a.x == 1234.5f && b.y == 1234.5f) grad[0] = a;
        return;
    }
    if (same) {
        const float4 a = corner_grad<c>(k0), b = corner_grad<c>(k1);
        atomicAdd(grad + v0.gidx[c], make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w));
    } else {
        if (ok0) atomicAdd(grad + v0.gidx[c], corner_grad<c>(k0));
        if (ok1) atomicAdd(grad + v1.gidx[c], corner_grad<c>(k1));
    }
}

// Warp-aggregated scatter of one lane's sample pair.  Along a ray consecutive samples share a
// cell ~40 % of the time, so beyond merging a lane's own two samples, the first cell run of
// lane l is handed to lane l-1 when it continues lane l-1's last run (one shuffle-down per
// component); lane l-1 folds it into its last run's atomics.  Every contribution is still
// issued exactly once: a lane that handed its only run away issues just what it received.
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 shfl_down4(float4 v) {
    return make_float4(__shfl_down_sync(kFull, v.x, 1), __shfl_down_sync(kFull, v.y, 1),
                       __shfl_down_sync(kFull, v.z, 1), __shfl_down_sync(kFull, v.w, 1));
}
template <int c>
__device__ __forceinline__ void scatter_corner_agg(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                                   const CornerCoef& k0, const CornerCoef& k1, bool ok0, bool ok1,
                                                   bool two, bool give, bool recv) {
    const float4 a0 = ok0 ? corner_grad<c>(k0) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 a1 = ok1 ? corner_grad<c>(k1) : make_float4(0.f, 0.f, 0.f, 0.f);
    // first run F (address fa) and last run L (address v1.gidx[c]); one run when !two
    const float4 F = two ? a0 : f4add(a0, a1);
    const float4 in = shfl_down4(F);  // lane l+1's first run (used only when recv)
    const uint32_t fa = ok0 ? v0.gidx[c] : v1.gidx[c];
    if (two) {
        if (!give) atomicAdd(grad + fa, a0);
        atomicAdd(grad + v1.gidx[c], recv ? f4add(a1, in) : a1);
    } else if (ok0 || ok1) {
        if (give) {
            if (recv) atomicAdd(grad + fa, in);
        } else {
            atomicAdd(grad + fa, recv ? f4add(F, in) : F);
        }
    }
}
__device__ __forceinline__ void scatter_pair_agg(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                                 const CornerCoef& k0, const CornerCoef& k1, bool ok0, bool ok1,
                                                 int lane) {
    const uint32_t first = ok0 ? v0.gidx[0] : (ok1 ? v1.gidx[0] : kInvalid);
    const uint32_t last = ok1 ? v1.gidx[0] : first;
    const bool two = ok0 && ok1 && v0.gidx[0] != v1.gidx[0];
    const uint32_t prev_last = __shfl_up_sync(kFull, last, 1);
    const bool give = lane > 0 && first != kInvalid && first == prev_last;
    const bool recv = __shfl_down_sync(kFull, give ? 1u : 0u, 1) != 0u && lane < 31;
    scatter_corner_agg<0>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<1>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<2>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<3>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<4>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<5>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<6>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
    scatter_corner_agg<7>(grad, v0, v1, k0, k1, ok0, ok1, two, give, recv);
}

// ---------------------------------------------------------------------------
// K6: backward.  Chunks of 64 samples are visited back to front; within a chunk the
// suffix S_k = sum_{m>k} w_m v_m comes from a warp suffix scan (no cancellation-prone
// "total minus prefix").  dL/dtau_k = T_{k+1} v_k - S_k, dL/ds_k = delta_k sigma' dL/dtau_k.
// Corner gradients are produced and issued one corner at a time (red.global.add.v4.f32);
// a lane whose two samples share a cell sums them first.
// ---------------------------------------------------------------------------
template <int kMinBlocks, int kMode, bool kRec>
__global__ void __launch_bounds__(256, kMinBlocks) k_backward(GridView g, const double* __restrict__ O,
                                                     const double* __restrict__ D, uint64_t n,
                                                     const uint32_t* __restrict__ order,
                                                     const uint32_t* __restrict__ counts,
                                                     const double* __restrict__ T, uint32_t S,
                                                     double step, float ib,
                                                     const float* __restrict__ d_rgb,
                                                     const float* __restrict__ d_depth,
                                                     const float* __restrict__ d_normal,
                                                     const float4* __restrict__ rec) {
    const int lane = threadIdx.x & 31;
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const uint64_t r = order ? order[w] : w;
    const uint32_t cnt = counts[r];
    if (cnt == 0) return;
    const double o[3] = {O[3 * r], O[3 * r + 1], O[3 * r + 2]};
    const double d[3] = {D[3 * r], D[3 * r + 1], D[3 * r + 2]};
    const double* tr = T + r * S;
    const float dC[3] = {d_rgb[3 * r], d_rgb[3 * r + 1], d_rgb[3 * r + 2]};
    const float dD = d_depth[r];
    const float dN[3] = {d_normal[3 * r], d_normal[3 * r + 1], d_normal[3 * r + 2]};
    const float ih = static_cast<float>(g.inv_h);
    const uint32_t nch = (cnt + 63) / 64;

    // Exclusive tau prefix of each chunk (lane c holds chunk c's); only for long rays.
    float my_prefix = 0.f;
    if (nch > 1) {
        float run = 0.f;
        for (uint32_t ch = 0; ch < nch; ++ch) {
            const PairT p = load_pair(tr, cnt, ch * 64, lane, step);
            SampleVal v0, v1;
            const float4* rr = rec + (r * S + ch * 64 + 2 * lane) * 2;
            const bool ok0 = kRec ? eval_from_record(g, o, d, p.in0, p.t0, rr, v0) : eval_slot(g, o, d, p.in0, p.t0, v0);
            const bool ok1 = kRec ? eval_from_record(g, o, d, p.in1, p.t1, rr + 2, v1) : eval_slot(g, o, d, p.in1, p.t1, v1);
            const float tau = (ok0 ? density(v0.s, ib) * p.d0 : 0.f) +
                              (ok1 ? density(v1.s, ib) * p.d1 : 0.f);
            const float incl = warp_incl_scan(tau, lane);
            if (lane == static_cast<int>(ch)) my_prefix = run;
            run += __shfl_sync(kFull, incl, 31);
        }
    }

    float S_after = 0.f;
    for (int ch = static_cast<int>(nch) - 1; ch >= 0; --ch) {
        const float tau_base = __shfl_sync(kFull, my_prefix, ch & 31);
        const PairT p = load_pair(tr, cnt, static_cast<uint32_t>(ch) * 64, lane, step);
        SampleVal v0, v1;
        const float4* rr = rec + (r * S + static_cast<uint32_t>(ch) * 64 + 2 * lane) * 2;
        const bool ok0 = kRec ? eval_from_record(g, o, d, p.in0, p.t0, rr, v0) : eval_slot(g, o, d, p.in0, p.t0, v0);
        const bool ok1 = kRec ? eval_from_record(g, o, d, p.in1, p.t1, rr + 2, v1) : eval_slot(g, o, d, p.in1, p.t1, v1);
        const float sg0 = ok0 ? density(v0.s, ib) : 0.f, sg1 = ok1 ? density(v1.s, ib) : 0.f;
        const float tau0 = sg0 * p.d0, tau1 = sg1 * p.d1;
        const float incl = warp_incl_scan(tau0 + tau1, lane);
        float excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = 0.f;
        const float P0 = tau_base + excl, P1 = P0 + tau0;
        const float w0 = ok0 ? expf(-P0) * -expm1f(-tau0) : 0.f;
        const float w1 = ok1 ? expf(-P1) * -expm1f(-tau1) : 0.f;
        const float Tn0 = expf(-P1), Tn1 = expf(-(P1 + tau1));
        const float vv0 = ok0 ? dC[0] * v0.r + dC[1] * v0.gc + dC[2] * v0.b +
                                    dD * static_cast<float>(p.t0) + dN[0] * v0.gx + dN[1] * v0.gy +
                                    dN[2] * v0.gz
                              : 0.f;
        const float vv1 = ok1 ? dC[0] * v1.r + dC[1] * v1.gc + dC[2] * v1.b +
                                    dD * static_cast<float>(p.t1) + dN[0] * v1.gx + dN[1] * v1.gy +
                                    dN[2] * v1.gz
                              : 0.f;
        const float u0 = w0 * vv0, u1 = w1 * vv1;
        const float sinc = warp_incl_suffix(u0 + u1, lane);
        float sexc = __shfl_down_sync(kFull, sinc, 1);
        if (lane == 31) sexc = 0.f;
        const float S1 = S_after + sexc, S0 = S1 + u1;
        const CornerCoef k0 = make_coef(v0, ok0 ? p.d0 * density_ds(v0.s, sg0, ib) * (Tn0 * vv0 - S0) : 0.f,
                                        w0, dC, dN, ih);
        const CornerCoef k1 = make_coef(v1, ok1 ? p.d1 * density_ds(v1.s, sg1, ib) * (Tn1 * vv1 - S1) : 0.f,
                                        w1, dC, dN, ih);
        if (ok0) mark_blocks(g, v0);
        if (ok1) mark_blocks(g, v1);
        if (kMode == 3) {
            scatter_pair_agg(g.grad, v0, v1, k0, k1, ok0, ok1, lane);
        } else {
            const bool same = ok0 && ok1 && v0.gidx[0] == v1.gidx[0];
            scatter_corner<0, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<1, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<2, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<3, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<4, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<5, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<6, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
            scatter_corner<7, kMode>(g.grad, v0, v1, k0, k1, ok0, ok1, same);
        }
        S_after += __shfl_sync(kFull, sinc, 0);
    }
}

// ---------------------------------------------------------------------------
// K6p: pipelined backward (records required, max_samples <= 64).  Persistent warps;
// each warp owns a ring of kStages shared-memory slots and streams the t row and the
// record row of the rays it will process next with cp.async.bulk (TMA bulk copy,
// completion on an mbarrier), so the per-ray load latency overlaps the compositing
// adjoint and the atomic scatter of the current ray.
// ---------------------------------------------------------------------------
constexpr int kPipeStages = 3;
constexpr int kPipeWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// The ray's scalars (kHdr): origin / direction, upstream gradients and sample count, copied
// into the slot by 14 lanes with cp.async and completed on the slot's mbarrier.
struct PipeHdr {
    double o[3], d[3];
    float dC[3], dD, dN[3];
    uint32_t cnt;
};
struct PipeSlot {
    double t[64];
    float4 rec[128];
    PipeHdr hdr;
};
__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrive on `bar` once this thread's earlier cp.async copies have landed (no pending-count
// increment: the barrier's expected count includes these arrivals)
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int kMinBlocks, int kMode = 0, int kStages = kPipeStages, bool kHdr = false>
__global__ void __launch_bounds__(kPipeWarps * 32, kMinBlocks)
    k_backward_pipe(GridView g, const double* __restrict__ O, const double* __restrict__ D, uint64_t n,
                    const uint32_t* __restrict__ order, const uint32_t* __restrict__ counts,
                    const double* __restrict__ T, uint32_t S, double step, float ib,
                    const float* __restrict__ d_rgb, const float* __restrict__ d_depth,
                    const float* __restrict__ d_normal, const float4* __restrict__ rec,
                    uint64_t warps_total) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    PipeSlot* slots = reinterpret_cast<PipeSlot*>(smem_raw) + wib * kStages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(PipeSlot) * kStages * kPipeWarps) +
                     wib * kStages;
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kPipeWarps + wib;
    const uint32_t tbytes = S * 8, rbytes = S * 32;
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(bars + st, kHdr ? 33 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto ray_of = [&](uint64_t i) -> uint64_t { return order ? order[i] : i; };
    auto issue = [&](uint64_t r, int st) {  // lane 0: stream ray r's t + record rows
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bars + st, tbytes + rbytes);
        bulk_g2s(slots[st].t, T + r * S, tbytes, bars + st);
        bulk_g2s(slots[st].rec, rec + r * S * 2, rbytes, bars + st);
    };
    auto issue_hdr = [&](uint64_t r, int st) {  // every lane (kHdr): ray r's scalars + arrive
        PipeHdr& h = slots[st].hdr;
        if (lane < 3) cp_async_8(&h.o[lane], O + 3 * r + lane);
        else if (lane < 6) cp_async_8(&h.d[lane - 3], D + 3 * r + lane - 3);
        else if (lane < 9) cp_async_4(&h.dC[lane - 6], d_rgb + 3 * r + lane - 6);
        else if (lane == 9) cp_async_4(&h.dD, d_depth + r);
        else if (lane < 13) cp_async_4(&h.dN[lane - 10], d_normal + 3 * r + lane - 10);
        else if (lane == 13) cp_async_4(&h.cnt, counts + r);
        cp_async_arrive(bars + st);
    };
    // prologue
    for (int st = 0; st < kStages - 1; ++st) {
        const uint64_t i = w0 + st * warps_total;
        if (i < n) {
            if (kHdr) {
                const uint64_t r = ray_of(i);
                if (lane == 0) issue(r, st);
                issue_hdr(r, st);
            } else if (lane == 0) {
                issue(ray_of(i), st);
            }
        }
    }
    // kHdr: the id of the next ray to stream, loaded one iteration before it is issued
    uint64_t pf_i = w0 + (kStages - 1) * warps_total;
    uint64_t r_pf = (kHdr && pf_i < n) ? ray_of(pf_i) : 0;
    const float ih = static_cast<float>(g.inv_h);
    uint32_t phase = 0;  // bit st = parity of stage st
    int st = 0;
    for (uint64_t i = w0; i < n; i += warps_total) {
        {  // keep kStages-1 rays in flight: refill the stage released last iteration
            const uint64_t nxt = i + (kStages - 1) * warps_total;
            const int nst = (st + kStages - 1) % kStages;
            if (kHdr) {
                if (nxt < n) {
                    if (lane == 0) issue(r_pf, nst);
                    issue_hdr(r_pf, nst);
                }
                pf_i += warps_total;
                if (pf_i < n) r_pf = ray_of(pf_i);
            } else if (lane == 0 && nxt < n) {
                issue(ray_of(nxt), nst);
            }
        }
        uint32_t cnt;
        double o_r[3], d_r[3];
        float dC[3], dD, dN[3];
        const double* o = o_r;
        const double* d = d_r;
        if (!kHdr) {
            const uint64_t r = ray_of(i);
            cnt = counts[r];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o_r[a] = O[3 * r + a], d_r[a] = D[3 * r + a];
                dC[a] = d_rgb[3 * r + a], dN[a] = d_normal[3 * r + a];
            }
            dD = d_depth[r];
        }
        mbar_wait(bars + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const PipeSlot& sl = slots[st];
        if (kHdr) {
            const PipeHdr& h = sl.hdr;
            cnt = h.cnt;
            o = h.o;
            d = h.d;
#pragma unroll
            for (int a = 0; a < 3; ++a) dC[a] = h.dC[a], dN[a] = h.dN[a];
            dD = h.dD;
        }
        if (cnt) {
            const uint32_t k0 = 2 * lane, k1 = k0 + 1;
            PairT p;
            p.in0 = k0 < cnt;
            p.in1 = k1 < cnt;
            p.t0 = p.in0 ? sl.t[k0] : 0.0;
            p.t1 = p.in1 ? sl.t[k1] : 0.0;
            p.d0 = p.in1 ? static_cast<float>(__dsub_rn(p.t1, p.t0)) : static_cast<float>(step);
            p.d1 = (k1 + 1 < cnt) ? static_cast<float>(__dsub_rn(sl.t[k1 + 1], p.t1)) : static_cast<float>(step);
            SampleVal v0, v1;
            const bool ok0 = eval_from_record(g, o, d, p.in0, p.t0, sl.rec + 2 * k0, v0);
            const bool ok1 = eval_from_record(g, o, d, p.in1, p.t1, sl.rec + 2 * k1, v1);
            const float sg0 = ok0 ? density(v0.s, ib) : 0.f, sg1 = ok1 ? density(v1.s, ib) : 0.f;
            const float tau0 = sg0 * p.d0, tau1 = sg1 * p.d1;
            const float incl = warp_incl_scan(tau0 + tau1, lane);
            float excl = __shfl_up_sync(kFull, incl, 1);
            if (lane == 0) excl = 0.f;
            const float P0 = excl, P1 = P0 + tau0;
            const float w0 = ok0 ? expf(-P0) * -expm1f(-tau0) : 0.f;
            const float w1 = ok1 ? expf(-P1) * -expm1f(-tau1) : 0.f;
            const float Tn0 = expf(-P1), Tn1 = expf(-(P1 + tau1));
            const float vv0 = ok0 ? dC[0] * v0.r + dC[1] * v0.gc + dC[2] * v0.b + dD * static_cast<float>(p.t0) +
                                        dN[0] * v0.gx + dN[1] * v0.gy + dN[2] * v0.gz
                                  : 0.f;
            const float vv1 = ok1 ? dC[0] * v1.r + dC[1] * v1.gc + dC[2] * v1.b + dD * static_cast<float>(p.t1) +
                                        dN[0] * v1.gx + dN[1] * v1.gy + dN[2] * v1.gz
                                  : 0.f;
            const float u0 = w0 * vv0, u1 = w1 * vv1;
            const float sinc = warp_incl_suffix(u0 + u1, lane);
            float sexc = __shfl_down_sync(kFull, sinc, 1);
            if (lane == 31) sexc = 0.f;
            const float S1 = sexc, S0 = S1 + u1;
            const CornerCoef c0 = make_coef(v0, ok0 ? p.d0 * density_ds(v0.s, sg0, ib) * (Tn0 * vv0 - S0) : 0.f,
                                            w0, dC, dN, ih);
            const CornerCoef c1 = make_coef(v1, ok1 ? p.d1 * density_ds(v1.s, sg1, ib) * (Tn1 * vv1 - S1) : 0.f,
                                            w1, dC, dN, ih);
            if (ok0) mark_blocks(g, v0);
            if (ok1) mark_blocks(g, v1);
            if (kMode == 3) {
                scatter_pair_agg(g.grad, v0, v1, c0, c1, ok0, ok1, lane);
            } else {
                const bool same = ok0 && ok1 && v0.gidx[0] == v1.gidx[0];
                scatter_corner<0, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<1, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<2, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<3, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<4, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<5, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<6, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
                scatter_corner<7, kMode>(g.grad, v0, v1, c0, c1, ok0, ok1, same);
            }
        }
        __syncwarp();  // every lane is done reading slot st before it is refilled
        st = (st + 1) % kStages;
    }
}

// ---------------------------------------------------------------------------
// K6s: the pipelined backward with one sample per lane per 32-sample pass (samples 32 h + l),
// like k_forward_seq: pass A turns the staged records into tau and the exclusive prefix of
// both halves; pass B walks the halves back to front (suffix S_k carried across), evaluates
// one sample per lane and scatters with the one-step warp hand-off (lane l's cell run joins
// lane l-1's when it is the same cell).  Fewer live registers per lane than K6p.
// ---------------------------------------------------------------------------
template <int kMinBlocks, int kStages>
__global__ void __launch_bounds__(kPipeWarps * 32, kMinBlocks)
    k_backward_seq(GridView g, const double* __restrict__ O, const double* __restrict__ D, uint64_t n,
                   const uint32_t* __restrict__ order, const uint32_t* __restrict__ counts,
                   const double* __restrict__ T, uint32_t S, double step, float ib,
                   const float* __restrict__ d_rgb, const float* __restrict__ d_depth,
                   const float* __restrict__ d_normal, const float4* __restrict__ rec,
                   uint64_t warps_total) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    PipeSlot* slots = reinterpret_cast<PipeSlot*>(smem_raw) + wib * kStages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(PipeSlot) * kStages * kPipeWarps) +
                     wib * kStages;
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kPipeWarps + wib;
    const uint32_t tbytes = S * 8, rbytes = S * 32;
    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(bars + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto ray_of = [&](uint64_t i) -> uint64_t { return order ? order[i] : i; };
    auto issue = [&](uint64_t i, int st) {
        const uint64_t r = ray_of(i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bars + st, tbytes + rbytes);
        bulk_g2s(slots[st].t, T + r * S, tbytes, bars + st);
        bulk_g2s(slots[st].rec, rec + r * S * 2, rbytes, bars + st);
    };
    if (lane == 0)
        for (int st = 0; st < kStages - 1; ++st) {
            const uint64_t i = w0 + st * warps_total;
            if (i < n) issue(i, st);
        }
    const float ih = static_cast<float>(g.inv_h);
    uint32_t phase = 0;
    int st = 0;
    for (uint64_t i = w0; i < n; i += warps_total) {
        {
            const uint64_t nxt = i + (kStages - 1) * warps_total;
            const int nst = (st + kStages - 1) % kStages;
            if (lane == 0 && nxt < n) issue(nxt, nst);
        }
        const uint64_t r = ray_of(i);
        const uint32_t cnt = counts[r];
        mbar_wait(bars + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const PipeSlot& sl = slots[st];
        if (cnt) {
            const double o[3] = {O[3 * r], O[3 * r + 1], O[3 * r + 2]};
            const double d[3] = {D[3 * r], D[3 * r + 1], D[3 * r + 2]};
            const float dC[3] = {d_rgb[3 * r], d_rgb[3 * r + 1], d_rgb[3 * r + 2]};
            const float dD = d_depth[r];
            const float dN[3] = {d_normal[3 * r], d_normal[3 * r + 1], d_normal[3 * r + 2]};
            // pass A: tau_k from the records (s, validity) and delta_k from the t row
            float tau[2], dl[2], P[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t k = 32 * h + lane;
                const bool in = k < cnt;
                dl[h] = (k + 1 < cnt) ? static_cast<float>(__dsub_rn(sl.t[k + 1], sl.t[k])) : static_cast<float>(step);
                const bool ok = in && __float_as_uint(sl.rec[2 * k + 1].w) != kInvalid;
                tau[h] = ok ? density(sl.rec[2 * k].x, ib) * dl[h] : 0.f;
            }
            const float inc0 = warp_incl_scan(tau[0], lane);
            const float inc1 = warp_incl_scan(tau[1], lane);
            P[0] = inc0 - tau[0];
            P[1] = __shfl_sync(kFull, inc0, 31) + inc1 - tau[1];
            // pass B: back to front
            float S_after = 0.f;
#pragma unroll
            for (int h = 1; h >= 0; --h) {
                const uint32_t k = 32 * h + lane;
                const bool in = k < cnt;
                const double t = in ? sl.t[k] : 0.0;
                SampleVal v;
                const bool ok = eval_from_record(g, o, d, in, t, sl.rec + 2 * k, v);
                const float sg = ok ? density(v.s, ib) : 0.f;
                const float w = ok ? -expf(-P[h]) * expm1f(-tau[h]) : 0.f;
                const float Tn = expf(-(P[h] + tau[h]));
                const float vv = ok ? dC[0] * v.r + dC[1] * v.gc + dC[2] * v.b + dD * static_cast<float>(t) +
                                          dN[0] * v.gx + dN[1] * v.gy + dN[2] * v.gz
                                    : 0.f;
                const float u = w * vv;
                const float sinc = warp_incl_suffix(u, lane);
                float sexc = __shfl_down_sync(kFull, sinc, 1);
                if (lane == 31) sexc = 0.f;
                const float Sk = S_after + sexc;
                const CornerCoef c = make_coef(v, ok ? dl[h] * density_ds(v.s, sg, ib) * (Tn * vv - Sk) : 0.f, w,
                                               dC, dN, ih);
                if (ok) mark_blocks(g, v);
                // one-step hand-off: lane l's run joins lane l-1's when it is the same cell
                const uint32_t cell = ok ? v.gidx[0] : kInvalid;
                const uint32_t prev = __shfl_up_sync(kFull, cell, 1);
                const bool give = lane > 0 && ok && cell == prev;
                const bool recv = __shfl_down_sync(kFull, give ? 1u : 0u, 1) != 0u && lane < 31;
#define SVR_SEQ_CORNER(cc)                                                                        \
    {                                                                                             \
        const float4 a = ok ? corner_grad<cc>(c) : make_float4(0.f, 0.f, 0.f, 0.f);               \
        const float4 inb = shfl_down4(a);                                                         \
        if (ok) {                                                                                 \
            if (give) {                                                                           \
                if (recv) atomicAdd(g.grad + v.gidx[cc], inb);                                    \
            } else {                                                                              \
                atomicAdd(g.grad + v.gidx[cc], recv ? f4add(a, inb) : a);                         \
            }                                                                                     \
        }                                                                                         \
    }
                SVR_SEQ_CORNER(0) SVR_SEQ_CORNER(1) SVR_SEQ_CORNER(2) SVR_SEQ_CORNER(3)
                SVR_SEQ_CORNER(4) SVR_SEQ_CORNER(5) SVR_SEQ_CORNER(6) SVR_SEQ_CORNER(7)
#undef SVR_SEQ_CORNER
                S_after += __shfl_sync(kFull, sinc, 0);
            }
        }
        __syncwarp();
        st = (st + 1) % kStages;
    }
}

// ---------------------------------------------------------------------------
// K5p: pipelined forward (max_samples <= 64, even).  Persistent warps, 3-stage ring of
// t rows streamed with cp.async.bulk; while ray i is gathered and composited, ray i+1's
// t row is already resident and its base-voxel block lookups are in flight, and ray i+2's
// t row is being copied.  Per-ray scalars (o, d) ride in lanes 0-5 and are broadcast.
// ---------------------------------------------------------------------------
constexpr int kFwdStages = 3;

struct RayPrep {  // state of the next ray, prepared one iteration ahead
    uint64_t r;
    uint32_t cnt;
    double od;          // lane k < 6 holds o[k] (k < 3) or d[k-3]
    uint32_t e0a, e0b;  // block entries of the base voxels of this lane's two samples
};

__device__ __forceinline__ void bcast_od(double od, double o[3], double d[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k] = __shfl_sync(kFull, od, k);
        d[k] = __shfl_sync(kFull, od, k + 3);
    }
}

__device__ __forceinline__ uint32_t base_lookup(const GridView& g, const double o[3], const double d[3],
                                                double t) {
    int base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = __dadd_rn(o[a], __dmul_rn(t, d[a]));
        base[a] = static_cast<int>(floor(__dmul_rn(x, g.inv_h)));
    }
    return lookup_block(g, base[0] >> 3, base[1] >> 3, base[2] >> 3);
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kPipeWarps * 32, kMinBlocks)
    k_forward_pipe(GridView g, const double* __restrict__ O, const double* __restrict__ D, uint64_t n,
                   const uint32_t* __restrict__ order, const uint32_t* __restrict__ counts,
                   const double* __restrict__ T, uint32_t S, double step, float ib, float* rgb,
                   float* depth, float* normal, float* wsum, float4* rec, uint64_t warps_total) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double(*trow)[64] = reinterpret_cast<double(*)[64]>(smem_raw) + wib * kFwdStages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + sizeof(double) * 64 * kFwdStages * kPipeWarps) +
                     wib * kFwdStages;
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kPipeWarps + wib;
    const uint32_t tbytes = S * 8;
    if (lane == 0) {
        for (int st = 0; st < kFwdStages; ++st) mbar_init(bars + st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto ray_of = [&](uint64_t i) -> uint64_t { return order ? order[i] : i; };
    auto issue = [&](uint64_t i, int st) {
        const uint64_t r = ray_of(i);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bars + st, tbytes);
        bulk_g2s(trow[st], T + r * S, tbytes, bars + st);
    };
    uint32_t phase = 0;
    auto prep = [&](uint64_t i, int st, RayPrep& p) {  // scalars + base lookups of ray i
        p.r = ray_of(i);
        p.cnt = counts[p.r];
        p.od = lane < 3 ? O[3 * p.r + lane] : (lane < 6 ? D[3 * p.r + lane - 3] : 0.0);
        double o[3], d[3];
        bcast_od(p.od, o, d);
        mbar_wait(bars + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const uint32_t k0 = 2 * lane, k1 = k0 + 1;
        p.e0a = k0 < p.cnt ? base_lookup(g, o, d, trow[st][k0]) : kInvalid;
        p.e0b = k1 < p.cnt ? base_lookup(g, o, d, trow[st][k1]) : kInvalid;
    };
    if (w0 >= n) return;
    if (lane == 0) {
        issue(w0, 0);
        if (w0 + warps_total < n) issue(w0 + warps_total, 1);
    }
    RayPrep cur;
    prep(w0, 0, cur);
    int st = 0;
    const float ih = static_cast<float>(g.inv_h);
    for (uint64_t i = w0; i < n; i += warps_total) {
        const uint64_t i1 = i + warps_total, i2 = i + 2 * warps_total;
        const int st1 = (st + 1) % kFwdStages, st2 = (st + 2) % kFwdStages;
        if (lane == 0 && i2 < n) issue(i2, st2);
        RayPrep nxt;
        nxt.cnt = 0;
        if (i1 < n) prep(i1, st1, nxt);  // its lookups are in flight during this ray
        // ---- gather + composite ray i (t row in stage st) ----
        double o[3], d[3];
        bcast_od(cur.od, o, d);
        const uint64_t r = cur.r;
        const uint32_t cnt = cur.cnt;
        const double* tr = trow[st];
        const uint32_t k0 = 2 * lane, k1 = k0 + 1;
        PairT p;
        p.in0 = k0 < cnt;
        p.in1 = k1 < cnt;
        p.t0 = p.in0 ? tr[k0] : 0.0;
        p.t1 = p.in1 ? tr[k1] : 0.0;
        p.d0 = p.in1 ? static_cast<float>(__dsub_rn(p.t1, p.t0)) : static_cast<float>(step);
        p.d1 = (k1 + 1 < cnt) ? static_cast<float>(__dsub_rn(tr[k1 + 1], p.t1)) : static_cast<float>(step);
        SampleVal v0, v1;
        bool ok0 = false, ok1 = false;
        float4 p0[8], p1[8];
        {
            int b0[3], b1[3];
            zero_sample(v0);
            zero_sample(v1);
            if (p.in0) {
                cell_geom(g, o, d, p.t0, b0, v0);
                ok0 = corner_addrs<true>(g, b0, cur.e0a, v0);
            }
            if (p.in1) {
                cell_geom(g, o, d, p.t1, b1, v1);
                ok1 = corner_addrs<true>(g, b1, cur.e0b, v1);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                p0[c] = ok0 ? __ldg(g.pay + v0.gidx[c]) : make_float4(0.f, 0.f, 0.f, 0.f);
                p1[c] = ok1 ? __ldg(g.pay + v1.gidx[c]) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        auto interp = [&](SampleVal& v, const float4* pp, bool ok, uint32_t e0) {
            const float x1 = v.fx, x0 = 1.f - x1, y1 = v.fy, y0 = 1.f - y1, z1 = v.fz, z0 = 1.f - z1;
            const float w[8] = {x0 * y0 * z0, x1 * y0 * z0, x0 * y1 * z0, x1 * y1 * z0,
                                x0 * y0 * z1, x1 * y0 * z1, x0 * y1 * z1, x1 * y1 * z1};
            float sv = 0.f, rv = 0.f, gv = 0.f, bv = 0.f;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                sv = fmaf(w[c], pp[c].x, sv);
                rv = fmaf(w[c], pp[c].y, rv);
                gv = fmaf(w[c], pp[c].z, gv);
                bv = fmaf(w[c], pp[c].w, bv);
            }
            v.s = sv, v.r = rv, v.gc = gv, v.b = bv;
            v.gx = ih * ((y0 * z0) * (pp[1].x - pp[0].x) + (y1 * z0) * (pp[3].x - pp[2].x) +
                         (y0 * z1) * (pp[5].x - pp[4].x) + (y1 * z1) * (pp[7].x - pp[6].x));
            v.gy = ih * ((x0 * z0) * (pp[2].x - pp[0].x) + (x1 * z0) * (pp[3].x - pp[1].x) +
                         (x0 * z1) * (pp[6].x - pp[4].x) + (x1 * z1) * (pp[7].x - pp[5].x));
            v.gz = ih * ((x0 * y0) * (pp[4].x - pp[0].x) + (x1 * y0) * (pp[5].x - pp[1].x) +
                         (x0 * y1) * (pp[6].x - pp[2].x) + (x1 * y1) * (pp[7].x - pp[3].x));
            v.e0 = ok ? e0 : kInvalid;
        };
        interp(v0, p0, ok0, cur.e0a);
        interp(v1, p1, ok1, cur.e0b);
        if (rec) {
            float4* rr = rec + (r * S + 2 * lane) * 2;
            if (p.in0) store_record(rr, v0);
            if (p.in1) store_record(rr + 2, v1);
        }
        const float tau0 = ok0 ? density(v0.s, ib) * p.d0 : 0.f;
        const float tau1 = ok1 ? density(v1.s, ib) * p.d1 : 0.f;
        const float incl = warp_incl_scan(tau0 + tau1, lane);
        float excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = 0.f;
        const float P0 = excl, P1 = P0 + tau0;
        const float w0v = ok0 ? expf(-P0) * -expm1f(-tau0) : 0.f;
        const float w1v = ok1 ? expf(-P1) * -expm1f(-tau1) : 0.f;
        float acc[8];
        acc[0] = w0v * v0.r + w1v * v1.r;
        acc[1] = w0v * v0.gc + w1v * v1.gc;
        acc[2] = w0v * v0.b + w1v * v1.b;
        acc[3] = w0v * static_cast<float>(p.t0) + w1v * static_cast<float>(p.t1);
        acc[4] = w0v * v0.gx + w1v * v1.gx;
        acc[5] = w0v * v0.gy + w1v * v1.gy;
        acc[6] = w0v * v0.gz + w1v * v1.gz;
        acc[7] = w0v + w1v;
        write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
        __syncwarp();  // stage st is free for refilling
        cur = nxt;
        st = st1;
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

static inline unsigned grid_for(uint64_t n, unsigned per_block) {
    return static_cast<unsigned>((n + per_block - 1) / per_block);
}

void launch_query(const GridView& g, const double* x, uint64_t n, double* sdf, double* grad,
                  double* rgb, double* logits, uint8_t* valid, cudaStream_t s) {
    if (!n) return;
    k_query<<<grid_for(n, 256), 256, 0, s>>>(g, x, n, sdf, grad, rgb, logits, valid);
}

void launch_march(const GridView& g, const double* o, const double* d, uint64_t n,
                  const uint32_t* order, double step, uint32_t S, uint32_t* counts, double* t,
                  double* delta, cudaStream_t s, int variant, uint32_t* pkeys, uint32_t* pids) {
    if (!n) return;
    const unsigned grid = grid_for(n, 128);
    if (pkeys) {  // the default kernel, also writing the post-march sort keys
        k_march<6, true><<<grid, 128, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta, pkeys, pids);
        return;
    }
    switch (variant) {
        case 1: k_march<8, true><<<grid, 128, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
        case 2: k_march<6, true><<<grid, 128, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
        case 3: k_march<7, true><<<grid, 128, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
        case 4: k_march<12, true, 64><<<grid_for(n, 64), 64, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
        case 5: k_march<3, true, 256><<<grid_for(n, 256), 256, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
        default: k_march<1, false><<<grid, 128, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta); break;
    }
}

void launch_render_forward(const GridView& g, const double* o, const double* d, uint64_t n,
                           const uint32_t* order, const uint32_t* counts, const double* t, uint32_t S,
                           double step, double beta, float* rgb, float* depth, float* normal,
                           float* wsum, unsigned long long* valid_counter, float4* rec,
                           cudaStream_t s, int min_blocks, const uint2* hdr) {
    if (!n) return;
    const float ib = static_cast<float>(1.0 / beta);
#define SVR_FWD(TH, MB)                                                                         \
    k_forward<TH, MB><<<grid_for(n * 32, TH), TH, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib, \
                                                          rgb, depth, normal, wsum, valid_counter, rec)
    switch (min_blocks) {
        case 1: SVR_FWD(256, 1); break;
        case 2: SVR_FWD(256, 2); break;
        case 4: SVR_FWD(256, 4); break;
        case 11: SVR_FWD(768, 1); break;  // one 24-warp CTA per SM: concurrent warps = adjacent rays
        case 12: SVR_FWD(512, 1); break;
        case 13: SVR_FWD(1024, 1); break;
        case 105: k_forward_seq<256, 4><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step,
                                                                              ib, rgb, depth, normal, wsum,
                                                                              valid_counter, rec);
            break;
        case 109: k_forward_seq<256, 4, true><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S,
                                                                                    step, ib, rgb, depth, normal,
                                                                                    wsum, valid_counter, rec);
            break;
        case 111: k_forward_seq<128, 8, true><<<grid_for(n * 32, 128), 128, 0, s>>>(g, o, d, n, order, counts, t, S,
                                                                                    step, ib, rgb, depth, normal,
                                                                                    wsum, valid_counter, rec);
            break;
        case 113: k_forward_seq<64, 16, true><<<grid_for(n * 32, 64), 64, 0, s>>>(g, o, d, n, order, counts, t, S,
                                                                                  step, ib, rgb, depth, normal,
                                                                                  wsum, valid_counter, rec);
            break;
#define SVR_FWD_MULTI(TH, MB, K)                                                                  \
    if (hdr)                                                                                      \
        k_forward_multi<TH, MB, K, true><<<grid_for((n + K - 1) / K * 32, TH), TH, 0, s>>>(         \
            g, o, d, n, order, counts, t, S, step, ib, rgb, depth, normal, wsum, valid_counter, rec, hdr); \
    else                                                                                          \
        k_forward_multi<TH, MB, K, false><<<grid_for((n + K - 1) / K * 32, TH), TH, 0, s>>>(        \
            g, o, d, n, order, counts, t, S, step, ib, rgb, depth, normal, wsum, valid_counter, rec, nullptr)
        case 114: SVR_FWD_MULTI(64, 16, 2); break;
        case 115: SVR_FWD_MULTI(64, 16, 4); break;
        case 116: SVR_FWD_MULTI(128, 8, 4); break;
        case 117: SVR_FWD_MULTI(64, 16, 3); break;
        case 118: SVR_FWD_MULTI(64, 16, 5); break;
        case 119: SVR_FWD_MULTI(64, 16, 1); break;
        case 120: SVR_FWD_MULTI(128, 8, 1); break;
        case 121: SVR_FWD_MULTI(256, 4, 1); break;
        case 122: SVR_FWD_MULTI(32, 32, 1); break;
#undef SVR_FWD_MULTI
        case 112: k_forward_seq<512, 2, true><<<grid_for(n * 32, 512), 512, 0, s>>>(g, o, d, n, order, counts, t, S,
                                                                                    step, ib, rgb, depth, normal,
                                                                                    wsum, valid_counter, rec);
            break;
        case 110: k_forward_seq<256, 5, true><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S,
                                                                                    step, ib, rgb, depth, normal,
                                                                                    wsum, valid_counter, rec);
            break;
        case 107: k_forward_seq<256, 5><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step,
                                                                              ib, rgb, depth, normal, wsum,
                                                                              valid_counter, rec);
            break;
        case 108: k_forward_seq<256, 6><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step,
                                                                              ib, rgb, depth, normal, wsum,
                                                                              valid_counter, rec);
            break;
        case 106: k_forward_seq<256, 3><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step,
                                                                              ib, rgb, depth, normal, wsum,
                                                                              valid_counter, rec);
            break;
        case 104: k_forward_split<256, 3><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step,
                                                                                ib, rgb, depth, normal, wsum,
                                                                                valid_counter, rec);
            break;
        // diagnostics (wrong results): 101 no payload loads, 102 no block lookup, 103 no records
        case 101: k_forward<256, 3, 1><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib,
                                                                           rgb, depth, normal, wsum, valid_counter, rec);
            break;
        case 102: k_forward<256, 3, 2><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib,
                                                                           rgb, depth, normal, wsum, valid_counter, rec);
            break;
        case 103: k_forward<256, 3, 3><<<grid_for(n * 32, 256), 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib,
                                                                           rgb, depth, normal, wsum, valid_counter, rec);
            break;
        default: SVR_FWD(256, 3); break;
    }
#undef SVR_FWD
}

void launch_render_backward(const GridView& g, const double* o, const double* d, uint64_t n,
                            const uint32_t* order, const uint32_t* counts, const double* t,
                            uint32_t S, double step, double beta, const float* d_rgb,
                            const float* d_depth, const float* d_normal, const float4* rec,
                            cudaStream_t s, int min_blocks, bool agg) {
    if (!n) return;
    const float ib = static_cast<float>(1.0 / beta);
    const unsigned grid = grid_for(n * 32, 256);
#define SVR_COMMA(a, b, c) a, b, c
#define SVR_BWD(...) k_backward<__VA_ARGS__><<<grid, 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib, \
                                                                d_rgb, d_depth, d_normal, rec)
    const bool r = rec != nullptr;
    switch (min_blocks) {
        case 2: r ? SVR_BWD(2, 0, true) : SVR_BWD(2, 0, false); break;
        case 4: r ? SVR_BWD(4, 0, true) : SVR_BWD(4, 0, false); break;
        case 103:  // diagnostics (wrong gradients): plain stores / arithmetic only
            r ? SVR_BWD(3, 1, true) : SVR_BWD(3, 1, false);
            break;
        case 203:
            r ? SVR_BWD(3, 2, true) : SVR_BWD(3, 2, false);
            break;
        default:
            if (agg)
                r ? SVR_BWD(3, 3, true) : SVR_BWD(3, 3, false);
            else
                r ? SVR_BWD(3, 0, true) : SVR_BWD(3, 0, false);
            break;
    }
#undef SVR_BWD
#undef SVR_COMMA
}

// {id, sample count} of every ray in sorted order, for the forward's first load level
__global__ void k_ray_headers(const uint32_t* __restrict__ order, const uint32_t* __restrict__ counts,
                              uint64_t n, uint2* __restrict__ hdr) {
    const uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= n) return;
    const uint32_t r = order[w];
    hdr[w] = make_uint2(r, counts[r]);
}

void launch_ray_headers(const uint32_t* order, const uint32_t* counts, uint64_t n, uint2* hdr, cudaStream_t s) {
    if (n) k_ray_headers<<<grid_for(n, 256), 256, 0, s>>>(order, counts, n, hdr);
}

void launch_ray_order(const GridView& g, const double* o, const double* d, uint64_t n,
                      const uint32_t* counts, const double* t, uint32_t S, uint32_t* keys,
                      uint32_t* ids, uint32_t* keys_alt, uint32_t* ids_alt, void* tmp,
                      size_t tmp_bytes, uint32_t** sorted_ids, cudaStream_t s, int key_mode) {
    if (!n) return;
    if (counts && t)  // post-march: first-sample block
        k_ray_keys<<<grid_for(n, 256), 256, 0, s>>>(g, o, d, n, counts, t, S, keys, ids, key_mode);
    else if (!counts)  // pre-march: origin + direction
        k_ray_keys_dir<<<grid_for(n, 256), 256, 0, s>>>(o, d, n, keys, ids);
    // (counts && !t: the march already wrote the post-march keys / ids)
    // sort only the key bits in use: 24 for the pre-march key; 3 x (bits per axis of the
    // block AABB) for the post-march Morton key (empty rays carry all ones and sort last)
    int end_bit = 24;
    if (counts) {
        const int sc = key_mode == 2 ? 2 : 1;
        int bits = 1;
        while (bits < 10 && ((1 << bits) < sc * g.dim[0] || (1 << bits) < sc * g.dim[1] || (1 << bits) < sc * g.dim[2]))
            ++bits;
        end_bit = 3 * bits;
    }
    cub::DoubleBuffer<uint32_t> kb(keys, keys_alt), vb(ids, ids_alt);
    size_t bytes = tmp_bytes;
    cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int>(n), 0, end_bit, s);
    *sorted_ids = vb.Current();
}

bool launch_render_backward_pipe(const GridView& g, const double* o, const double* d, uint64_t n,
                                 const uint32_t* order, const uint32_t* counts, const double* t,
                                 uint32_t S, double step, double beta, const float* d_rgb,
                                 const float* d_depth, const float* d_normal, const float4* rec,
                                 cudaStream_t s, int min_blocks, int num_sms, bool agg, bool hdr) {
    if (!n) return true;
    if (!rec || S > 64 || (S & 1)) return false;
    // the default (agg + ray scalars in the ring) runs a 2-stage ring: one ray of look-ahead
    // covers the loads once the scalars travel with the rows, and the smaller ring leaves
    // more of the SM's 256 KB to L1 (2.40 vs 2.45 ms with 3 stages)
    const bool def2 = agg && hdr && (min_blocks == 3 || min_blocks == 0 || min_blocks > 5) && min_blocks != 203 &&
                      min_blocks != 310 && min_blocks != 311 && min_blocks < 600;
    const int stages = (min_blocks == 4 || min_blocks == 5 || def2) ? 2 : (min_blocks == 311 ? 4 : kPipeStages);
    const size_t smem = sizeof(PipeSlot) * stages * kPipeWarps + 8 * stages * kPipeWarps;
    const float ib = static_cast<float>(1.0 / beta);
    const int mb_eff = min_blocks == 310 ? 3 : min_blocks == 311 ? 2
                       : min_blocks >= 600 ? (min_blocks == 601 ? 3 : (min_blocks == 602 ? 4 : 5)) : min_blocks % 100;
    uint64_t ctas = static_cast<uint64_t>(num_sms) * mb_eff;
    const uint64_t need = (n + kPipeWarps - 1) / kPipeWarps;
    if (ctas > need) ctas = need;
    const uint64_t warps_total = ctas * kPipeWarps;
#define SVR_COMMA2(a, b) a, b
#define SVR_COMMA3(a, b, c) a, b, c
#define SVR_COMMA4(a, b, c, e) a, b, c, e
#define SVR_SEQ(MB, ST)                                                                           \
    do {                                                                                          \
        const size_t sm = sizeof(PipeSlot) * (ST) * kPipeWarps + 8 * (ST) * kPipeWarps;           \
        cudaFuncSetAttribute(k_backward_seq<MB, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             static_cast<int>(sm));                                               \
        k_backward_seq<MB, ST><<<static_cast<unsigned>(ctas), kPipeWarps * 32, sm, s>>>(          \
            g, o, d, n, order, counts, t, S, step, ib, d_rgb, d_depth, d_normal, rec, warps_total); \
    } while (0)
#define SVR_PIPE(...)                                                                             \
    do {                                                                                          \
        cudaFuncSetAttribute(k_backward_pipe<__VA_ARGS__>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             static_cast<int>(smem));                                             \
        k_backward_pipe<__VA_ARGS__><<<static_cast<unsigned>(ctas), kPipeWarps * 32, smem, s>>>(  \
            g, o, d, n, order, counts, t, S, step, ib, d_rgb, d_depth, d_normal, rec, warps_total); \
    } while (0)
    switch (min_blocks) {
        case 1:
            if (agg) SVR_PIPE(SVR_COMMA2(1, 3));
            else SVR_PIPE(1);
            break;
        case 2:
            if (agg) SVR_PIPE(SVR_COMMA2(2, 3));
            else SVR_PIPE(2);
            break;
        case 4: SVR_PIPE(SVR_COMMA3(4, 3, 2)); break;  // 2-stage ring, 64 registers
        case 5: SVR_PIPE(SVR_COMMA3(5, 3, 2)); break;
        case 203: SVR_PIPE(SVR_COMMA2(3, 2)); break;  // diagnostic: no atomics (wrong gradients)
        case 310: SVR_PIPE(SVR_COMMA4(3, 3, 3, true)); break;  // 3-stage ring with the ray scalars
        case 311: SVR_PIPE(SVR_COMMA4(2, 3, 4, true)); break;  // experiment: 4-stage ring, 2 CTAs
        case 601: SVR_SEQ(3, 3); break;  // one sample per lane per pass
        case 602: SVR_SEQ(4, 2); break;
        case 603: SVR_SEQ(5, 2); break;
        default:
            if (agg && hdr) SVR_PIPE(SVR_COMMA4(3, 3, 2, true));
            else if (agg) SVR_PIPE(SVR_COMMA2(3, 3));
            else SVR_PIPE(3);
            break;
    }
#undef SVR_COMMA4
#undef SVR_PIPE
#undef SVR_SEQ
#undef SVR_COMMA2
#undef SVR_COMMA3
    return true;
}

bool launch_render_forward_pipe(const GridView& g, const double* o, const double* d, uint64_t n,
                                const uint32_t* order, const uint32_t* counts, const double* t,
                                uint32_t S, double step, double beta, float* rgb, float* depth,
                                float* normal, float* wsum, float4* rec, cudaStream_t s,
                                int min_blocks, int num_sms) {
    if (!n) return true;
    if (S > 64 || (S & 1)) return false;
    const size_t smem = sizeof(double) * 64 * kFwdStages * kPipeWarps + 8 * kFwdStages * kPipeWarps;
    const float ib = static_cast<float>(1.0 / beta);
    uint64_t ctas = static_cast<uint64_t>(num_sms) * min_blocks;
    const uint64_t need = (n + kPipeWarps - 1) / kPipeWarps;
    if (ctas > need) ctas = need;
    const uint64_t warps_total = ctas * kPipeWarps;
#define SVR_FPIPE(MB)                                                                                 \
    k_forward_pipe<MB><<<static_cast<unsigned>(ctas), kPipeWarps * 32, smem, s>>>(                  \
        g, o, d, n, order, counts, t, S, step, ib, rgb, depth, normal, wsum, rec, warps_total)
    switch (min_blocks) {
        case 1: SVR_FPIPE(1); break;
        case 2: SVR_FPIPE(2); break;
        case 4: SVR_FPIPE(4); break;
        default: SVR_FPIPE(3); break;
    }
#undef SVR_FPIPE
    return true;
}

size_t ray_order_tmp_bytes(uint64_t n) {
    size_t bytes = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, static_cast<int>(n), 0, 32);
    return bytes;
}

}  // namespace svr_internal
