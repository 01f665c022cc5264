// sm_100a kernels of the rendering hot path:
//   K2 k_query     -- fp64 trilinear query, bit-exact with grid.cpp:112-261
//   K4 k_march     -- ray-block DDA + fixed-step sampling, bit-exact with grid.cpp:263-353
//   K5 k_forward   -- fused gather/interpolate/Laplace density/compositing, warp per ray;
//                     leaves the per-sample records; stores a pending zeroing's zeros
//   K6p k_backward_pipe -- persistent warps streaming t + record rows (cp.async.bulk ring):
//                     compositing adjoint (warp scans) + factored trilinear adjoint +
//                     predicated red.global.add.v4.f32 scatter into the float4 gradient
//                     planes; active blocks through the touch table (k_touch_expand)
//   K6 k_backward  -- the same for max_samples > 64 / no records (64-sample chunks)
// Discrete decisions (which block/cell, sample t) use fp64 with explicit _rn
// intrinsics so nvcc cannot contract them into FMA (the reference's x86-64 Release
// build has no FMA, proj/CMakeLists.txt:9-11).  Continuous interpolation and
// compositing run in fp32 (tolerance 1e-4 |ref| + 1e-6 max |ref|, tests/common.py).
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
        // the estimate is exact again: the early stop below keeps its one-per-run slack
        // for the runs recorded from here on
        est = cnt;
        est_cursor = cursor;
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
        } else if (g.use_dense) {
            alloc = ((__ldg(g.occ + (static_cast<uint32_t>(cell) >> 5)) >> (cell & 31)) & 1u) != 0;
        } else {
            // hash mode: a superblock at Chebyshev distance dsb >= 1 from every occupied one has
            // every block within 8 (dsb - 1) of this one empty -- no probe, and a jump when that
            // radius allows (dist - 1 = 8 (dsb - 1)); otherwise the block's own hash probe
            int dsb = 0;
            if (g.sbinfo) {  // bricks: the block's own distance near blocks, no probe at all
                const uint32_t sx = static_cast<uint32_t>((b0 >> 3) - g.sb_lo[0]);
                const uint32_t sy = static_cast<uint32_t>((b1 >> 3) - g.sb_lo[1]);
                const uint32_t sz = static_cast<uint32_t>((b2 >> 3) - g.sb_lo[2]);
                const uint32_t inf = __ldg(g.sbinfo + (static_cast<size_t>(sz) * g.sb_dim[1] + sy) * g.sb_dim[0] + sx);
                if (inf & kNoBrick) {
                    dist = 8 * (static_cast<int>(inf & 0xFFu) - 1) + 1;
                } else {
                    dist = __ldg(g.bricks + static_cast<size_t>(inf) * kVox + (b0 & 7) + 8 * ((b1 & 7) + 8 * (b2 & 7)));
                }
                alloc = dist == 0;
            } else {
                if (g.sbdist) {
                    const uint32_t sx = static_cast<uint32_t>((b0 >> 3) - g.sb_lo[0]);
                    const uint32_t sy = static_cast<uint32_t>((b1 >> 3) - g.sb_lo[1]);
                    const uint32_t sz = static_cast<uint32_t>((b2 >> 3) - g.sb_lo[2]);
                    dsb = __ldg(g.sbdist + (static_cast<size_t>(sz) * g.sb_dim[1] + sy) * g.sb_dim[0] + sx);
                }
                if (dsb >= 1) {
                    alloc = false;
                    dist = 8 * (dsb - 1) + 1;
                } else {
                    alloc = hash_find(g, pack_key(b0, b1, b2)) != kInvalid;
                }
            }
        }
        // jump only when every walking lane of the warp can: a partial set of jumpers would run
        // the jump's exact crossing counts while the others idle (measured: all 0.536 ms, >= 3/4
        // 0.545, >= 1/2 0.56, any 0.588); stepping instead is always exact
        const unsigned walkers = __activemask();
        const unsigned jumpers = __ballot_sync(walkers, dist >= 3);
        if (dist >= 3 && jumpers == walkers) {
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

// thread per ray; o / d in shared memory (SoA) instead of 12 registers: 6 CTAs of 128 per SM
constexpr int kMarchThreads = 128;
__global__ void __launch_bounds__(kMarchThreads, 6) k_march(GridView g, const double* __restrict__ O,
                                                            const double* __restrict__ D, uint64_t n,
                                                            const uint32_t* __restrict__ order, double step,
                                                            uint32_t S, uint32_t* counts, double* T, double* delta,
                                                            uint32_t* pkeys, uint32_t* pids,
                                                            unsigned long long* valid_counter) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i == 0 && valid_counter) *valid_counter = 0;  // the forward that follows counts into it
    if (i >= n) return;
    const uint64_t r = order ? order[i] : i;
    double* tr = T + r * S;
    double t_first = 0.0;
    __shared__ double s_od[6][kMarchThreads];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        s_od[a][threadIdx.x] = O[3 * r + a];
        s_od[3 + a][threadIdx.x] = D[3 * r + a];
    }
    const StridedVec o{&s_od[0][threadIdx.x], kMarchThreads}, d{&s_od[3][threadIdx.x], kMarchThreads};
    // t values leave in aligned pairs (one 16 B store per two samples: half the store
    // instructions of this thread-per-ray kernel, whose stores never coalesce across lanes)
    double t_even = 0.0;
    const bool pairs = (S & 1u) == 0;
    const uint32_t cnt = march_dev(g, o, d, step, S, [&](uint32_t k, double t) {
        if (!pairs) {
            tr[k] = t;
        } else if (k & 1u) {
            *reinterpret_cast<double2*>(tr + k - 1) = make_double2(t_even, t);
        } else {
            t_even = t;
        }
        if (k == 0) t_first = t;
    });
    if (pairs && (cnt & 1u)) tr[cnt - 1] = t_even;
    counts[r] = cnt;
    if (pkeys) {  // the post-march sort key without re-reading the t row
        pkeys[r] = first_sample_key(g, o, d, cnt, t_first);
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
    uint32_t bpar;  // parity of the base voxel: (bx & 1) | (by & 1) << 1 | (bz & 1) << 2
    uint32_t e0;    // block entry of the base voxel (kInvalid: invalid sample)
};

__device__ __forceinline__ void zero_sample(SampleVal& v) {
    v.s = v.gx = v.gy = v.gz = v.r = v.gc = v.b = 0.f;
    v.fx = v.fy = v.fz = 0.f;
    v.smask = 0;
    v.bpar = 0;
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
    v.bpar = (lx & 1u) | ((ly & 1u) << 1) | ((lz & 1u) << 2);
}

// Corner c of the cell lies in block (base + bits(c)) >> 3; only axes with local
// coordinate 7 cross a face (smask), and those corners take their block entry from the
// per-block neighbour table; verifies presence + validity (weight > 0).
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
        ok = ok && ec != kInvalid;
        full &= ec;
        v.gidx[c] = (ec & ~kFullBit) * kVox + (X[c & 1] + Y[(c >> 1) & 1] + Z[c >> 2]);
    }
    if (ok && !(full & kFullBit)) {  // some corner block is partially observed
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t gi = v.gidx[c];
            ok = ok && ((__ldg(g.vmask + (gi >> 5)) >> (gi & 31)) & 1u);
        }
    }
    return ok;
}

// Parity-ordered corner addresses (the backward's scatter order, see scatter_pair_par):
// gidx[p] = the cell corner whose voxel coordinates have parities p = (px, py, pz).  On axis a
// that voxel is the base voxel when p_a equals the base parity, else base + 1; it lies in the
// next block exactly when the base is at local 7 and p_a is even (the base is odd there), so
// the neighbour-table slot of parity p is smask & ~p.
__device__ __forceinline__ void corner_addrs_par(const GridView& g, const int base[3], uint32_t e0, SampleVal& v) {
    const uint32_t lx = base[0] & 7, ly = base[1] & 7, lz = base[2] & 7;
    const uint32_t blk0 = e0 & ~kFullBit;
    // local offset of the parity-q voxel per axis (upper = base + 1 wraps to 0 across a face)
    const uint32_t X[2] = {(lx + (lx & 1u)) & 7u, (lx + (~lx & 1u)) & 7u};
    const uint32_t Y[2] = {((ly + (ly & 1u)) & 7u) * 8u, ((ly + (~ly & 1u)) & 7u) * 8u};
    const uint32_t Z[2] = {((lz + (lz & 1u)) & 7u) * 64u, ((lz + (~lz & 1u)) & 7u) * 64u};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t k = v.smask & (~static_cast<uint32_t>(q) & 7u);
        const uint32_t ec = k ? __ldg(g.nbr + static_cast<size_t>(blk0) * 8 + k) : e0;
        v.gidx[q] = (ec & ~kFullBit) * kVox + (X[q & 1] + Y[(q >> 1) & 1] + Z[q >> 2]);
    }
    v.bpar = (lx & 1u) | ((ly & 1u) << 1) | ((lz & 1u) << 2);
}

// Full gather + trilinear interpolation of sdf, grad(sdf) and rgb (fp32 payload math).
__device__ __forceinline__ bool eval_sample(const GridView& g, const double o[3], const double d[3],
                                            double t, SampleVal& v) {
    int base[3];
    cell_geom(g, o, d, t, base, v);
    const uint32_t e0 = lookup_block(g, base[0] >> 3, base[1] >> 3, base[2] >> 3);
    const bool ok = corner_addrs(g, base, e0, v);
    if (!ok) {
        v.s = v.gx = v.gy = v.gz = v.r = v.gc = v.b = 0.f;
        v.e0 = kInvalid;
        return false;
    }
    v.e0 = e0;
    float4 p[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) p[c] = __ldg(g.pay + v.gidx[c]);
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
__device__ __forceinline__ bool eval_slot(const GridView& g, const double o[3], const double d[3],
                                          bool in, double t, SampleVal& v) {
    if (in) return eval_sample(g, o, d, t, v);
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

// The backward's invalid sample: zeros, and no corner addresses (the scatter keys on them).
__device__ __forceinline__ void zero_sample_bwd(SampleVal& v) {
    zero_sample(v);
#pragma unroll
    for (int c = 0; c < 8; ++c) v.gidx[c] = kInvalid;
}

// `rec` may point to global memory (k_backward) or shared memory (k_backward_pipe):
// generic loads only.
__device__ __forceinline__ bool eval_from_record(const GridView& g, const double o[3],
                                                 const double d[3], bool in, double t,
                                                 const float4* rec, SampleVal& v) {
    if (!in) {
        zero_sample_bwd(v);
        return false;
    }
    const float4 a = rec[0], b = rec[1];
    const uint32_t e0 = __float_as_uint(b.w);
    if (e0 == kInvalid) {
        zero_sample_bwd(v);
        return false;
    }
    int base[3];
    cell_geom(g, o, d, t, base, v);
    corner_addrs_par(g, base, e0, v);
    v.e0 = e0;
    v.s = a.x, v.r = a.y, v.gc = a.z, v.b = a.w;
    v.gx = b.x, v.gy = b.y, v.gz = b.z;
    return true;
}

// Laplace density and its derivative.
// One exponential for both branches: -|s| ib is exactly -s ib for s > 0 and s ib otherwise.
__device__ __forceinline__ float density(float s, float ib) {
    const float e = expf(-fabsf(s) * ib);
    return s > 0.f ? ib * (0.5f * e) : ib * (1.f - 0.5f * e);
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
// K5: forward.  One warp per ray (one-warp CTAs, 32 resident per SM at <= 64 registers),
// one sample per lane per 32-sample pass; the exclusive prefix of tau by a warp scan gives
// T_k = exp(-sum_{j<k} tau_j).  The ray's o / d sit in a per-warp shared slot (6 lanes load
// them), and each lane's t value is fetched one pass ahead so a pass starts with its cell
// decision instead of a dependent load.  Leaves a 32 B record per sample for the backward.
// ---------------------------------------------------------------------------
constexpr int kFwdThreads = 32;
// the gradient rows a pending svr_grad_zero_active leaves to the next forward
struct ZeroRows {
    float4* grad;
    uint8_t* active;
    const uint32_t* list;               // ascending active rows (nullptr: nothing pending)
    const unsigned long long* count;    // device-side row count
};
__global__ void __launch_bounds__(kFwdThreads, 32) k_forward(GridView g, const double* __restrict__ O,
                                                             const double* __restrict__ D, uint64_t n,
                                                             const uint32_t* __restrict__ order,
                                                             const uint32_t* __restrict__ counts,
                                                             const double* __restrict__ T, uint32_t S,
                                                             double step, float ib, float* rgb, float* depth,
                                                             float* normal, float* wsum,
                                                             unsigned long long* valid_counter, float4* rec,
                                                             ZeroRows z) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    __shared__ double s_od[kFwdThreads / 32][6];
    const uint32_t r = order ? order[w] : static_cast<uint32_t>(w);
    if (lane < 6) s_od[wib][lane] = lane < 3 ? O[3ull * r + lane] : D[3ull * r + lane - 3];
    const uint32_t cnt = counts[r];
    __syncwarp();
    const double* o = s_od[wib];
    const double* d = o + 3;
    const double* tr = T + static_cast<uint64_t>(r) * S;
    // t of the upcoming pass and of the sample after it (delta_k = t_{k+1} - t_k), both loaded
    // one pass ahead (no shuffles: they share the L1 data path with the gathers)
    double t_cur = static_cast<uint32_t>(lane) < cnt ? tr[lane] : 0.0;
    double tn_cur = static_cast<uint32_t>(lane) + 1 < cnt ? tr[lane + 1] : 0.0;
    uint32_t nvalid = 0;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // C, D, N, W
    float tau_base = 0.f;
    for (uint32_t base = 0; base < cnt; base += 32) {
        const uint32_t k0 = base + lane;
        const bool in0 = k0 < cnt;
        const double t0 = in0 ? t_cur : 0.0;
        const double tn0 = tn_cur;
        t_cur = k0 + 32 < cnt ? tr[k0 + 32] : 0.0;  // one pass ahead
        tn_cur = k0 + 33 < cnt ? tr[k0 + 33] : 0.0;
        const float d0 = (k0 + 1 < cnt) ? static_cast<float>(__dsub_rn(tn0, t0)) : static_cast<float>(step);
        SampleVal v0;
        const bool ok0 = eval_slot(g, o, d, in0, t0, v0);
        if (rec && in0) store_record(rec + (static_cast<uint64_t>(r) * S + k0) * 2, v0);
        const float tau0 = ok0 ? density(v0.s, ib) * d0 : 0.f;
        const float inc0 = warp_incl_scan(tau0, lane);
        const float wk = -expf(-(tau_base + inc0 - tau0)) * expm1f(-tau0);
        acc[0] += wk * v0.r;
        acc[1] += wk * v0.gc;
        acc[2] += wk * v0.b;
        acc[3] += wk * static_cast<float>(t0);
        acc[4] += wk * v0.gx;
        acc[5] += wk * v0.gy;
        acc[6] += wk * v0.gz;
        acc[7] += wk;
        if (valid_counter) nvalid += __popc(__ballot_sync(kFull, ok0));
        tau_base += __shfl_sync(kFull, inc0, 31);
    }
    write_ray_outputs(warp_sum8(acc, lane), lane, r, rgb, depth, normal, wsum);
    if (lane == 0 && valid_counter && nvalid) atomicAdd(valid_counter, static_cast<unsigned long long>(nvalid));
    if (z.list) {  // a pending svr_grad_zero_active: this warp's share of the active rows, 512 B a store
        const unsigned long long chunks = *z.count * (kVox / 32);
        for (unsigned long long j = w; j < chunks; j += n) {
            const uint32_t row = z.list[j / (kVox / 32)];
            const uint32_t part = static_cast<uint32_t>(j % (kVox / 32));
            z.grad[static_cast<size_t>(row) * kVox + part * 32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (part == 0 && lane == 0) z.active[row] = 0;
        }
    }
}

// Gradient of corner c of one sample: (g_sdf, g_r, g_g, g_b) with
//   g_sdf = w_c dL/ds + dw_c . (w_k dN),  g_rgb = w_c w_k dC.
// The sdf term is evaluated factored, g_sdf = wz (wy (wx ds + sx wn_x) + sy wx wn_y) + sz wx wy
// wn_z, so the corners sharing (x, y) share the x and xy partial products:
// ax[i] = w_x(i) ds + s_x(i) wn_x, bx[i] = w_x(i) wn_y (i = the corner's x bit).
struct CornerCoef {
    float x0, x1, y0, y1, z0, z1, ax0, ax1, bx0, bx1, wn2, wc0, wc1, wc2;
};
struct XYPart {
    float bxy, wxy, cxy;
};
template <int q>  // the xy partials of corners q and q + 4 (q = x bit | y bit << 1)
__device__ __forceinline__ XYPart xy_part(const CornerCoef& k) {
    const float wx = (q & 1) ? k.x1 : k.x0, wy = (q & 2) ? k.y1 : k.y0;
    const float ax = (q & 1) ? k.ax1 : k.ax0, bx = (q & 1) ? k.bx1 : k.bx0;
    XYPart r;
    r.bxy = fmaf(wy, ax, (q & 2) ? bx : -bx);
    r.wxy = wx * wy;
    r.cxy = r.wxy * k.wn2;
    return r;
}
template <int c>
__device__ __forceinline__ float4 corner_grad(const CornerCoef& k, const XYPart& xy) {
    const float wz = (c & 4) ? k.z1 : k.z0;
    const float gs = fmaf(wz, xy.bxy, (c & 4) ? xy.cxy : -xy.cxy);
    const float w = xy.wxy * wz;
    return make_float4(gs, w * k.wc0, w * k.wc1, w * k.wc2);
}

// Active-block marking through the touch table: a valid sample with base block b and
// face-crossing mask k (corners in the blocks b + bits(c), c a subset of k) sets
// touch[8 b + k] with a plain byte store -- no load, so the warp never waits on it -- once
// per run of equal (b, k) along the ray (a lane's pair, and the previous lane's last sample).
// k_touch_expand then marks the blocks of every flagged (b, k) and clears the table.
__device__ __forceinline__ uint32_t touch_key(const SampleVal& v) {
    return ((v.e0 & ~kFullBit) << 3) | v.smask;
}
__device__ __forceinline__ void touch_pair(const GridView& g, const SampleVal& v0, const SampleVal& v1, bool ok0,
                                           bool ok1, int lane) {
    const uint32_t k0 = ok0 ? touch_key(v0) : kInvalid, k1 = ok1 ? touch_key(v1) : kInvalid;
    const uint32_t last = ok1 ? k1 : k0;
    uint32_t prev = __shfl_up_sync(kFull, last, 1);
    if (lane == 0) prev = kInvalid;
    if (ok0 && k0 != prev) g.touch[k0] = 1;
    if (ok1 && k1 != (ok0 ? k0 : prev)) g.touch[k1] = 1;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 shfl_down4(float4 v) {
    return make_float4(__shfl_down_sync(kFull, v.x, 1), __shfl_down_sync(kFull, v.y, 1),
                       __shfl_down_sync(kFull, v.z, 1), __shfl_down_sync(kFull, v.w, 1));
}

// Parity-ordered scatter.  Every voxel of a cell has a distinct coordinate parity
// p = (vx & 1) | (vy & 1) << 1 | (vz & 1) << 2, and a voxel shared by two cells has the same
// parity in both -- so "the parity-p corner" is a label that persists as the ray moves from cell
// to cell, whereas the corner index c = p ^ parity(base) flips on every face crossing.  Along a
// ray the samples touching one voxel are consecutive (the 2x2x2 cells around it form a convex
// box), so keying the warp hand-off by the parity-p voxel address merges the corners two
// face-adjacent cells share, not only identical cells.  to_parity_order permutes the gidx
// array (XOR butterfly on the base parity) and make_coef_par swaps the 1-D weight factors /
// derivative signs of the odd axes, so corner_grad<p> yields the parity-p corner's gradient.
__device__ __forceinline__ void to_parity_order(SampleVal& v) {
    uint32_t* g = v.gidx;
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1) {
        const bool sw = (v.bpar & bit) != 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (!(i & bit)) {
                const uint32_t a = g[i], b = g[i | bit];
                g[i] = sw ? b : a;
                g[i | bit] = sw ? a : b;
            }
    }
}
__device__ __forceinline__ CornerCoef make_coef_par(const SampleVal& v, float ds, float wk, const float dC[3],
                                                   const float dN[3], float ih) {
    CornerCoef k;
    const bool bx = v.bpar & 1u, by = v.bpar & 2u, bz = v.bpar & 4u;
    k.x1 = bx ? 1.f - v.fx : v.fx, k.x0 = bx ? v.fx : 1.f - v.fx;
    k.y1 = by ? 1.f - v.fy : v.fy, k.y0 = by ? v.fy : 1.f - v.fy;
    k.z1 = bz ? 1.f - v.fz : v.fz, k.z0 = bz ? v.fz : 1.f - v.fz;
    const float wn0 = (bx ? -wk : wk) * dN[0] * ih, wn1 = (by ? -wk : wk) * dN[1] * ih;
    k.wn2 = (bz ? -wk : wk) * dN[2] * ih;
    k.ax0 = fmaf(k.x0, ds, -wn0), k.ax1 = fmaf(k.x1, ds, wn0);
    k.bx0 = k.x0 * wn1, k.bx1 = k.x1 * wn1;
    k.wc0 = wk * dC[0], k.wc1 = wk * dC[1], k.wc2 = wk * dC[2];
    return k;
}
// red.global.add.v4.f32 under a predicate: the scatter has no divergent branches.
__device__ __forceinline__ void red_v4_if(float4* addr, float4 v, bool p) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n}" ::"l"(addr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(static_cast<uint32_t>(p))
        : "memory");
}

// Parity-p corner of the lane's two samples.  Runs: F (first, address `first`) and the last
// run (address `last`; the same run when !two).  A lane whose first run continues the
// previous lane's last run gives F away (`give`); the previous lane adds it (`recv`) to the
// atomic of its last run.  Every contribution is issued exactly once, by at most two
// predicated reductions per lane.
template <int p>
__device__ __forceinline__ void scatter_parity(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                               const CornerCoef& k0, const CornerCoef& k1, const XYPart& x0,
                                               const XYPart& x1, bool ok0, bool ok1, int lane) {
    const uint32_t a0k = v0.gidx[p], a1k = v1.gidx[p];  // kInvalid for an invalid sample
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    // an invalid sample's coefficients are zero (ds = w = 0, zeroed geometry), so its corner
    // gradients are zero without a select
    const float4 a0 = corner_grad<p>(k0, x0);
    const float4 a1 = corner_grad<p>(k1, x1);
    const bool two = ok0 && ok1 && a0k != a1k;
    const uint32_t first = ok0 ? a0k : a1k, last = ok1 ? a1k : a0k;
    const uint32_t prev_last = __shfl_up_sync(kFull, last, 1);
    const bool give = lane > 0 && first != kInvalid && first == prev_last;
    const bool recv = __shfl_down_sync(kFull, give ? 1u : 0u, 1) != 0u && lane < 31;
    const float4 F = two ? a0 : f4add(a0, a1);
    const float4 in = shfl_down4(F);  // lane l+1's first run (used only when recv)
    red_v4_if(grad + a0k, a0, two && !give);
    const float4 own = two ? a1 : (give ? z : F);
    red_v4_if(grad + last, recv ? f4add(own, in) : own, last != kInvalid && (two || !give || recv));
}
template <int q>
__device__ __forceinline__ void scatter_xy(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                           const CornerCoef& k0, const CornerCoef& k1, bool ok0, bool ok1, int lane) {
    const XYPart x0 = xy_part<q>(k0), x1 = xy_part<q>(k1);
    scatter_parity<q>(grad, v0, v1, k0, k1, x0, x1, ok0, ok1, lane);
    scatter_parity<q + 4>(grad, v0, v1, k0, k1, x0, x1, ok0, ok1, lane);
}
__device__ __forceinline__ void scatter_pair_par(float4* grad, const SampleVal& v0, const SampleVal& v1,
                                                 const CornerCoef& k0, const CornerCoef& k1, bool ok0, bool ok1,
                                                 int lane) {
    scatter_xy<0>(grad, v0, v1, k0, k1, ok0, ok1, lane);
    scatter_xy<1>(grad, v0, v1, k0, k1, ok0, ok1, lane);
    scatter_xy<2>(grad, v0, v1, k0, k1, ok0, ok1, lane);
    scatter_xy<3>(grad, v0, v1, k0, k1, ok0, ok1, lane);
}

// ---------------------------------------------------------------------------
// K6: backward.  Chunks of 64 samples are visited back to front; within a chunk the
// suffix S_k = sum_{m>k} w_m v_m comes from a warp suffix scan (no cancellation-prone
// "total minus prefix").  dL/dtau_k = T_{k+1} v_k - S_k, dL/ds_k = delta_k sigma' dL/dtau_k.
// The scatter is K6p's (scatter_pair_par: parity-keyed runs, predicated red.v4); without
// records the corner addresses are permuted into parity order first.
// ---------------------------------------------------------------------------
template <bool kRec>
__global__ void __launch_bounds__(256, 3) k_backward(GridView g, const double* __restrict__ O,
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
        const float P0 = tau_base + excl;
        // T_k = exp(-P_k); T_(k+1) = T_k e^(-tau_k) = T_k + T_k m_k with m_k = expm1(-tau_k),
        // w_k = -T_k m_k (one exp per lane; an invalid sample has tau = 0, m = 0)
        const float T0 = expf(-P0), m0 = expm1f(-tau0), m1 = expm1f(-tau1);
        const float Tn0 = fmaf(T0, m0, T0), Tn1 = fmaf(Tn0, m1, Tn0);
        const float w0 = ok0 ? -T0 * m0 : 0.f;
        const float w1 = ok1 ? -Tn0 * m1 : 0.f;
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
        const float ds0 = ok0 ? p.d0 * density_ds(v0.s, sg0, ib) * (Tn0 * vv0 - S0) : 0.f;
        const float ds1 = ok1 ? p.d1 * density_ds(v1.s, sg1, ib) * (Tn1 * vv1 - S1) : 0.f;
        touch_pair(g, v0, v1, ok0, ok1, lane);
        if (!kRec) {  // records give the parity order directly
            if (!ok0) zero_sample_bwd(v0);
            if (!ok1) zero_sample_bwd(v1);
            to_parity_order(v0);
            to_parity_order(v1);
        }
        const CornerCoef k0 = make_coef_par(v0, ds0, w0, dC, dN, ih);
        const CornerCoef k1 = make_coef_par(v1, ds1, w1, dC, dN, ih);
        scatter_pair_par(g.grad, v0, v1, k0, k1, ok0, ok1, lane);
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
constexpr int kStages = 2;  // one ray of look-ahead per warp
constexpr int kPipeWarps = 12;  // 2 CTAs of 12 warps per SM (80 registers): 1.73 vs 1.79 ms with 3 x 8

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

// The ray's scalars: origin / direction, upstream gradients and sample count, copied
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

__global__ void __launch_bounds__(kPipeWarps * 32, 2)
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
        for (int st = 0; st < kStages; ++st) mbar_init(bars + st, 33);
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
    auto issue_hdr = [&](uint64_t r, int st) {  // every lane: ray r's scalars + arrive
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
            const uint64_t r = ray_of(i);
            if (lane == 0) issue(r, st);
            issue_hdr(r, st);
        }
    }
    // the id of the next ray to stream, loaded one iteration before it is issued
    uint64_t pf_i = w0 + (kStages - 1) * warps_total;
    uint64_t r_pf = pf_i < n ? ray_of(pf_i) : 0;
    const float ih = static_cast<float>(g.inv_h);
    uint32_t phase = 0;  // bit st = parity of stage st
    int st = 0;
    for (uint64_t i = w0; i < n; i += warps_total) {
        {  // keep kStages-1 rays in flight: refill the stage released last iteration
            const uint64_t nxt = i + (kStages - 1) * warps_total;
            const int nst = (st + kStages - 1) % kStages;
            if (nxt < n) {
                if (lane == 0) issue(r_pf, nst);
                issue_hdr(r_pf, nst);
            }
            pf_i += warps_total;
            if (pf_i < n) r_pf = ray_of(pf_i);
        }
        mbar_wait(bars + st, (phase >> st) & 1u);
        phase ^= 1u << st;
        const PipeSlot& sl = slots[st];
        const PipeHdr& h = sl.hdr;
        const uint32_t cnt = h.cnt;
        const double* o = h.o;
        const double* d = h.d;
        float dC[3], dN[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) dC[a] = h.dC[a], dN[a] = h.dN[a];
        const float dD = h.dD;
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
            const float P0 = excl;
            // T_k = exp(-P_k); T_(k+1) = T_k e^(-tau_k) = T_k + T_k m_k with m_k = expm1(-tau_k),
            // w_k = -T_k m_k (one exp per lane; an invalid sample has tau = 0, m = 0)
            const float T0 = expf(-P0), m0 = expm1f(-tau0), m1 = expm1f(-tau1);
            const float Tn0 = fmaf(T0, m0, T0), Tn1 = fmaf(Tn0, m1, Tn0);
            const float w0 = ok0 ? -T0 * m0 : 0.f;
            const float w1 = ok1 ? -Tn0 * m1 : 0.f;
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
            const float ds0 = ok0 ? p.d0 * density_ds(v0.s, sg0, ib) * (Tn0 * vv0 - S0) : 0.f;
            const float ds1 = ok1 ? p.d1 * density_ds(v1.s, sg1, ib) * (Tn1 * vv1 - S1) : 0.f;
            touch_pair(g, v0, v1, ok0, ok1, lane);
            const CornerCoef c0 = make_coef_par(v0, ds0, w0, dC, dN, ih);
            const CornerCoef c1 = make_coef_par(v1, ds1, w1, dC, dN, ih);
            scatter_pair_par(g.grad, v0, v1, c0, c1, ok0, ok1, lane);
        }
        __syncwarp();  // every lane is done reading slot st before it is refilled
        st = (st + 1) % kStages;
    }
}

// Fold the backward's touch table into the active flags: (b, k) flagged -> blocks
// b + bits(c) for every c subset of k (the neighbour table), then clear the entry.
__global__ void __launch_bounds__(256) k_touch_expand(GridView g) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= g.n_blocks) return;
    uint2* t = reinterpret_cast<uint2*>(g.touch) + b;
    const uint2 v = *t;
    if (!(v.x | v.y)) return;
    uint32_t need = 0;  // bit c: the block of corner offset c is touched
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t byte = ((k < 4 ? v.x : v.y) >> (8 * (k & 3))) & 0xFFu;
        if (byte)
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (!(c & ~k)) need |= 1u << c;
    }
    g.active[b] = 1;
#pragma unroll
    for (int c = 1; c < 8; ++c)
        if (need & (1u << c)) {
            const uint32_t e = g.nbr[static_cast<size_t>(b) * 8 + c];
            if (e != kInvalid) g.active[e & ~kFullBit] = 1;
        }
    *t = make_uint2(0u, 0u);
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
                  double* delta, cudaStream_t s, uint32_t* pkeys, uint32_t* pids,
                  unsigned long long* valid_counter) {
    if (!n) return;
    k_march<<<grid_for(n, kMarchThreads), kMarchThreads, 0, s>>>(g, o, d, n, order, step, S, counts, t, delta,
                                                                 pkeys, pids, valid_counter);
}

void launch_render_forward(const GridView& g, const double* o, const double* d, uint64_t n,
                           const uint32_t* order, const uint32_t* counts, const double* t, uint32_t S,
                           double step, double beta, float* rgb, float* depth, float* normal,
                           float* wsum, unsigned long long* valid_counter, float4* rec, cudaStream_t s,
                           float4* zgrad, uint8_t* zactive, const uint32_t* zlist, const unsigned long long* zcount) {
    if (!n) return;
    const float ib = static_cast<float>(1.0 / beta);
    k_forward<<<grid_for(n * 32, kFwdThreads), kFwdThreads, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib, rgb,
                                                                    depth, normal, wsum, valid_counter, rec,
                                                                    ZeroRows{zgrad, zactive, zlist, zcount});
}

void launch_render_backward(const GridView& g, const double* o, const double* d, uint64_t n,
                            const uint32_t* order, const uint32_t* counts, const double* t,
                            uint32_t S, double step, double beta, const float* d_rgb,
                            const float* d_depth, const float* d_normal, const float4* rec,
                            cudaStream_t s) {
    if (!n) return;
    const float ib = static_cast<float>(1.0 / beta);
    const unsigned grid = grid_for(n * 32, 256);
    if (rec)
        k_backward<true><<<grid, 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib, d_rgb, d_depth, d_normal,
                                              rec);
    else
        k_backward<false><<<grid, 256, 0, s>>>(g, o, d, n, order, counts, t, S, step, ib, d_rgb, d_depth, d_normal,
                                               rec);
    if (g.n_blocks) k_touch_expand<<<grid_for(g.n_blocks, 256), 256, 0, s>>>(g);
}

bool launch_render_backward_pipe(const GridView& g, const double* o, const double* d, uint64_t n,
                                 const uint32_t* order, const uint32_t* counts, const double* t,
                                 uint32_t S, double step, double beta, const float* d_rgb,
                                 const float* d_depth, const float* d_normal, const float4* rec,
                                 cudaStream_t s, int num_sms) {
    if (!n) return true;
    if (!rec || S > 64 || (S & 1)) return false;
    const size_t smem = sizeof(PipeSlot) * kStages * kPipeWarps + 8 * kStages * kPipeWarps;
    const float ib = static_cast<float>(1.0 / beta);
    uint64_t ctas = static_cast<uint64_t>(num_sms) * 2;  // persistent: 2 CTAs of 12 warps per SM
    const uint64_t need = (n + kPipeWarps - 1) / kPipeWarps;
    if (ctas > need) ctas = need;
    const uint64_t warps_total = ctas * kPipeWarps;
    static bool attr_set = false;  // per process; the attribute is per function, not per device
    if (!attr_set) {
        SVR_LCK(cudaFuncSetAttribute(k_backward_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        attr_set = true;
    }
    k_backward_pipe<<<static_cast<unsigned>(ctas), kPipeWarps * 32, smem, s>>>(
        g, o, d, n, order, counts, t, S, step, ib, d_rgb, d_depth, d_normal, rec, warps_total);
    if (g.n_blocks) k_touch_expand<<<grid_for(g.n_blocks, 256), 256, 0, s>>>(g);
    return true;
}

void launch_ray_order(const double* o, const double* d, uint64_t n, const GridView& g, bool post_march,
                      uint32_t* keys, uint32_t* ids, uint32_t* keys_alt, uint32_t* ids_alt, void* tmp,
                      size_t tmp_bytes, uint32_t** sorted_ids, cudaStream_t s) {
    if (!n) return;
    // pre-march: origin + direction keys (24 bits); post-march: the march already wrote the
    // Morton key of each ray's first-sample block (3 x bits per axis of the block AABB; empty
    // rays carry all ones and sort last)
    int end_bit = 24;
    if (post_march) {
        int bits = 1;
        while (bits < 10 && ((1 << bits) < g.dim[0] || (1 << bits) < g.dim[1] || (1 << bits) < g.dim[2])) ++bits;
        end_bit = 3 * bits;
    } else {
        k_ray_keys_dir<<<grid_for(n, 256), 256, 0, s>>>(o, d, n, keys, ids);
    }
    cub::DoubleBuffer<uint32_t> kb(keys, keys_alt), vb(ids, ids_alt);
    size_t bytes = tmp_bytes;
    SVR_LCK(cub::DeviceRadixSort::SortPairs(tmp, bytes, kb, vb, static_cast<int>(n), 0, end_bit, s));
    *sorted_ids = vb.Current();
}

size_t ray_order_tmp_bytes(uint64_t n) {
    size_t bytes = 0;
    cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr), vb(nullptr, nullptr);
    SVR_LCK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, static_cast<int>(n), 0, 32));
    return bytes;
}

}  // namespace svr_internal
