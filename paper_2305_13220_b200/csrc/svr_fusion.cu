// sm_100a kernels for the producer side of the rendering path:
//   K12  k_fuse          -- projective TSDF / color / logit fusion of a batch of frames into
//                           32.32 fixed-point running sums (PAPER Eq. 9-11)
//   K12f k_fuse_finalize -- means -> payload, unit-norm logits, weight = count, validity
//   K13  k_denoise       -- Gaussian over the (2r+1)^3 valid neighbourhood as num/den of two
//                           separable passes staged in shared memory
// The association rules and the operation order are restated in oracle/svr_oracle.cpp
// (the checker); every decision-making double op is an explicit _rn intrinsic so results
// are bit-identical to the oracle.
#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr double kFix = 4294967296.0;          // 2^32
constexpr double kInvFix = 1.0 / 4294967296.0;  // 2^-32
constexpr int kFuseThreads = 512;               // one voxel per thread

// round-to-nearest-even of v * 2^32 through the 1.5 * 2^52 shifter: one DADD + one integer
// subtract instead of an XU conversion; exact (== llrint) for |v| < 2^19, the input domain
// svr_fuse_frames documents.
__device__ __forceinline__ long long to_fix(double v) {
    const double t = __dadd_rn(__dmul_rn(v, kFix), 6755399441055744.0);
    return __double_as_longlong(t) - 0x4338000000000000LL;
}

// Conservative per-(block, frame) cull: the block's voxel centres span the box
// [c*8, c*8+7] * h.  bit0: corner surely behind the camera (z < -1e-6); bit5: corner not
// safely in front (z < 1e-3); bits1-4: corner beyond an image edge by > 1 px.  Perspective
// projection maps a box wholly in front of the camera into the hull of its projected
// corners, so the block is skipped when every corner is behind, or when every corner is
// safely in front and beyond the same edge.  Everything else runs the exact per-voxel test.
__device__ __forceinline__ unsigned corner_flags(const svr_camera& c, const double x[3]) {
    const double d[3] = {x[0] - c.t[0], x[1] - c.t[1], x[2] - c.t[2]};
    double xc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) xc[r] = c.R[r] * d[0] + c.R[3 + r] * d[1] + c.R[6 + r] * d[2];
    if (xc[2] < 1e-3) return 32u | (xc[2] < -1e-6 ? 1u : 0u);
    const double u = c.fx * xc[0] / xc[2] + c.cx, v = c.fy * xc[1] / xc[2] + c.cy;
    return (u < -1.0 ? 2u : 0u) | (u > c.width ? 4u : 0u) | (v < -1.0 ? 8u : 0u) |
           (v > c.height ? 16u : 0u);
}

struct FuseArgs {
    const int4* coords;
    const svr_camera* cams;
    uint32_t n_frames;
    int32_t W, H, C;
    const float* depth;
    const float* rgb;
    const float* sem;
    const double* scales;
    int32_t rows, cols;
    double h, mu;
    long long* fsum;  // [A][4 + C][512]
    uint32_t* fcount;  // [A][512]
    unsigned long long* counters;  // in_view, rejected
};

// One CTA of 512 threads per block (one voxel per thread), the frame batch looped inside so
// the running sums live in registers for the whole launch (KC > 0: the C logit sums too;
// KC <= 0: logit sums read-modify-written in HBM, each voxel owned by one thread).  Frames
// are taken 64 at a time: one pass evaluates the block-vs-frame cull for all 64 (thread =
// frame * 8 + corner), then the CTA walks only the visible frames without further barriers.
template <int KC>
__global__ void __launch_bounds__(kFuseThreads) k_fuse(FuseArgs a) {
    __shared__ unsigned s_vis[kFuseThreads / 32];
    const uint32_t b = blockIdx.x;
    const int4 bc = a.coords[b];
    const int K = 4 + a.C;
    constexpr int KR = KC > 0 ? KC : 1;
    const int v = threadIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long* base = a.fsum + static_cast<size_t>(b) * K * kVox;
    long long acc[4];
    long long lacc[KR];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] = base[k * kVox + v];
    if (KC > 0) {
#pragma unroll
        for (int k = 0; k < KR; ++k) lacc[k] = base[(4 + k) * kVox + v];
    }
    uint32_t cnt = a.fcount[static_cast<size_t>(b) * kVox + v];
    // voxel_to_world (grid.hpp:124-126)
    const double x0 = __dmul_rn(static_cast<double>(bc.x * kRes + (v & 7)), a.h);
    const double x1 = __dmul_rn(static_cast<double>(bc.y * kRes + ((v >> 3) & 7)), a.h);
    const double x2 = __dmul_rn(static_cast<double>(bc.z * kRes + (v >> 6)), a.h);
    unsigned long long in_view = 0, rejected = 0;
    const size_t npx = static_cast<size_t>(a.W) * a.H;
    for (uint32_t f0 = 0; f0 < a.n_frames; f0 += 64) {
        const uint32_t nf = min(64u, a.n_frames - f0);
        {
            const uint32_t fr = threadIdx.x >> 3;
            const int cc = threadIdx.x & 7;
            unsigned fl = 63u;
            if (fr < nf) {
                const double cx[3] = {(bc.x * kRes + 7.0 * (cc & 1)) * a.h,
                                      (bc.y * kRes + 7.0 * ((cc >> 1) & 1)) * a.h,
                                      (bc.z * kRes + 7.0 * (cc >> 2)) * a.h};
                fl = corner_flags(a.cams[f0 + fr], cx);
            }
            unsigned all = fl, any_near = fl & 32u;
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                all &= __shfl_xor_sync(kFull, all, off);
                any_near |= __shfl_xor_sync(kFull, any_near, off);
            }
            const bool vis = fr < nf && !((all & 1u) || (!any_near && (all & 30u)));
            const unsigned bal = __ballot_sync(kFull, vis && cc == 0);  // bits 0, 8, 16, 24
            if (lane == 0)
                s_vis[warp] = (bal & 1u) | ((bal >> 7) & 2u) | ((bal >> 14) & 4u) | ((bal >> 21) & 8u);
        }
        __syncthreads();
        unsigned long long mask = 0;
#pragma unroll
        for (int w = 0; w < 16; ++w) mask |= static_cast<unsigned long long>(s_vis[w]) << (4 * w);
        __syncthreads();
        while (mask) {
            const uint32_t f = f0 + __ffsll(static_cast<long long>(mask)) - 1;
            mask &= mask - 1;
            const svr_camera& c = a.cams[f];
            // Camera::project (camera.cpp:7-18): x_c = R^T (x - t), accumulated left to right
            const double d0 = __dsub_rn(x0, c.t[0]), d1 = __dsub_rn(x1, c.t[1]), d2 = __dsub_rn(x2, c.t[2]);
            double xc[3];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                xc[r] = __dadd_rn(__dadd_rn(__dmul_rn(c.R[r], d0), __dmul_rn(c.R[3 + r], d1)),
                                  __dmul_rn(c.R[6 + r], d2));
            if (xc[2] <= 1e-6) continue;
            const double px = __dadd_rn(__ddiv_rn(__dmul_rn(c.fx, xc[0]), xc[2]), c.cx);
            const double py = __dadd_rn(__ddiv_rn(__dmul_rn(c.fy, xc[1]), xc[2]), c.cy);
            if (!(px >= 0.0 && px <= static_cast<double>(a.W - 1) && py >= 0.0 &&
                  py <= static_cast<double>(a.H - 1)))
                continue;
            const int ix = static_cast<int>(floor(__dadd_rn(px, 0.5)));
            const int iy = static_cast<int>(floor(__dadd_rn(py, 0.5)));
            const size_t pix = static_cast<size_t>(iy) * a.W + ix;
            const size_t gp = f * npx + pix;
            const float D = __ldg(a.depth + gp);
            if (!(D > 0.0f)) continue;
            double phi = 1.0;
            if (a.scales) {
                phi = scale_field_value(a.scales + static_cast<size_t>(f) * a.rows * a.cols, a.rows, a.cols,
                                        a.W, a.H, ix, iy);
                if (!(phi > 0.0)) continue;
            }
            ++in_view;
            const double sd = __dsub_rn(__dmul_rn(static_cast<double>(D), phi), xc[2]);
            if (sd < -a.mu) {
                ++rejected;
                continue;
            }
            acc[0] += to_fix(smin(sd, a.mu));
            if (a.rgb) {
#pragma unroll
                for (int k = 0; k < 3; ++k) acc[1 + k] += to_fix(static_cast<double>(__ldg(a.rgb + 3 * gp + k)));
            }
            if (a.sem) {
                const float* sp = a.sem + static_cast<size_t>(a.C) * gp;
                if (KC > 0) {
#pragma unroll
                    for (int k = 0; k < KR; ++k) lacc[k] += to_fix(static_cast<double>(__ldg(sp + k)));
                } else {
                    for (int k = 0; k < a.C; ++k) base[(4 + k) * kVox + v] += to_fix(static_cast<double>(__ldg(sp + k)));
                }
            }
            ++cnt;
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) base[k * kVox + v] = acc[k];
    if (KC > 0) {
#pragma unroll
        for (int k = 0; k < KR; ++k) base[(4 + k) * kVox + v] = lacc[k];
    }
    a.fcount[static_cast<size_t>(b) * kVox + v] = cnt;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        in_view += __shfl_xor_sync(kFull, in_view, off);
        rejected += __shfl_xor_sync(kFull, rejected, off);
    }
    if (lane == 0 && in_view) {
        atomicAdd(a.counters, in_view);
        if (rejected) atomicAdd(a.counters + 1, rejected);
    }
}

// Means -> payload (one CTA of 512 threads per block).  Voxels never associated keep their
// payload and get weight 0 (invalid); the validity mask / all-valid bit are rebuilt.
__global__ void __launch_bounds__(512) k_fuse_finalize(const long long* __restrict__ fsum,
                                                       const uint32_t* __restrict__ fcount, int32_t C,
                                                       int flags, float4* pay, float* weight, float* logits,
                                                       uint32_t* vmask, uint32_t* meta) {
    const uint32_t b = blockIdx.x, v = threadIdx.x;
    const size_t i = static_cast<size_t>(b) * kVox + v;
    const int K = 4 + C;
    const long long* s = fsum + static_cast<size_t>(b) * K * kVox + v;
    const uint32_t n = fcount[i];
    weight[i] = static_cast<float>(n);
    if (n) {
        const double dn = static_cast<double>(n);
        float4 p = pay[i];
        p.x = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(s[0]), kInvFix), dn));
        if (flags & 1) {
            p.y = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(s[kVox]), kInvFix), dn));
            p.z = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(s[2 * kVox]), kInvFix), dn));
            p.w = __double2float_rn(__ddiv_rn(__dmul_rn(static_cast<double>(s[3 * kVox]), kInvFix), dn));
        }
        pay[i] = p;
        if (flags & 2) {  // Eq. 11: s* / ||s*||
            double n2 = 0.0;
            for (int k = 0; k < C; ++k) {
                const double m = __ddiv_rn(__dmul_rn(static_cast<double>(s[(4 + k) * kVox]), kInvFix), dn);
                n2 = __dadd_rn(n2, __dmul_rn(m, m));
            }
            const double nrm = __dsqrt_rn(n2);
            for (int k = 0; k < C; ++k) {
                const double m = __ddiv_rn(__dmul_rn(static_cast<double>(s[(4 + k) * kVox]), kInvFix), dn);
                logits[i * C + k] = nrm > 0.0 ? __double2float_rn(__ddiv_rn(m, nrm)) : 0.0f;
            }
        }
    }
    const unsigned bits = __ballot_sync(kFull, n > 0);  // grid.hpp:57-58: valid iff weight > 0
    __shared__ unsigned words[16];
    if ((v & 31) == 0) {
        words[v >> 5] = bits;
        vmask[static_cast<size_t>(b) * 16 + (v >> 5)] = bits;
    }
    __syncthreads();
    if (v == 0) {
        unsigned all = kFull;
        for (int k = 0; k < 16; ++k) all &= words[k];
        meta[b] = all == kFull ? 1u : 0u;
    }
}

// ---------------------------------------------------------------------------------------
// K13 de-noising.  For a valid centre voxel c and each property p:
//   num = sum_dz g[dz] * sum_dy g[dy] * sum_dx g[dx] * (valid(u) ? p(u) : 0)
//   den = the same with p = 1;  p'(c) = float(num / den)
// Each sum runs from the most negative offset, starting at 0.0, in fp64 (the oracle's
// loop order).  The inner sums are shared between centres: pass X produces them for every
// halo row, pass Y for every halo plane, pass Z finishes each centre.
// ---------------------------------------------------------------------------------------
struct DenoiseArgs {
    GridView g;
    const int4* coords;
    float4* pay_out;
    float* logits_out;
    int32_t r;
    double gw[9];
};

constexpr int kDnThreads = 256;

__host__ __device__ constexpr size_t denoise_smem_bytes(int r) {
    // halo float4 + valid u8 (padded) + pass X (5 doubles per row sample) + pass Y
    return static_cast<size_t>((8 + 2 * r) * (8 + 2 * r) * (8 + 2 * r)) * 17 + 16 +
           static_cast<size_t>((8 + 2 * r) * (8 + 2 * r) * 8) * 40 + static_cast<size_t>((8 + 2 * r) * 64) * 40;
}

// The radius is a template parameter (0..4, the Gaussian table holds 2r + 1 <= 9 taps): the
// halo extent S is a compile-time constant, so the halo index arithmetic (div / mod by S)
// becomes multiply-shift and every tap loop unrolls.
template <int kR>
__global__ void __launch_bounds__(kDnThreads) k_denoise(DenoiseArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_nb[27];
    __shared__ double s_gw[9];
    constexpr int r = kR, S = 8 + 2 * r, S3 = S * S * S, NX = S * S * 8, NY = S * 64;
    float4* halo = reinterpret_cast<float4*>(smem);
    unsigned char* hval = smem + static_cast<size_t>(S3) * 16;
    double* tx = reinterpret_cast<double*>(smem + ((static_cast<size_t>(S3) * 17 + 15) & ~size_t(15)));
    double* ty = tx + static_cast<size_t>(NX) * 5;
    const uint32_t b = blockIdx.x;
    const int4 bc = a.coords[b];
    if (threadIdx.x < 27) {
        const int t = threadIdx.x;
        s_nb[t] = lookup_block(a.g, bc.x + t % 3 - 1, bc.y + (t / 3) % 3 - 1, bc.z + t / 9 - 1);
        if (t <= 2 * r) s_gw[t] = a.gw[t];
    }
    __syncthreads();
    // centre validity + den, kept per owned output voxel across the channel groups
    double den[2];
    const int C = a.g.C, groups = 1 + (C + 3) / 4;
    for (int grp = 0; grp < groups; ++grp) {
        // stage the halo of this channel group: group 0 = (sdf, r, g, b), group k = logits 4k-4..
        // 16 B channel groups go global -> shared with cp.async (zero-filled for a missing
        // block), so no load round-trips through registers; the validity bit is applied
        // where the halo is read (pass X)
        const bool vec = grp == 0 || (C & 3) == 0;
        for (int i = threadIdx.x; i < S3; i += kDnThreads) {
            const int hx = i % S - r, hy = (i / S) % S - r, hz = i / (S * S) - r;
            const int nbi = ((hx >> 3) + 1) + 3 * ((hy >> 3) + 1) + 9 * ((hz >> 3) + 1);
            const uint32_t e = s_nb[nbi];
            const uint32_t local = (hx & 7) + 8 * (hy & 7) + 64 * (hz & 7);
            if (vec) {
                const bool blk = e != kInvalid;
                const size_t gi = blk ? static_cast<size_t>(e & ~kFullBit) * kVox + local : 0;
                const void* src = grp == 0 ? static_cast<const void*>(a.g.pay + gi)
                                           : static_cast<const void*>(a.g.logits + gi * C + 4 * (grp - 1));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                                 static_cast<uint32_t>(__cvta_generic_to_shared(halo + i))),
                             "l"(src), "r"(blk ? 16u : 0u)
                             : "memory");
                if (grp == 0) hval[i] = blk && voxel_valid(a.g, e, local);
                continue;
            }
            const bool ok = e != kInvalid && voxel_valid(a.g, e, local);
            float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) {
                const size_t gi = static_cast<size_t>(e & ~kFullBit) * kVox + local;
                if (grp == 0) {
                    val = __ldg(a.g.pay + gi);
                } else {
                    const int k0 = 4 * (grp - 1);
                    const float* lp = a.g.logits + gi * C + k0;
                    if ((C & 3) == 0) {  // 16 B aligned: one vector load
                        val = __ldg(reinterpret_cast<const float4*>(lp));
                    } else {
                        val.x = __ldg(lp);
                        if (k0 + 1 < C) val.y = __ldg(lp + 1);
                        if (k0 + 2 < C) val.z = __ldg(lp + 2);
                        if (k0 + 3 < C) val.w = __ldg(lp + 3);
                    }
                }
            }
            halo[i] = val;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // pass X: rows (hz, hy) over the halo, x in [0, 8)
        for (int i = threadIdx.x; i < NX; i += kDnThreads) {
            const int x = i & 7, row = i >> 3;  // row = hz * S + hy
            double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0, dd = 0.0;
            for (int dx = 0; dx <= 2 * r; ++dx) {
                const int hi = row * S + x + dx;
                const double w = s_gw[dx];
                const bool hv = hval[hi];
                const float4 hr = halo[hi];
                const float4 v = hv ? hr : make_float4(0.f, 0.f, 0.f, 0.f);  // unobserved: zero
                n0 = __dadd_rn(n0, __dmul_rn(w, static_cast<double>(v.x)));
                n1 = __dadd_rn(n1, __dmul_rn(w, static_cast<double>(v.y)));
                n2 = __dadd_rn(n2, __dmul_rn(w, static_cast<double>(v.z)));
                n3 = __dadd_rn(n3, __dmul_rn(w, static_cast<double>(v.w)));
                if (grp == 0) dd = __dadd_rn(dd, __dmul_rn(w, hv ? 1.0 : 0.0));
            }
            tx[i] = n0, tx[NX + i] = n1, tx[2 * NX + i] = n2, tx[3 * NX + i] = n3;
            if (grp == 0) tx[4 * NX + i] = dd;  // the denominator: group 0 only
        }
        __syncthreads();
        // pass Y: planes hz, (y, x) in [0, 8)^2
        for (int i = threadIdx.x; i < NY; i += kDnThreads) {
            const int x = i & 7, y = (i >> 3) & 7, hz = i >> 6;
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            for (int dy = 0; dy <= 2 * r; ++dy) {
                const int ti = (hz * S + y + dy) * 8 + x;
                const double w = s_gw[dy];
#pragma unroll
                for (int k = 0; k < 5; ++k)
                    if (k < 4 || grp == 0) acc[k] = __dadd_rn(acc[k], __dmul_rn(w, tx[k * NX + ti]));
            }
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if (k < 4 || grp == 0) ty[k * NY + i] = acc[k];
        }
        __syncthreads();
        // pass Z + output
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int v = threadIdx.x + j * kDnThreads;
            const int x = v & 7, y = (v >> 3) & 7, z = v >> 6;
            double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            for (int dz = 0; dz <= 2 * r; ++dz) {
                const int ti = ((z + dz) * 8 + y) * 8 + x;
                const double w = s_gw[dz];
#pragma unroll
                for (int k = 0; k < 5; ++k)
                    if (k < 4 || grp == 0) acc[k] = __dadd_rn(acc[k], __dmul_rn(w, ty[k * NY + ti]));
            }
            if (grp == 0) den[j] = acc[4];
            const int hc = ((z + r) * S + y + r) * S + x + r;
            const bool centre = hval[hc];
            const size_t gi = static_cast<size_t>(b) * kVox + v;
            if (grp == 0) {
                float4 o = __ldg(a.g.pay + gi);
                if (centre) {
                    o.x = __double2float_rn(__ddiv_rn(acc[0], den[j]));
                    o.y = __double2float_rn(__ddiv_rn(acc[1], den[j]));
                    o.z = __double2float_rn(__ddiv_rn(acc[2], den[j]));
                    o.w = __double2float_rn(__ddiv_rn(acc[3], den[j]));
                }
                a.pay_out[gi] = o;
            } else {
                const int k0 = 4 * (grp - 1);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k0 + k >= C) break;
                    const size_t li = gi * C + k0 + k;
                    a.logits_out[li] = centre ? __double2float_rn(__ddiv_rn(acc[k], den[j])) : __ldg(a.g.logits + li);
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

void launch_fuse(const int32_t* coords4, uint32_t n_blocks, const svr_camera* cams, uint32_t n_frames,
                 int32_t W, int32_t H, int32_t C, const float* depth, const float* rgb, const float* sem,
                 const double* scales, int32_t rows, int32_t cols, double h, double mu, long long* fsum,
                 uint32_t* fcount, unsigned long long* counters, cudaStream_t s) {
    if (!n_blocks || !n_frames) return;
    FuseArgs a{reinterpret_cast<const int4*>(coords4), cams, n_frames, W, H, C, depth, rgb, sem, scales,
               rows, cols, h, mu, fsum, fcount, counters};
    switch (sem ? C : 0) {
#define SVR_FUSE_CASE(k) \
    case k:              \
        k_fuse<k><<<n_blocks, kFuseThreads, 0, s>>>(a); \
        break;
        SVR_FUSE_CASE(0)
        SVR_FUSE_CASE(1)
        SVR_FUSE_CASE(2)
        SVR_FUSE_CASE(3)
        SVR_FUSE_CASE(4)
        SVR_FUSE_CASE(5)
        SVR_FUSE_CASE(6)
        SVR_FUSE_CASE(7)
        SVR_FUSE_CASE(8)
#undef SVR_FUSE_CASE
        default:
            k_fuse<-1><<<n_blocks, kFuseThreads, 0, s>>>(a);
    }
}

void launch_fuse_finalize(const long long* fsum, const uint32_t* fcount, uint32_t n_blocks, int32_t C,
                          int flags, float4* pay, float* weight, float* logits, uint32_t* vmask,
                          uint32_t* meta, cudaStream_t s) {
    if (!n_blocks) return;
    k_fuse_finalize<<<n_blocks, 512, 0, s>>>(fsum, fcount, C, flags, pay, weight, logits, vmask, meta);
}

size_t denoise_smem(int radius) { return denoise_smem_bytes(radius); }

void launch_denoise(const GridView& g, const int32_t* coords4, float4* pay_out, float* logits_out,
                    int32_t radius, const double* gw, cudaStream_t s) {
    if (!g.n_blocks) return;
    DenoiseArgs a{};
    a.g = g;
    a.coords = reinterpret_cast<const int4*>(coords4);
    a.pay_out = pay_out;
    a.logits_out = logits_out;
    a.r = radius;
    for (int i = 0; i <= 2 * radius; ++i) a.gw[i] = gw[i];
    const size_t smem = denoise_smem_bytes(radius);
#define SVR_DN(R)                                                                                       \
    SVR_LCK(cudaFuncSetAttribute(k_denoise<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem))); \
    k_denoise<R><<<g.n_blocks, kDnThreads, smem, s>>>(a)
    switch (radius) {
        case 0: SVR_DN(0); break;
        case 1: SVR_DN(1); break;
        case 2: SVR_DN(2); break;
        case 3: SVR_DN(3); break;
        default: SVR_DN(4); break;
    }
#undef SVR_DN
}

}  // namespace svr_internal
