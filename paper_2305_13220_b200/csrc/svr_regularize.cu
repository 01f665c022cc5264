// sm_100a kernels for the step around the rendering path:
//   K9  k_sample_uniform   -- points uniform over the allocated blocks (grid.cpp:355-370)
//   K10 k_eik_stats / k_eik_scatter -- Eikonal loss (PAPER Eq. 16/18) and
//       its analytic gradient through the trilinear weight derivatives, fp64 gather
//   K11 k_rmsprop          -- RMSProp on the active blocks, fused with zeroing the gradients
//       (the reference declares rms_* buffers, grid.hpp:70)
#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    return mix64(x);
}
__device__ __forceinline__ double unit53(unsigned long long x) {  // [0, 1)
    return static_cast<double>(x >> 11) * 0x1.0p-53;
}

__global__ void __launch_bounds__(256) k_sample_uniform(const int4* __restrict__ coords, uint32_t A,
                                                        double L, uint64_t n, unsigned long long seed,
                                                        double* out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long s = seed ^ (static_cast<unsigned long long>(i) * 0xD1B54A32D192ED03ull);
    const uint32_t b = static_cast<uint32_t>(__umul64hi(splitmix(s), static_cast<unsigned long long>(A)));
    const int4 c = coords[b];
    const int cc[3] = {c.x, c.y, c.z};
#pragma unroll
    for (int a = 0; a < 3; ++a)  // (c + unit) * L, grid.cpp:366-367
        out[3 * i + a] = __dmul_rn(__dadd_rn(static_cast<double>(cc[a]), unit53(splitmix(s + a + 1))), L);
}

__device__ __forceinline__ bool eik_eval(const GridView& g, const double* x, uint32_t gidx[8],
                                         double dw[8][3], double gr[3]) {
    double w[8];
    if (!gather_fp64(g, x, gidx, w, dw)) return false;
    gr[0] = gr[1] = gr[2] = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // sdf_gradient_impl order (grid.cpp:165-175)
        const double v = __ldg(g.pay + gidx[c]).x;
        gr[0] = __dadd_rn(gr[0], __dmul_rn(dw[c][0], v));
        gr[1] = __dadd_rn(gr[1], __dmul_rn(dw[c][1], v));
        gr[2] = __dadd_rn(gr[2], __dmul_rn(dw[c][2], v));
    }
    return true;
}

// pass 1: sum over valid points of (|g| - 1)^2 and the valid count
__global__ void __launch_bounds__(256) k_eik_stats(GridView g, const double* __restrict__ X, uint64_t n,
                                                   double* sums) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double l = 0.0, cnt = 0.0;
    if (i < n) {
        const double x[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
        uint32_t gidx[8];
        double dw[8][3], gr[3];
        if (eik_eval(g, x, gidx, dw, gr)) {
            const double nrm = sqrt(gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
            l = (nrm - 1.0) * (nrm - 1.0);
            cnt = 1.0;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        l += __shfl_xor_sync(kFull, l, off);
        cnt += __shfl_xor_sync(kFull, cnt, off);
    }
    if ((threadIdx.x & 31) == 0 && cnt > 0.0) {
        atomicAdd(sums, l);
        atomicAdd(sums + 1, cnt);
    }
}

// pass 2: dL/dtheta_c = coef (1 - 1/|g|) (g . dw_c), coef = 2 scale / n_valid
__global__ void __launch_bounds__(256) k_eik_scatter(GridView g, const double* __restrict__ X, uint64_t n,
                                                     double coef) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x[3] = {X[3 * i], X[3 * i + 1], X[3 * i + 2]};
    uint32_t gidx[8];
    double dw[8][3], gr[3];
    if (!eik_eval(g, x, gidx, dw, gr)) return;
    const double nrm = sqrt(gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]);
    if (!(nrm > 0.0)) return;  // direction undefined: zero subgradient
    const double k = coef * (1.0 - 1.0 / nrm);
    uint32_t prev = kInvalid;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double gs = k * (gr[0] * dw[c][0] + gr[1] * dw[c][1] + gr[2] * dw[c][2]);
        atomicAdd(&g.grad[gidx[c]].x, static_cast<float>(gs));
        const uint32_t blk = gidx[c] >> 9;
        if (blk != prev) {
            if (!g.active[blk]) g.active[blk] = 1;
            prev = blk;
        }
    }
}

// RMSProp on active blocks: one CTA of 128 threads per block (4 voxels each), grid-stride.
// The three planes are distinct allocations (__restrict__): all 12 loads of a thread's four
// voxels are issued before the first store.  (Skipping the payload of zero-gradient voxels
// was measured slower: the dependent load costs more than the bytes it saves.)
__global__ void __launch_bounds__(128) k_rmsprop(float4* __restrict__ pay, float4* __restrict__ grad,
                                                 float4* __restrict__ rms, uint8_t* __restrict__ active,
                                                 const uint32_t* __restrict__ list,
                                                 const unsigned long long* count, float lr, float alpha,
                                                 float eps) {
    const unsigned long long nb = *count;
    const float beta = 1.f - alpha;
    for (unsigned long long j = blockIdx.x; j < nb; j += gridDim.x) {
        const uint32_t b = list[j];
        float4 G[4], R[4], Pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const size_t v = static_cast<size_t>(b) * kVox + threadIdx.x + 128 * k;
            G[k] = __ldcs(grad + v);
            R[k] = __ldcs(rms + v);
            Pv[k] = __ldcs(pay + v);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const size_t v = static_cast<size_t>(b) * kVox + threadIdx.x + 128 * k;
            const float4 gv = G[k];
            float4 r = R[k], p = Pv[k];
            r.x = alpha * r.x + beta * gv.x * gv.x;
            r.y = alpha * r.y + beta * gv.y * gv.y;
            r.z = alpha * r.z + beta * gv.z * gv.z;
            r.w = alpha * r.w + beta * gv.w * gv.w;
            p.x -= lr * gv.x / (sqrtf(r.x) + eps);
            p.y -= lr * gv.y / (sqrtf(r.y) + eps);
            p.z -= lr * gv.z / (sqrtf(r.z) + eps);
            p.w -= lr * gv.w / (sqrtf(r.w) + eps);
            rms[v] = r;
            pay[v] = p;
            grad[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (threadIdx.x == 0) active[b] = 0;
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

void launch_sample_uniform(const int32_t* coords4, uint32_t A, double L, uint64_t n, uint64_t seed,
                           double* out, cudaStream_t s) {
    if (!n) return;
    k_sample_uniform<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const int4*>(coords4), A, L, n, seed, out);
}

void launch_eikonal_stats(const GridView& g, const double* x, uint64_t n, double* sums, cudaStream_t s) {
    if (!n) return;
    k_eik_stats<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(g, x, n, sums);
}

void launch_eikonal_scatter(const GridView& g, const double* x, uint64_t n, double coef, cudaStream_t s) {
    if (!n) return;
    k_eik_scatter<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(g, x, n, coef);
}

void launch_rmsprop(float4* pay, float4* grad, float4* rms, uint8_t* active, const uint32_t* list,
                    const unsigned long long* count, uint32_t n_max, float lr, float alpha, float eps,
                    cudaStream_t s) {
    if (!n_max) return;
    const unsigned cap = sm_count() * 16u;
    const unsigned grid = n_max < cap ? n_max : cap;
    k_rmsprop<<<grid, 128, 0, s>>>(pay, grad, rms, active, list, count, lr, alpha, eps);
}

}  // namespace svr_internal
