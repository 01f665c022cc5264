// sm_100a refinement losses (SPEC.md:286-319 backward_step, PAPER Eq. 12-14 / 23): the
// per-ray upstream gradients render_backward consumes, from the rendered colour / depth /
// normal of the last forward and the frame targets.  Restated in oracle/svr_oracle.cpp
// (svro_render_losses) with the same decisions:
//   participating ray: wsum > 0;  L_c = mean sum_ch |C - C*|
//   L_d = mean (t - (a D + b))^2 over D > 0, (a, b) least squares over the batch (fp64
//         normal equations; singular or < 2 rays: a = 1, b = mean(t - D))
//   L_n = mean |normalize(R^T N) - n*|_1 over |n*| > 0 and |R^T N| > 1e-12
//   K15a k_loss_sums -> K15f k_loss_fit (one thread) -> K15b k_loss_grad
#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

struct LossArgs {
    uint64_t n;
    const float *rgb, *depth, *normal, *wsum;
    const float *tgt, *pdepth, *pnormal;
    const uint32_t* cam_idx;
    const svr_camera* cams;
    double lambda_d, lambda_n;
    float *d_rgb, *d_depth, *d_normal;
    double* acc;  // [0..4] depth sums, [5] n_c, [6] n_n, [7] a, [8] b, [9] singular,
                  // [10] sum |dC|, [11] sum r^2, [12] sum |dn|
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// camera-frame normal R^T N and its length; false when the normal term does not apply
__device__ __forceinline__ bool cam_normal(const LossArgs& a, uint64_t i, double nc[3], double& len) {
    if (!a.pnormal) return false;
    const float p0 = a.pnormal[3 * i], p1 = a.pnormal[3 * i + 1], p2 = a.pnormal[3 * i + 2];
    if (!(p0 != 0.f || p1 != 0.f || p2 != 0.f)) return false;
    const double* R = a.cams[a.cam_idx[i]].R;
    const double N[3] = {a.normal[3 * i], a.normal[3 * i + 1], a.normal[3 * i + 2]};
#pragma unroll
    for (int r = 0; r < 3; ++r)
        nc[r] = __dadd_rn(__dadd_rn(__dmul_rn(R[r], N[0]), __dmul_rn(R[3 + r], N[1])), __dmul_rn(R[6 + r], N[2]));
    len = sqrt(nc[0] * nc[0] + nc[1] * nc[1] + nc[2] * nc[2]);
    return len > 1e-12;
}

__global__ void __launch_bounds__(256) k_loss_sums(LossArgs a) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double s[7] = {0, 0, 0, 0, 0, 0, 0};
    if (i < a.n && a.wsum[i] > 0.f) {
        s[5] = 1.0;
        if (a.pdepth && a.pdepth[i] > 0.f) {
            const double D = a.pdepth[i], t = a.depth[i];
            s[0] = 1.0, s[1] = D, s[2] = D * D, s[3] = t, s[4] = D * t;
        }
        double nc[3], len;
        if (cam_normal(a, i, nc, len)) s[6] = 1.0;
    }
#pragma unroll
    for (int k = 0; k < 7; ++k) s[k] = warp_sum_d(s[k]);
    if ((threadIdx.x & 31) == 0 && s[5] > 0.0)
#pragma unroll
        for (int k = 0; k < 7; ++k)
            if (s[k] != 0.0) atomicAdd(a.acc + k, s[k]);
}

__global__ void k_loss_fit(double* acc) {  // depth_fit of svr_oracle.cpp
    const double* S = acc;
    const double det = S[0] * S[2] - S[1] * S[1];
    const bool singular = !(S[0] >= 2.0) || !(det > 1e-12 * S[0] * S[2]);
    double a, b;
    if (singular) {
        a = 1.0;
        b = S[0] > 0.0 ? (S[3] - S[1]) / S[0] : 0.0;
    } else {
        a = (S[0] * S[4] - S[1] * S[3]) / det;
        b = (S[3] - a * S[1]) / S[0];
    }
    acc[7] = a, acc[8] = b, acc[9] = singular ? 1.0 : 0.0;
}

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

__global__ void __launch_bounds__(256) k_loss_grad(LossArgs a) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double lc = 0.0, ld = 0.0, ln = 0.0;
    if (i < a.n) {
        const double nc_rays = a.acc[5], nd = a.acc[0], nn = a.acc[6];
        double gc[3] = {0, 0, 0}, gn[3] = {0, 0, 0}, gd = 0.0;
        if (a.wsum[i] > 0.f) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double e = static_cast<double>(a.rgb[3 * i + k]) - a.tgt[3 * i + k];
                lc += fabs(e);
                gc[k] = sgn(e) / nc_rays;
            }
            if (a.pdepth && a.pdepth[i] > 0.f) {
                const double r = static_cast<double>(a.depth[i]) - (a.acc[7] * a.pdepth[i] + a.acc[8]);
                ld = r * r;
                gd = a.lambda_d * 2.0 * r / nd;
            }
            double c[3], len;
            if (cam_normal(a, i, c, len)) {
                const double nh[3] = {c[0] / len, c[1] / len, c[2] / len};
                double sg[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double e = nh[k] - a.pnormal[3 * i + k];
                    ln += fabs(e);
                    sg[k] = sgn(e);
                }
                const double dot = nh[0] * sg[0] + nh[1] * sg[1] + nh[2] * sg[2];
                double gcam[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) gcam[k] = (sg[k] - nh[k] * dot) / len * (a.lambda_n / nn);
                const double* R = a.cams[a.cam_idx[i]].R;
#pragma unroll
                for (int r = 0; r < 3; ++r) gn[r] = R[3 * r] * gcam[0] + R[3 * r + 1] * gcam[1] + R[3 * r + 2] * gcam[2];
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a.d_rgb[3 * i + k] = static_cast<float>(gc[k]);
            a.d_normal[3 * i + k] = static_cast<float>(gn[k]);
        }
        a.d_depth[i] = static_cast<float>(gd);
    }
    lc = warp_sum_d(lc), ld = warp_sum_d(ld), ln = warp_sum_d(ln);
    if ((threadIdx.x & 31) == 0) {
        if (lc != 0.0) atomicAdd(a.acc + 10, lc);
        if (ld != 0.0) atomicAdd(a.acc + 11, ld);
        if (ln != 0.0) atomicAdd(a.acc + 12, ln);
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

void launch_render_losses(uint64_t n, const float* rgb, const float* depth, const float* normal,
                          const float* wsum, const float* tgt, const float* pdepth, const float* pnormal,
                          const uint32_t* cam_idx, const svr_camera* cams, double lambda_d, double lambda_n,
                          float* d_rgb, float* d_depth, float* d_normal, double* acc, cudaStream_t s) {
    SVR_LCK(cudaMemsetAsync(acc, 0, 16 * sizeof(double), s));
    if (!n) return;
    LossArgs a{n, rgb, depth, normal, wsum, tgt, pdepth, pnormal, cam_idx, cams, lambda_d, lambda_n,
               d_rgb, d_depth, d_normal, acc};
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    k_loss_sums<<<grid, 256, 0, s>>>(a);
    k_loss_fit<<<1, 1, 0, s>>>(acc);
    k_loss_grad<<<grid, 256, 0, s>>>(a);
}

}  // namespace svr_internal
