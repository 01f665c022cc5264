// sm_100a pieces of the refinement loop around the rendering path:
//   K17 k_sample_frame_rays -- a training batch straight from device-resident frames: per
//        image slot a random frame, per ray a random pixel (counter-based splitmix64), the
//        ray of Camera::ray_direction (camera.cpp:27-30, fp64, reference order) and the
//        pixel's colour / prior depth / prior normal targets
//   K16 k_band_count / k_band_write -- sample_eikonal_points part (a): the samples of the
//        last forward whose sdf is inside the surface band, in (ray, sample) order
#include <cub/device/device_scan.cuh>

#include "svr_internal.h"

namespace svr_dev {
namespace {

__device__ __forceinline__ unsigned long long smix(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    return mix64(x);
}

struct RayBatchArgs {
    const svr_camera* cams;
    uint32_t n_frames;
    int32_t W, H;
    uint32_t rays_per_image;
    uint64_t n;
    unsigned long long seed;
    const float *rgb_img, *depth_img, *normal_img;
    double *o, *d;
    float *tgt, *pdepth, *pnormal;
    uint32_t *cam_idx, *pixel;
};

__global__ void __launch_bounds__(256) k_sample_frame_rays(RayBatchArgs a) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const uint64_t slot = i / a.rays_per_image;
    const uint32_t f = static_cast<uint32_t>(
        __umul64hi(smix(a.seed ^ ((slot + 1) * 0xD1B54A32D192ED03ull)), static_cast<unsigned long long>(a.n_frames)));
    const uint64_t npx = static_cast<uint64_t>(a.W) * a.H;
    const uint64_t p = __umul64hi(smix((a.seed + 0x632BE59BD9B4E019ull) ^ ((i + 1) * 0x9E3779B97F4A7C15ull)),
                                  static_cast<unsigned long long>(npx));
    const int32_t x = static_cast<int32_t>(p % a.W), y = static_cast<int32_t>(p / a.W);
    const svr_camera& c = a.cams[f];
    // Camera::ray_direction: (R ((x - cx) / fx, (y - cy) / fy, 1)).normalized()
    const double dc[3] = {__ddiv_rn(__dsub_rn(static_cast<double>(x), c.cx), c.fx),
                          __ddiv_rn(__dsub_rn(static_cast<double>(y), c.cy), c.fy), 1.0};
    double rd[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
        rd[r] = __dadd_rn(__dadd_rn(__dmul_rn(c.R[3 * r], dc[0]), __dmul_rn(c.R[3 * r + 1], dc[1])),
                          __dmul_rn(c.R[3 * r + 2], dc[2]));
    const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(rd[0], rd[0]), __dmul_rn(rd[1], rd[1])),
                                            __dmul_rn(rd[2], rd[2])));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a.o[3 * i + k] = c.t[k];
        a.d[3 * i + k] = __ddiv_rn(rd[k], nrm);
    }
    const uint64_t px = static_cast<uint64_t>(f) * npx + p;
    if (a.tgt)
#pragma unroll
        for (int k = 0; k < 3; ++k) a.tgt[3 * i + k] = a.rgb_img[3 * px + k];
    if (a.pdepth) a.pdepth[i] = a.depth_img ? a.depth_img[px] : 0.f;
    if (a.pnormal)
#pragma unroll
        for (int k = 0; k < 3; ++k) a.pnormal[3 * i + k] = a.normal_img ? a.normal_img[3 * px + k] : 0.f;
    if (a.cam_idx) a.cam_idx[i] = f;
    if (a.pixel) a.pixel[i] = static_cast<uint32_t>(px);
}

// |sdf| < band per sample of the retained forward (records hold the fp32 interpolated sdf)
// Warp per ray, lane per sample (coalesced record reads); the band flags of 32 samples are
// counted / placed with one ballot, so the points keep (ray, sample) order.
__device__ __forceinline__ bool band_flag(const float4* __restrict__ rec, uint64_t r, uint32_t S, uint32_t k,
                                          uint32_t cnt, float band) {
    if (k >= cnt) return false;
    const float* q = reinterpret_cast<const float*>(rec + (r * S + k) * 2);
    return __float_as_uint(__ldg(q + 7)) != kInvalid && fabsf(__ldg(q)) < band;  // entry, sdf
}

__global__ void __launch_bounds__(256) k_band_count(const uint32_t* __restrict__ counts, const float4* __restrict__ rec,
                                                    uint64_t n, uint32_t S, float band, uint32_t* out) {
    const uint64_t r = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= n) return;
    const uint32_t cnt = counts[r];
    uint32_t m = 0;
    for (uint32_t base = 0; base < cnt; base += 32)
        m += __popc(__ballot_sync(0xFFFFFFFFu, band_flag(rec, r, S, base + lane, cnt, band)));
    if (lane == 0) out[r] = m;
}

__global__ void __launch_bounds__(256) k_band_write(const double* __restrict__ O, const double* __restrict__ D,
                                                    const uint32_t* __restrict__ counts, const double* __restrict__ T,
                                                    const float4* __restrict__ rec, uint64_t n, uint32_t S, float band,
                                                    const uint32_t* __restrict__ off, uint64_t cap, double* pts) {
    const uint64_t r = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= n) return;
    const uint32_t cnt = counts[r];
    uint64_t j = off[r];
    for (uint32_t base = 0; base < cnt && j < cap; base += 32) {
        const uint32_t k = base + lane;
        const bool f = band_flag(rec, r, S, k, cnt, band);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
        const uint64_t pos = j + __popc(bal & ((1u << lane) - 1u));
        if (f && pos < cap) {
            const double t = T[r * S + k];
#pragma unroll
            for (int q = 0; q < 3; ++q) pts[3 * pos + q] = __dadd_rn(O[3 * r + q], __dmul_rn(t, D[3 * r + q]));
        }
        j += __popc(bal);
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

void launch_sample_frame_rays(const svr_camera* cams, uint32_t n_frames, int32_t W, int32_t H,
                              uint32_t rays_per_image, uint64_t n, uint64_t seed, const float* rgb_img,
                              const float* depth_img, const float* normal_img, double* o, double* d, float* tgt,
                              float* pdepth, float* pnormal, uint32_t* cam_idx, uint32_t* pixel, cudaStream_t s) {
    if (!n) return;
    RayBatchArgs a{cams, n_frames, W, H, rays_per_image, n, seed, rgb_img, depth_img, normal_img,
                   o, d, tgt, pdepth, pnormal, cam_idx, pixel};
    k_sample_frame_rays<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a);
}

uint64_t band_points(const double* o, const double* d, const uint32_t* counts, const double* t,
                     const float4* rec, uint64_t n, uint32_t S, float band, uint32_t* scratch, void* tmp,
                     size_t tmp_bytes, uint64_t cap, double* pts, cudaStream_t s) {
    if (!n) return 0;
    const unsigned grid = static_cast<unsigned>((n * 32 + 255) / 256);  // warp per ray
    uint32_t* cnt = scratch;
    uint32_t* off = scratch + n;
    k_band_count<<<grid, 256, 0, s>>>(counts, rec, n, S, band, cnt);
    size_t bytes = tmp_bytes;
    SVR_LCK(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, off, static_cast<int>(n), s));
    uint32_t h[2];
    SVR_LCK(cudaMemcpyAsync(&h[0], off + n - 1, 4, cudaMemcpyDeviceToHost, s));
    SVR_LCK(cudaMemcpyAsync(&h[1], cnt + n - 1, 4, cudaMemcpyDeviceToHost, s));
    if (pts) k_band_write<<<grid, 256, 0, s>>>(o, d, counts, t, rec, n, S, band, off, cap, pts);
    SVR_LCK(cudaStreamSynchronize(s));
    return static_cast<uint64_t>(h[0]) + h[1];
}

size_t band_points_tmp_bytes(uint64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<int>(n));
    return bytes;
}

}  // namespace svr_internal
