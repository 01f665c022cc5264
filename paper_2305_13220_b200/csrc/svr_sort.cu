// Ray ordering for locality: an in-house bucketed counting sort (no library kernels on
// the hot path).  Only locality matters (results never depend on the order), so rays are
// binned into 2^18 buckets and the order inside a bucket is whatever the atomics give.
//
//   mode DIR   (before the march): bucket = 6-bit origin hash (1 mm cells) above a 12-bit
//              Morton code of the octahedral direction (64 x 64 cells, ~3 deg) -- rays of
//              one camera with nearby pixels are marched by the same warps.
//   mode BLOCK (after the march):  bucket = 18-bit Morton code of the first sample's block,
//              coarsened so the AABB fits in 64^3 cells; rays without samples go last.
//
// Three launches: bucket + histogram, scan (one CTA), scatter.
#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr int kBucketBits = 18;
constexpr uint32_t kBuckets = 1u << kBucketBits;

__device__ __forceinline__ uint32_t spread3_6(uint32_t v) {  // 6 bits -> every 3rd bit
    v &= 63u;
    v = (v | (v << 8)) & 0x0000F00Fu;
    v = (v | (v << 4)) & 0x000C30C3u;
    v = (v | (v << 2)) & 0x00249249u;
    return v;
}
__device__ __forceinline__ uint32_t spread2_6(uint32_t v) {  // 6 bits -> every 2nd bit
    v &= 63u;
    v = (v | (v << 4)) & 0x0F0Fu;
    v = (v | (v << 2)) & 0x3333u;
    v = (v | (v << 1)) & 0x5555u;
    return v;
}

__device__ __forceinline__ uint32_t dir_bucket(const double* O, const double* D, uint64_t r) {
    const double dx = D[3 * r], dy = D[3 * r + 1], dz = D[3 * r + 2];
    const double l1 = fabs(dx) + fabs(dy) + fabs(dz);
    double u = dx / l1, v = dy / l1;
    if (dz < 0.0) {
        const double uu = (1.0 - fabs(v)) * (u >= 0.0 ? 1.0 : -1.0);
        const double vv = (1.0 - fabs(u)) * (v >= 0.0 ? 1.0 : -1.0);
        u = uu, v = vv;
    }
    const uint32_t qu = min(63u, static_cast<uint32_t>((u * 0.5 + 0.5) * 64.0));
    const uint32_t qv = min(63u, static_cast<uint32_t>((v * 0.5 + 0.5) * 64.0));
    unsigned long long h = 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int a = 0; a < 3; ++a) h = mix64(h ^ static_cast<unsigned long long>(llrint(O[3 * r + a] * 1000.0)));
    return (static_cast<uint32_t>(h >> 58) << 12) | spread2_6(qu) | (spread2_6(qv) << 1);
}

__device__ __forceinline__ uint32_t block_bucket(const GridView& g, const double* O, const double* D,
                                                 uint64_t r, const uint32_t* counts, const double* T,
                                                 uint32_t S, int shift) {
    if (!counts[r]) return kBuckets - 1;
    const double t = T[r * S];
    uint32_t c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = O[3 * r + a] + t * D[3 * r + a];
        int32_t v = static_cast<int32_t>(floor(x / g.L)) - g.lo[a];
        v = v < 0 ? 0 : v;
        c[a] = min(63u, static_cast<uint32_t>(v) >> shift);
    }
    return spread3_6(c[0]) | (spread3_6(c[1]) << 1) | (spread3_6(c[2]) << 2);
}

__global__ void __launch_bounds__(256) k_bucket_count(GridView g, const double* __restrict__ O,
                                                      const double* __restrict__ D, uint64_t n,
                                                      const uint32_t* __restrict__ counts,
                                                      const double* __restrict__ T, uint32_t S,
                                                      int shift, uint32_t* bucket, uint32_t* hist) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t b = counts ? block_bucket(g, O, D, r, counts, T, S, shift) : dir_bucket(O, D, r);
    bucket[r] = b;
    // warp-aggregated histogram increment (neighbouring rays often share a bucket)
    const unsigned peers = __match_any_sync(__activemask(), b);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + b, static_cast<uint32_t>(__popc(peers)));
}

// Exclusive scan of kBuckets counters in one CTA of 1024 threads (256 per thread).
__global__ void __launch_bounds__(1024) k_bucket_scan(uint32_t* hist) {
    constexpr int kPer = kBuckets / 1024;
    __shared__ uint32_t part[1024];
    uint32_t* h = hist + threadIdx.x * kPer;
    uint32_t sum = 0;
    for (int i = 0; i < kPer; ++i) sum += h[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - sum;
    for (int i = 0; i < kPer; ++i) {
        const uint32_t c = h[i];
        h[i] = run;
        run += c;
    }
}

__global__ void __launch_bounds__(256) k_bucket_scatter(uint64_t n, const uint32_t* __restrict__ bucket,
                                                        uint32_t* offs, uint32_t* order) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t b = bucket[r];
    const unsigned peers = __match_any_sync(__activemask(), b);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(offs + b, static_cast<uint32_t>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    order[base + __popc(peers & ((1u << lane) - 1))] = static_cast<uint32_t>(r);
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

size_t ray_order_scratch_words(uint64_t n) { return 2 * n + kBuckets; }

void launch_ray_bucket_order(const GridView& g, const double* o, const double* d, uint64_t n,
                             const uint32_t* counts, const double* t, uint32_t S, uint32_t* scratch,
                             cudaStream_t s) {
    if (!n) return;
    uint32_t* order = scratch;
    uint32_t* bucket = scratch + n;
    uint32_t* hist = scratch + 2 * n;
    int shift = 0;
    if (counts) {
        int dmax = 1;
        for (int a = 0; a < 3; ++a) dmax = dmax > g.dim[a] ? dmax : g.dim[a];
        while ((dmax - 1) >> shift >= 64) ++shift;
    }
    cudaMemsetAsync(hist, 0, kBuckets * sizeof(uint32_t), s);
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    k_bucket_count<<<grid, 256, 0, s>>>(g, o, d, n, counts, t, S, shift, bucket, hist);
    k_bucket_scan<<<1, 1024, 0, s>>>(hist);
    k_bucket_scatter<<<grid, 256, 0, s>>>(n, bucket, hist, order);
}

}  // namespace svr_internal
