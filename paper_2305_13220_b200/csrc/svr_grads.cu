// sm_100a kernels around the payload and gradient planes:
//   payload in/out (reference per-block layout <-> float4 (sdf,r,g,b) planes + validity
//   bitmask), dense AABB index build, gradient readback, K7 active-block compaction,
//   and the pack / unpack / zero kernels of the multi-GPU active-block reduction (K8's
//   device side; the collective itself is NCCL through torch.distributed).
#include "svr_internal.h"

namespace svr_dev {
namespace {

// One CTA of 512 threads per block: thread v handles voxel v (coalesced float4 stores).
__global__ void __launch_bounds__(512) k_payload_in(float4* pay, float* weight, float* logits,
                                                    uint32_t* vmask, uint32_t* meta, uint32_t first,
                                                    int32_t C, const float* __restrict__ sdf,
                                                    const float* __restrict__ w,
                                                    const float* __restrict__ rgb,
                                                    const float* __restrict__ lg) {
    const uint32_t b = blockIdx.x, v = threadIdx.x;
    const size_t src = static_cast<size_t>(b) * kVox + v;
    const size_t dst = static_cast<size_t>(first + b) * kVox + v;
    if (sdf || rgb) {
        float4 p = pay[dst];
        if (sdf) p.x = sdf[src];
        if (rgb) p.y = rgb[3 * src], p.z = rgb[3 * src + 1], p.w = rgb[3 * src + 2];
        pay[dst] = p;
    }
    if (lg)
        for (int k = 0; k < C; ++k) logits[dst * C + k] = lg[src * C + k];
    if (w) {
        const float wv = w[src];
        weight[dst] = wv;
        const unsigned bits = __ballot_sync(0xFFFFFFFFu, wv > 0.0f);  // grid.cpp:142
        __shared__ unsigned words[16];
        if ((v & 31) == 0) {
            words[v >> 5] = bits;
            vmask[static_cast<size_t>(first + b) * 16 + (v >> 5)] = bits;
        }
        __syncthreads();
        if (v == 0) {
            unsigned all = 0xFFFFFFFFu;
            for (int i = 0; i < 16; ++i) all &= words[i];
            meta[first + b] = (all == 0xFFFFFFFFu) ? 1u : 0u;
        }
    }
}

__global__ void __launch_bounds__(512) k_payload_out(const float4* __restrict__ pay,
                                                     const float* __restrict__ weight,
                                                     const float* __restrict__ logits,
                                                     uint32_t first, int32_t C, float* sdf,
                                                     float* w, float* rgb, float* lg) {
    const uint32_t b = blockIdx.x, v = threadIdx.x;
    const size_t dst = static_cast<size_t>(b) * kVox + v;
    const size_t src = static_cast<size_t>(first + b) * kVox + v;
    const float4 p = pay[src];
    if (sdf) sdf[dst] = p.x;
    if (rgb) rgb[3 * dst] = p.y, rgb[3 * dst + 1] = p.z, rgb[3 * dst + 2] = p.w;
    if (w) w[dst] = weight[src];
    if (lg)
        for (int k = 0; k < C; ++k) lg[dst * C + k] = logits[src * C + k];
}

__global__ void k_dense_build(const int4* __restrict__ coords, const uint32_t* __restrict__ meta,
                              uint32_t n, int32_t lx, int32_t ly, int32_t lz, int32_t dx,
                              int32_t dy, uint32_t* dense, uint32_t* occ) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    const size_t cell = (static_cast<size_t>(c.z - lz) * dy + (c.y - ly)) * dx + (c.x - lx);
    dense[cell] = i | ((meta[i] & 1u) ? kFullBit : 0u);
    atomicOr(occ + (cell >> 5), 1u << (cell & 31));
}

// Superblock occupancy (hash mode): bit of superblock (coord >> 3) set for every block.
__global__ void k_superblock_occ(const int4* __restrict__ coords, uint32_t n, int32_t lx, int32_t ly, int32_t lz,
                                 int32_t dx, int32_t dy, uint32_t* occ) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    const size_t cell = (static_cast<size_t>((c.z >> 3) - lz) * dy + ((c.y >> 3) - ly)) * dx + ((c.x >> 3) - lx);
    atomicOr(occ + (cell >> 5), 1u << (cell & 31));
}

// Chebyshev block-distance field over the dense AABB (for empty-space jumps in the march):
// three separable windowed passes, out = min_k max(|k|, in[cell + k e_axis]), |k| <= cap;
// pass 0 reads the occupancy bits (allocated = 0, empty = cap + 1).
constexpr int kDistCap = 15;
__global__ void k_bdist_pass(const uint32_t* __restrict__ occ, const uint8_t* __restrict__ in, uint8_t* out,
                             int32_t dx, int32_t dy, int32_t dz, int axis) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t n = static_cast<uint64_t>(dx) * dy * dz;
    if (i >= n) return;
    const int32_t x = static_cast<int32_t>(i % dx), y = static_cast<int32_t>((i / dx) % dy),
                  z = static_cast<int32_t>(i / (static_cast<uint64_t>(dx) * dy));
    const int32_t pos = axis == 0 ? x : (axis == 1 ? y : z);
    const int32_t len = axis == 0 ? dx : (axis == 1 ? dy : dz);
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? dx : static_cast<int64_t>(dx) * dy);
    int best = kDistCap + 1;
    for (int k = -kDistCap; k <= kDistCap; ++k) {
        const int32_t q = pos + k;
        if (q < 0 || q >= len) continue;
        const uint64_t j = static_cast<uint64_t>(static_cast<int64_t>(i) + k * stride);
        const int v = axis == 0 ? (((occ[j >> 5] >> (j & 31)) & 1u) ? 0 : kDistCap + 1) : in[j];
        const int ak = k < 0 ? -k : k;
        const int m = v > ak ? v : ak;
        if (m < best) best = m;
    }
    out[i] = static_cast<uint8_t>(best);
}

// Hash mode: block-distance bricks.  Every superblock at superblock distance <= 1 from an
// occupied one owns a brick of 8^3 u8 block distances: the exact Chebyshev distance to the
// nearest allocated block, capped at kBrickCap + 1.  A block of a superblock at distance >= 2
// is at least 8 + 1 blocks from every allocated one, so reading brick-less superblocks as
// kBrickCap + 1 = 9 keeps the three separable passes exact up to the cap.
constexpr int kBrickCap = 8;
__global__ void k_brick_assign(const uint8_t* __restrict__ sbdist, uint64_t n, uint32_t* info, uint32_t* brick_sb,
                               uint32_t* counter) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t d = sbdist[i];
    if (d <= 1) {
        const uint32_t b = atomicAdd(counter, 1u);
        info[i] = b;
        brick_sb[b] = static_cast<uint32_t>(i);
    } else {
        info[i] = kNoBrick | d;
    }
}
__global__ void k_brick_occ(const int4* __restrict__ coords, uint32_t n, int32_t lx, int32_t ly, int32_t lz,
                            int32_t dx, int32_t dy, const uint32_t* __restrict__ info, uint8_t* bricks) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    const size_t sb = (static_cast<size_t>((c.z >> 3) - lz) * dy + ((c.y >> 3) - ly)) * dx + ((c.x >> 3) - lx);
    bricks[static_cast<size_t>(info[sb]) * kVox + (c.x & 7) + 8 * ((c.y & 7) + 8 * (c.z & 7))] = 0;
}
// out = min_k max(|k|, in[cell + k e_axis]), |k| <= kBrickCap, across brick boundaries
__global__ void k_brick_pass(const uint8_t* __restrict__ in, uint8_t* out, const uint32_t* __restrict__ info,
                             const uint32_t* __restrict__ brick_sb, uint32_t n_bricks, int32_t dx, int32_t dy,
                             int32_t dz, int axis) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<uint64_t>(n_bricks) * kVox) return;
    const uint32_t local = static_cast<uint32_t>(i & (kVox - 1));
    const uint32_t sb = brick_sb[i / kVox];
    int32_t sc[3] = {static_cast<int32_t>(sb % dx), static_cast<int32_t>((sb / dx) % dy),
                     static_cast<int32_t>(sb / (static_cast<uint32_t>(dx) * dy))};
    const int32_t dims[3] = {dx, dy, dz};
    int32_t lc[3] = {static_cast<int32_t>(local & 7), static_cast<int32_t>((local >> 3) & 7),
                     static_cast<int32_t>(local >> 6)};
    const int32_t pos = lc[axis];
    int best = kBrickCap + 1;
    for (int k = -kBrickCap; k <= kBrickCap; ++k) {
        const int32_t q = pos + k;
        const int32_t off = q < 0 ? -1 : (q > 7 ? 1 : 0);
        int32_t nc[3] = {sc[0], sc[1], sc[2]};
        nc[axis] += off;
        int v = kBrickCap + 1;
        if (nc[axis] >= 0 && nc[axis] < dims[axis]) {
            const uint32_t inf = info[(static_cast<size_t>(nc[2]) * dy + nc[1]) * dx + nc[0]];
            if (!(inf & kNoBrick)) {
                int32_t l2[3] = {lc[0], lc[1], lc[2]};
                l2[axis] = q & 7;
                v = in[static_cast<size_t>(inf) * kVox + l2[0] + 8 * (l2[1] + 8 * l2[2])];
            }
        }
        const int ak = k < 0 ? -k : k;
        const int m = v > ak ? v : ak;
        if (m < best) best = m;
    }
    out[i] = static_cast<uint8_t>(best);
}

// K8p: active-block gradient all-reduce directly over the ranks' gradient planes (peer memory:
// NVLink P2P through CUDA IPC mappings).  Rank r owns the slice [r n / W, (r + 1) n / W) of
// the ascending active list; for each of its rows every thread sums one float4 over the W
// planes in rank order (bitwise identical on every rank) and stores the sum into all W
// planes -- reduce-scatter and all-gather in one pass, no pack / unpack buffers.
constexpr int kMaxPeers = 8;
struct PeerPlanes {
    float4* p[kMaxPeers];
};
__global__ void __launch_bounds__(512) k_peer_allreduce(PeerPlanes pl, uint32_t world, const uint32_t* __restrict__ rows,
                                                        uint64_t first, uint64_t count) {
    for (uint64_t j = blockIdx.x; j < count; j += gridDim.x) {
        const size_t v = static_cast<size_t>(rows[first + j]) * kVox + threadIdx.x;
        float4 acc = pl.p[0][v];
        for (uint32_t q = 1; q < world; ++q) {
            const float4 x = pl.p[q][v];
            acc.x += x.x, acc.y += x.y, acc.z += x.z, acc.w += x.w;
        }
        for (uint32_t q = 0; q < world; ++q) pl.p[q][v] = acc;
    }
}

// AABB extension over new blocks (grid.cpp:96-106): warp min / max, one atomic per warp.
__global__ void k_bounds(const int4* __restrict__ c, uint64_t n, int32_t* b) {
    int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int4 v = c[i];
        lo[0] = min(lo[0], v.x), lo[1] = min(lo[1], v.y), lo[2] = min(lo[2], v.z);
        hi[0] = max(hi[0], v.x), hi[1] = max(hi[1], v.y), hi[2] = max(hi[2], v.z);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xFFFFFFFFu, lo[a], off));
            hi[a] = max(hi[a], __shfl_xor_sync(0xFFFFFFFFu, hi[a], off));
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(b + a, lo[a]);
            atomicMax(b + 3 + a, hi[a]);
        }
    }
}

// Per-block table of the 8 blocks a trilinear cell can touch: entry k = lookup of
// coord + (k & 1, (k >> 1) & 1, k >> 2) (k = 0 is the block itself), with the all-valid bit.
__global__ void k_nbr_build(GridView g, const int4* __restrict__ coords, uint32_t n, uint32_t* nbr) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 c = coords[i];
    uint32_t e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = lookup_block(g, c.x + (k & 1), c.y + ((k >> 1) & 1), c.z + (k >> 2));
    uint4* out = reinterpret_cast<uint4*>(nbr + static_cast<size_t>(i) * 8);
    out[0] = make_uint4(e[0], e[1], e[2], e[3]);
    out[1] = make_uint4(e[4], e[5], e[6], e[7]);
}

__global__ void k_grad_out(const float4* __restrict__ grad, uint64_t nvox, float* g_sdf,
                           float* g_rgb) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nvox) return;
    const float4 g = grad[i];
    if (g_sdf) g_sdf[i] = g.x;
    if (g_rgb) g_rgb[3 * i] = g.y, g_rgb[3 * i + 1] = g.z, g_rgb[3 * i + 2] = g.w;
}

// K7: ascending compaction of the active mask. Each CTA scans 1024 flags, takes a
// base offset with one atomic, and the final list is made ascending by a sort-free
// two-pass scheme: pass 1 counts per CTA, pass 2 (below) writes at exclusive offsets.
__global__ void __launch_bounds__(1024) k_active_count(const uint8_t* __restrict__ active,
                                                       uint32_t n, uint32_t* per_cta) {
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    const bool a = i < n && active[i];
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, a);
    __shared__ uint32_t warp_tot[32];
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < 32; ++w) s += warp_tot[w];
        per_cta[blockIdx.x] = s;
    }
}

__global__ void k_active_scan(uint32_t* per_cta, uint32_t nctas, unsigned long long* count) {
    // single-CTA exclusive scan over <= a few thousand CTA totals
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nctas; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        uint32_t v = i < nctas ? per_cta[i] : 0;
        // block-wide inclusive scan
        __shared__ uint32_t tmp[1024];
        tmp[threadIdx.x] = v;
        __syncthreads();
        for (uint32_t off = 1; off < 1024; off <<= 1) {
            const uint32_t add = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0;
            __syncthreads();
            tmp[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < nctas) per_cta[i] = carry + tmp[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += tmp[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = carry;
}

__global__ void __launch_bounds__(1024) k_active_write(const uint8_t* __restrict__ active,
                                                       uint32_t n,
                                                       const uint32_t* __restrict__ per_cta,
                                                       uint32_t* list) {
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    const bool a = i < n && active[i];
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, a);
    __shared__ uint32_t warp_off[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) warp_off[w] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int k = 0; k < 32; ++k) {
            const uint32_t t = warp_off[k];
            warp_off[k] = s;
            s += t;
        }
    }
    __syncthreads();
    if (a) list[per_cta[blockIdx.x] + warp_off[w] + __popc(bal & ((1u << lane) - 1))] = i;
}

__global__ void k_set_active(uint8_t* active, const uint8_t* __restrict__ mask, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) active[i] = mask[i] ? 1 : 0;
}

// pack / unpack: one CTA of 128 threads moves one block (512 float4 = 8 KB).
__global__ void __launch_bounds__(128) k_grad_pack(const float4* __restrict__ grad,
                                                   const uint32_t* __restrict__ blocks,
                                                   float4* out) {
    const size_t src = static_cast<size_t>(blocks[blockIdx.x]) * kVox;
    const size_t dst = static_cast<size_t>(blockIdx.x) * kVox;
#pragma unroll
    for (int k = 0; k < 4; ++k) out[dst + threadIdx.x + 128 * k] = grad[src + threadIdx.x + 128 * k];
}
__global__ void __launch_bounds__(128) k_grad_unpack(float4* grad, const uint32_t* __restrict__ blocks,
                                                     const float4* __restrict__ in) {
    const size_t dst = static_cast<size_t>(blocks[blockIdx.x]) * kVox;
    const size_t src = static_cast<size_t>(blockIdx.x) * kVox;
#pragma unroll
    for (int k = 0; k < 4; ++k) grad[dst + threadIdx.x + 128 * k] = in[src + threadIdx.x + 128 * k];
}
// zero active blocks' gradients (grid-stride over the device-side count)
__global__ void __launch_bounds__(128) k_grad_zero_active(float4* grad, uint8_t* active,
                                                          const uint32_t* __restrict__ list,
                                                          const unsigned long long* count) {
    const unsigned long long n = *count;
    for (unsigned long long j = blockIdx.x; j < n; j += gridDim.x) {
        const uint32_t b = list[j];
        const size_t base = static_cast<size_t>(b) * kVox;
#pragma unroll
        for (int k = 0; k < 4; ++k) grad[base + threadIdx.x + 128 * k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (threadIdx.x == 0) active[b] = 0;
    }
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

void launch_payload_in(float4* pay, float* weight, float* logits, uint32_t* vmask, uint32_t* meta,
                       uint32_t first, uint32_t n, int32_t C, const float* sdf, const float* w,
                       const float* rgb, const float* lg, cudaStream_t s) {
    if (!n) return;
    k_payload_in<<<n, 512, 0, s>>>(pay, weight, logits, vmask, meta, first, C, sdf, w, rgb, lg);
}

void launch_payload_out(const float4* pay, const float* weight, const float* logits,
                        uint32_t first, uint32_t n, int32_t C, float* sdf, float* w, float* rgb,
                        float* lg, cudaStream_t s) {
    if (!n) return;
    k_payload_out<<<n, 512, 0, s>>>(pay, weight, logits, first, C, sdf, w, rgb, lg);
}

void launch_dense_build(const int32_t* coords4, const uint32_t* meta, uint32_t n, const int32_t* lo,
                        const int32_t* dim, uint32_t* dense, uint32_t* occ, cudaStream_t s) {
    if (!n) return;
    k_dense_build<<<(n + 255) / 256, 256, 0, s>>>(reinterpret_cast<const int4*>(coords4), meta, n,
                                                  lo[0], lo[1], lo[2], dim[0], dim[1], dense, occ);
}

void launch_superblock_occ(const int32_t* coords4, uint32_t n, const int32_t* sb_lo, const int32_t* sb_dim,
                           uint32_t* occ, cudaStream_t s) {
    if (!n) return;
    k_superblock_occ<<<(n + 255) / 256, 256, 0, s>>>(reinterpret_cast<const int4*>(coords4), n, sb_lo[0], sb_lo[1],
                                                      sb_lo[2], sb_dim[0], sb_dim[1], occ);
}

void launch_bdist(const uint32_t* occ, const int32_t* dim, uint8_t* out, uint8_t* tmp, cudaStream_t s) {
    const uint64_t n = static_cast<uint64_t>(dim[0]) * dim[1] * dim[2];
    if (!n) return;
    const unsigned grid = static_cast<unsigned>((n + 255) / 256);
    k_bdist_pass<<<grid, 256, 0, s>>>(occ, nullptr, tmp, dim[0], dim[1], dim[2], 0);
    k_bdist_pass<<<grid, 256, 0, s>>>(occ, tmp, out, dim[0], dim[1], dim[2], 1);
    k_bdist_pass<<<grid, 256, 0, s>>>(occ, out, tmp, dim[0], dim[1], dim[2], 2);
    SVR_LCK(cudaMemcpyAsync(out, tmp, n, cudaMemcpyDeviceToDevice, s));
}

uint32_t launch_brick_assign(const int32_t* sb_dim, const uint8_t* sbdist, uint32_t* info, uint32_t* brick_sb,
                             uint32_t* counter, cudaStream_t s) {
    const uint64_t sc = static_cast<uint64_t>(sb_dim[0]) * sb_dim[1] * sb_dim[2];
    if (!sc) return 0;
    SVR_LCK(cudaMemsetAsync(counter, 0, 4, s));
    k_brick_assign<<<static_cast<unsigned>((sc + 255) / 256), 256, 0, s>>>(sbdist, sc, info, brick_sb, counter);
    uint32_t nb = 0;
    SVR_LCK(cudaMemcpyAsync(&nb, counter, 4, cudaMemcpyDeviceToHost, s));
    SVR_LCK(cudaStreamSynchronize(s));
    return nb;
}

void launch_brick_fill(const int32_t* coords4, uint32_t n, const int32_t* sb_lo, const int32_t* sb_dim,
                       const uint32_t* info, const uint32_t* brick_sb, uint32_t n_bricks, uint8_t* bricks,
                       uint8_t* tmp, cudaStream_t s) {
    if (!n || !n_bricks) return;
    const size_t bytes = static_cast<size_t>(n_bricks) * kVox;
    SVR_LCK(cudaMemsetAsync(tmp, kBrickCap + 1, bytes, s));
    k_brick_occ<<<(n + 255) / 256, 256, 0, s>>>(reinterpret_cast<const int4*>(coords4), n, sb_lo[0], sb_lo[1],
                                                 sb_lo[2], sb_dim[0], sb_dim[1], info, tmp);
    const unsigned grid = static_cast<unsigned>((bytes + 255) / 256);
    k_brick_pass<<<grid, 256, 0, s>>>(tmp, bricks, info, brick_sb, n_bricks, sb_dim[0], sb_dim[1], sb_dim[2], 0);
    k_brick_pass<<<grid, 256, 0, s>>>(bricks, tmp, info, brick_sb, n_bricks, sb_dim[0], sb_dim[1], sb_dim[2], 1);
    k_brick_pass<<<grid, 256, 0, s>>>(tmp, bricks, info, brick_sb, n_bricks, sb_dim[0], sb_dim[1], sb_dim[2], 2);
}

void launch_peer_allreduce(float4* const* planes, uint32_t world, uint32_t rank, const uint32_t* rows,
                           uint64_t n_rows, cudaStream_t s) {
    if (!n_rows || !world) return;
    PeerPlanes pl{};
    for (uint32_t q = 0; q < world; ++q) pl.p[q] = planes[q];
    const uint64_t first = n_rows * rank / world, last = n_rows * (rank + 1) / world;
    if (last <= first) return;
    const uint64_t count = last - first;
    const uint64_t cap = sm_count() * 8ull;
    const unsigned grid = static_cast<unsigned>(count < cap ? count : cap);
    k_peer_allreduce<<<grid, 512, 0, s>>>(pl, world, rows, first, count);
}

void launch_bounds(const int32_t* coords4, uint64_t n, int32_t* b, cudaStream_t s) {
    if (!n) return;
    const uint64_t want = (n + 255) / 256, cap = sm_count() * 4ull;
    k_bounds<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, s>>>(reinterpret_cast<const int4*>(coords4), n, b);
}

void launch_nbr_build(const GridView& g, const int32_t* coords4, uint32_t n, uint32_t* nbr,
                      cudaStream_t s) {
    if (!n) return;
    k_nbr_build<<<(n + 255) / 256, 256, 0, s>>>(g, reinterpret_cast<const int4*>(coords4), n, nbr);
}

void launch_grad_out(const float4* grad, uint32_t n, float* g_sdf, float* g_rgb, cudaStream_t s) {
    const uint64_t nvox = static_cast<uint64_t>(n) * kVox;
    if (!nvox) return;
    k_grad_out<<<static_cast<unsigned>((nvox + 255) / 256), 256, 0, s>>>(grad, nvox, g_sdf, g_rgb);
}

void launch_active_list(const uint8_t* active, uint32_t n, uint32_t* list,
                        unsigned long long* count, cudaStream_t s) {
    // per_cta scratch lives right after the count (caller provides >= nctas+2 words there)
    const uint32_t nctas = (n + 1023) / 1024;
    uint32_t* per_cta = reinterpret_cast<uint32_t*>(count + 1);
    if (nctas == 0) {
        SVR_LCK(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
        return;
    }
    k_active_count<<<nctas, 1024, 0, s>>>(active, n, per_cta);
    k_active_scan<<<1, 1024, 0, s>>>(per_cta, nctas, count);
    k_active_write<<<nctas, 1024, 0, s>>>(active, n, per_cta, list);
}

void launch_set_active(uint8_t* active, const uint8_t* mask, uint32_t n, cudaStream_t s) {
    if (!n) return;
    k_set_active<<<(n + 255) / 256, 256, 0, s>>>(active, mask, n);
}

void launch_grad_pack(const float4* grad, const uint32_t* blocks, uint64_t n, float4* out,
                      cudaStream_t s) {
    if (!n) return;
    k_grad_pack<<<static_cast<unsigned>(n), 128, 0, s>>>(grad, blocks, out);
}

void launch_grad_unpack(float4* grad, const uint32_t* blocks, uint64_t n, const float4* in,
                        cudaStream_t s) {
    if (!n) return;
    k_grad_unpack<<<static_cast<unsigned>(n), 128, 0, s>>>(grad, blocks, in);
}

void launch_grad_zero_active(float4* grad, uint8_t* active, const uint32_t* list,
                             const unsigned long long* count, uint32_t n_max, cudaStream_t s,
                             unsigned ctas_per_sm) {
    if (!n_max) return;
    const unsigned cap = sm_count() * ctas_per_sm;
    const unsigned grid = n_max < cap ? n_max : cap;
    k_grad_zero_active<<<grid, 128, 0, s>>>(grad, active, list, count);
}

}  // namespace svr_internal
