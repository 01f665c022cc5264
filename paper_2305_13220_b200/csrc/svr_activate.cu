// sm_100a kernels for block activation and the block hash table:
//   K1 hash insert / find over 64-bit packed keys (grid.cpp:28-67, 88-108)
//   K3 depth / points -> base block keys -> L-inf dilation -> new-key filter
//      (allocation.cpp:19-83).  Dedup uses device key sets (open addressing, CAS);
//      warps first collapse equal keys with __match_any_sync so a run of pixels that
//      land in one block costs one probe.
// All discrete math (unproject, floor(x / L)) is fp64 with explicit _rn intrinsics.
#include <cub/device/device_radix_sort.cuh>

#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Insert into a key set; returns true if this call added the key.
__device__ __forceinline__ bool keyset_insert(unsigned long long* slots, unsigned long long mask,
                                              unsigned long long key) {
    unsigned long long i = mix64(key) & mask;
    for (unsigned long long probes = 0; probes <= mask; ++probes) {
        const unsigned long long cur = slots[i];
        if (cur == key) return false;
        if (cur == kEmptyKey) {
            const unsigned long long prev = atomicCAS(slots + i, kEmptyKey, key);
            if (prev == kEmptyKey) return true;
            if (prev == key) return false;
        }
        i = (i + 1) & mask;
    }
    return false;  // full; caller detects via the count
}

__device__ __forceinline__ void append_key(unsigned long long key, bool add,
                                           const svr_internal::KeySet& ks,
                                           unsigned long long* count) {
    if (!add) return;
    const unsigned long long pos = atomicAdd(count, 1ull);
    if (pos < ks.cap) ks.list[pos] = key;
}

// Warp-collapse equal keys, then one leader per distinct key probes the set.
__device__ __forceinline__ void warp_insert(bool have, unsigned long long key,
                                            const svr_internal::KeySet& ks,
                                            unsigned long long* count) {
    const unsigned active = __ballot_sync(kFull, have);
    if (!have) return;
    const unsigned peers = __match_any_sync(active, key);
    const int lane = threadIdx.x & 31;
    if (lane == __ffs(peers) - 1) append_key(key, keyset_insert(ks.slots, ks.mask, key), ks, count);
}

// Pixels along an image row map to runs of equal block keys: one insert per run (a lane whose
// left neighbour holds the same key skips it) -- cheaper than a full match, and a key that
// reappears later in the warp is simply inserted again (the set keeps it once).
__device__ __forceinline__ void warp_insert_runs(bool have, unsigned long long key,
                                                 const svr_internal::KeySet& ks,
                                                 unsigned long long* count) {
    const int lane = threadIdx.x & 31;
    const unsigned long long k = have ? key : ~0ull;
    const unsigned long long prev = __shfl_up_sync(kFull, k, 1);
    if (have && (lane == 0 || prev != k)) append_key(key, keyset_insert(ks.slots, ks.mask, key), ks, count);
}

// block_of_point (grid.hpp:136-141): floor(x / L) of the correctly rounded quotient.  Fast
// path: q = x * (1/L) (both rounded) is within |x/L| 2^-51.9 <= 2^-31.9 of x/L for the
// representable block range |x/L| < 2^20, and RN(x/L) within 2^-33 of it; so when q's
// fraction keeps 2^-28 away from an integer, floor(RN(x / L)) = floor(q).  Otherwise (and out
// of range) the exactly rounded division decides.
__device__ __forceinline__ double floor_div(double x, double L, double inv_L) {
    const double q = __dmul_rn(x, inv_L);
    const double fq = floor(q);
    const double fr = __dsub_rn(q, fq);
    if (fabs(q) < 0x1p20 && fr > 0x1p-28 && fr < 1.0 - 0x1p-28) return fq;
    return floor(__ddiv_rn(x, L));
}
__device__ __forceinline__ bool block_of_point(const double p[3], double L, double inv_L, int32_t b[3]) {
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double f = floor_div(p[a], L, inv_L);
        ok = ok && f >= -static_cast<double>(kCoordLim) && f < static_cast<double>(kCoordLim);
        b[a] = ok ? static_cast<int32_t>(f) : 0;
    }
    return ok;
}

__global__ void k_keyset_clear(unsigned long long* slots, unsigned long long n) {
    for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
         i < n; i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
        slots[i] = kEmptyKey;
}

__global__ void k_points_to_keys(const double* __restrict__ xyz, uint64_t n, double L,
                                 svr_internal::KeySet ks, unsigned long long* count,
                                 uint32_t* flags) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool have = i < n;
    unsigned long long key = 0;
    if (have) {
        const double p[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
        int32_t b[3];
        if (block_of_point(p, L, 1.0 / L, b)) {
            key = pack_key(b[0], b[1], b[2]);
        } else {
            atomicOr(flags, 1u);
            have = false;
        }
    }
    warp_insert(have, key, ks, count);
}

// Per-frame ray tables: u[x] = (x - cx) / fx and v[y] = (y - cy) / fy, exactly as
// Camera::unproject computes them per pixel (camera.cpp:20-25) -- a pixel then costs two
// multiplications by its depth instead of two divisions.
__global__ void k_frame_tables(const svr_camera* __restrict__ cams, int32_t W, int32_t H, double* tab) {
    const uint32_t f = blockIdx.x;
    const svr_camera& c = cams[f];
    double* t = tab + static_cast<size_t>(f) * (W + H);
    for (int32_t i = threadIdx.x; i < W + H; i += blockDim.x)
        t[i] = i < W ? __ddiv_rn(__dsub_rn(static_cast<double>(i), c.cx), c.fx)
                     : __ddiv_rn(__dsub_rn(static_cast<double>(i - W), c.cy), c.fy);
}

// allocate_for_frames pixel loop (allocation.cpp:63-79): valid depth, optional
// ScaleField::value (scale_field.cpp:15-60), Camera::unproject (camera.cpp:20-25) with
// R x_c evaluated row-wise left to right, then block_of_point.  Warp per image row (rows of
// all frames grid-strided over the warps, 32 pixels per pass: no per-pixel index division,
// a warp-uniform trip count for the warp-collapsed key insert); the used-pixel count is
// summed per lane and added once per warp.
__global__ void __launch_bounds__(256) k_depth_to_keys(const float* __restrict__ depth, const svr_camera* __restrict__ cams,
                                                       const double* __restrict__ tab, uint32_t n_frames, int32_t W,
                                                       int32_t H, const double* __restrict__ scales, int32_t rows,
                                                       int32_t cols, double L, svr_internal::KeySet ks,
                                                       unsigned long long* count, unsigned long long* pixels,
                                                       uint32_t* flags) {
    const int lane = threadIdx.x & 31;
    const uint32_t nrows = n_frames * static_cast<uint32_t>(H);
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const double inv_L = 1.0 / L;
    unsigned long long used = 0;
    for (uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nrows; row += warps) {
        const uint32_t f = row / static_cast<uint32_t>(H);
        const int y = static_cast<int>(row - f * static_cast<uint32_t>(H));
        const svr_camera& c = cams[f];
        const double* t = tab + static_cast<size_t>(f) * (W + H);
        const double vy = t[W + y];
        const float* drow = depth + static_cast<size_t>(row) * W;
        const double* sf = scales ? scales + static_cast<size_t>(f) * rows * cols : nullptr;
        // four 32-pixel chunks per group: their depth loads are in flight together
        for (int xg = 0; xg < W; xg += 128) {
        float dq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) dq[u] = xg + 32 * u + lane < W ? __ldg(drow + xg + 32 * u + lane) : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x0 = xg + 32 * u;
            if (x0 >= W) break;  // warp-uniform
            const int x = x0 + lane;
            bool have = x < W;
            unsigned long long key = 0;
            if (have) {
                const float dv = dq[u];
                have = dv > 0.0f;
                double scale = 1.0;
                if (have && sf) {
                    scale = scale_field_value(sf, rows, cols, W, H, x, y);
                    have = scale > 0.0;
                }
                if (have) {
                    const double dep = __dmul_rn(static_cast<double>(dv), scale);
                    const double xc[3] = {__dmul_rn(t[x], dep), __dmul_rn(vy, dep), dep};
                    double p[3];
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        double acc = __dmul_rn(c.R[3 * r], xc[0]);
                        acc = __dadd_rn(acc, __dmul_rn(c.R[3 * r + 1], xc[1]));
                        acc = __dadd_rn(acc, __dmul_rn(c.R[3 * r + 2], xc[2]));
                        p[r] = __dadd_rn(acc, c.t[r]);
                    }
                    int32_t b[3];
                    if (block_of_point(p, L, inv_L, b)) {
                        key = pack_key(b[0], b[1], b[2]);
                    } else {
                        atomicOr(flags, 1u);
                        have = false;
                    }
                }
            }
            used += have ? 1u : 0u;
            warp_insert_runs(have, key, ks, count);
        }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) used += __shfl_xor_sync(kFull, used, off);
    if (lane == 0 && used) atomicAdd(pixels, used);
}

// commit's dilation (allocation.cpp:22-26): base x (2R+1)^3 offsets into `wanted`.
__global__ void k_dilate(const unsigned long long* __restrict__ base, uint64_t nbase, int32_t R,
                         svr_internal::KeySet ks, unsigned long long* count, uint32_t* flags) {
    const uint64_t side = 2 * static_cast<uint64_t>(R) + 1, per = side * side * side;
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool have = i < nbase * per;
    unsigned long long key = 0;
    if (have) {
        const uint64_t bi = i / per, off = i - bi * per;
        int32_t x, y, z;
        unpack_key(base[bi], x, y, z);
        x += static_cast<int32_t>(off % side) - R;
        y += static_cast<int32_t>((off / side) % side) - R;
        z += static_cast<int32_t>(off / (side * side)) - R;
        if (packable(x, y, z)) {
            key = pack_key(x, y, z);
        } else {
            atomicOr(flags, 1u);
            have = false;
        }
    }
    warp_insert(have, key, ks, count);
}

// commit's "already allocated?" test (allocation.cpp:31).
__global__ void k_filter_fresh(GridView g, const unsigned long long* __restrict__ keys, uint64_t n,
                               unsigned long long* fresh, unsigned long long* nfresh) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = keys[i];
    const bool is_new = g.n_blocks == 0 || hash_find(g, k) == kInvalid;
    if (is_new) fresh[atomicAdd(nfresh, 1ull)] = k;
}

// Warp-cooperative insert (the counterpart of k_hash_find): 8 lanes per key read one 128 B
// line (8 slots) per probe step through L2 (ld.cg: a slot claimed by another key since is not
// hidden by a stale L1 line) and the group claims the first empty slot in probe order with one
// CAS from the lane holding it; a lost race moves to the next empty slot of the line, then to
// the next line.  Keys are unique and absent (filtered above), so the CAS on the empty marker
// is the only synchronisation.  keys[i] -> first + i; coords4 gets (x, y, z, 0).
// (BlockMap::insert, grid.cpp:41-67: linear probing; slot positions are not observable.)
__global__ void k_hash_insert(HashSlot* slots, unsigned long long mask,
                              const unsigned long long* __restrict__ keys, uint64_t n,
                              uint32_t first, int32_t* coords4) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t q = tid >> 3;
    if (q >= n) return;  // whole 8-lane groups leave together
    const int sub = threadIdx.x & 7;
    const unsigned shift = threadIdx.x & 24;
    const unsigned group = 0xFFu << shift;
    const unsigned long long k = keys[q];
    const unsigned long long start = mix64(k) & mask;
    for (unsigned long long step = 0;; step += 8) {
        const unsigned long long s = (start + step + sub) & mask;
        const unsigned long long cur = __ldcg(&slots[s].key);
        unsigned e8 = (__ballot_sync(group, cur == kEmptyKey) >> shift) & 0xFFu;
        bool placed = false;
        while (e8) {
            const int lead = __ffs(e8) - 1;
            bool won = false;
            if (sub == lead) {
                won = atomicCAS(&slots[s].key, kEmptyKey, k) == kEmptyKey;
                if (won) slots[s].val = first + static_cast<uint32_t>(q);
            }
            if (__shfl_sync(group, won ? 1u : 0u, lead + static_cast<int>(shift))) {
                placed = true;
                break;
            }
            e8 &= e8 - 1;  // the slot went to another key: next empty slot of the line
        }
        if (placed) break;
    }
    if (sub == 0) {
        int32_t x, y, z;
        unpack_key(k, x, y, z);
        reinterpret_cast<int4*>(coords4)[first + q] = make_int4(x, y, z, 0);
    }
}

// Warp-cooperative find: 8 lanes probe one 128 B line (8 slots) per step.
__global__ void k_hash_find(const HashSlot* __restrict__ slots, unsigned long long mask,
                            const int32_t* __restrict__ coords3, uint64_t n, uint32_t* out) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t q = tid >> 3;
    const int sub = threadIdx.x & 7;
    const unsigned group = 0xFFu << (threadIdx.x & 24);
    const bool have = q < n;
    unsigned long long key = 0;
    bool ok = have;
    if (have) {
        const int32_t x = coords3[3 * q], y = coords3[3 * q + 1], z = coords3[3 * q + 2];
        ok = packable(x, y, z);
        key = ok ? pack_key(x, y, z) : 0;
    }
    uint32_t result = kInvalid;
    bool done = !ok;
    unsigned long long start = ok ? (mix64(key) & mask) : 0;
    for (unsigned long long step = 0; !__all_sync(kFull, done); step += 8) {
        if (!done) {
            const unsigned long long s = (start + step + sub) & mask;
            const HashSlot hs = slots[s];
            const unsigned hit = __ballot_sync(group, hs.key == key) & group;
            const unsigned empty = __ballot_sync(group, hs.key == kEmptyKey) & group;
            // first empty or hit in probe order decides
            const unsigned shift = threadIdx.x & 24;
            const unsigned h8 = (hit >> shift) & 0xFFu, e8 = (empty >> shift) & 0xFFu;
            const int fh = h8 ? __ffs(h8) - 1 : 8, fe = e8 ? __ffs(e8) - 1 : 8;
            if (fh < 8 && fh < fe) {
                result = __shfl_sync(group, hs.val, (threadIdx.x & 24) + fh);
                done = true;
            } else if (fe < 8) {
                done = true;
            } else if (step > mask) {
                done = true;
            }
        }
    }
    if (have && sub == 0) out[q] = result;
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

static inline unsigned grid_for(uint64_t n, unsigned per_block) {
    return static_cast<unsigned>((n + per_block - 1) / per_block);
}

void launch_keyset_clear(KeySet& ks, cudaStream_t s) {
    k_keyset_clear<<<1184, 256, 0, s>>>(ks.slots, ks.mask + 1);
}

void launch_points_to_keys(const double* xyz, uint64_t n, double L, KeySet ks,
                           unsigned long long* count, uint32_t* flags, cudaStream_t s) {
    if (!n) return;
    k_points_to_keys<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, L, ks, count, flags);
}

void launch_depth_to_keys(const float* depth, const svr_camera* cams, uint32_t n_frames, int32_t W,
                          int32_t H, const double* scales, int32_t rows, int32_t cols, double L,
                          KeySet ks, unsigned long long* count, unsigned long long* pixels,
                          uint32_t* flags, double* tab, cudaStream_t s) {
    const uint64_t n = static_cast<uint64_t>(W) * H * n_frames;
    if (!n) return;
    k_frame_tables<<<n_frames, 256, 0, s>>>(cams, W, H, tab);
    const uint64_t want = (static_cast<uint64_t>(n_frames) * H + 7) / 8, cap = sm_count() * 8ull;  // 8 rows per CTA
    k_depth_to_keys<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, s>>>(
        depth, cams, tab, n_frames, W, H, scales, rows, cols, L, ks, count, pixels, flags);
}

void launch_dilate(const unsigned long long* base, uint64_t nbase, int32_t R, KeySet ks,
                   unsigned long long* count, uint32_t* flags, cudaStream_t s) {
    const uint64_t side = 2 * static_cast<uint64_t>(R) + 1;
    const uint64_t n = nbase * side * side * side;
    if (!n) return;
    k_dilate<<<grid_for(n, 256), 256, 0, s>>>(base, nbase, R, ks, count, flags);
}

void launch_filter_fresh(const GridView& g, const unsigned long long* keys, uint64_t n,
                         unsigned long long* fresh, unsigned long long* nfresh, cudaStream_t s) {
    if (!n) return;
    k_filter_fresh<<<grid_for(n, 256), 256, 0, s>>>(g, keys, n, fresh, nfresh);
}

// Ascending sort of n 64-bit keys in place; tmp must hold sort_keys_tmp_bytes(n).
size_t sort_keys_tmp_bytes(uint64_t n) {
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, static_cast<unsigned long long*>(nullptr),
                                   static_cast<unsigned long long*>(nullptr), static_cast<int>(n), 0, 63);
    return ((need + 255) / 256) * 256 + n * sizeof(unsigned long long) + 256;
}
void launch_sort_keys(unsigned long long* keys, uint64_t n, void* tmp, cudaStream_t s) {
    if (n < 2) return;
    size_t need = 0;
    SVR_LCK(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, keys, static_cast<int>(n), 0, 63, s));
    auto* alt = reinterpret_cast<unsigned long long*>(static_cast<char*>(tmp) + ((need + 255) / 256) * 256);
    SVR_LCK(cudaMemcpyAsync(alt, keys, n * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    SVR_LCK(cub::DeviceRadixSort::SortKeys(tmp, need, alt, keys, static_cast<int>(n), 0, 63, s));
}

void launch_hash_insert(HashSlot* slots, unsigned long long mask, const unsigned long long* keys,
                        uint64_t n, uint32_t first, int32_t* coords4, cudaStream_t s) {
    if (!n) return;
    k_hash_insert<<<grid_for(n * 8, 256), 256, 0, s>>>(slots, mask, keys, n, first, coords4);
}

void launch_hash_find(const HashSlot* slots, unsigned long long mask, const int32_t* coords3,
                      uint64_t n, uint32_t* out, cudaStream_t s) {
    if (!n) return;
    k_hash_find<<<grid_for(n * 8, 256), 256, 0, s>>>(slots, mask, coords3, n, out);
}

}  // namespace svr_internal
