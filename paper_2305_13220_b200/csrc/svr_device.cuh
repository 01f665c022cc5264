// Device-side views and helpers shared by the sm_100a kernels.
//
// HBM layout:
//   slots   : HashSlot[pow2 >= 2*capacity]  {u64 packed key, u32 block index, u32 pad}
//   pay     : float4[A*512]  (sdf, r, g, b) per voxel, x fastest (grid.hpp:142-147)
//   weight  : float[A*512]   (kept for get_payload / SDGV round trips)
//   logits  : float[A*512*C] interleaved like the reference (grid.hpp:66)
//   vmask   : u32[A*16]      512-bit "weight > 0" mask per block (grid.hpp:58-59)
//   meta    : u32[A]         bit0 = every voxel of the block is valid
//   grad    : float4[A*512]  (g_sdf, g_r, g_g, g_b) -- one 16 B red.global.add.v4 per corner
//   active  : u8[A]          block received a scatter since the last grad zero
//   dense   : u32[dx*dy*dz]  block index (| 1<<31 when all-valid) over the block AABB,
//                            0xFFFFFFFF = unallocated; occ: bit per AABB cell
//   nbr     : u32[A*8]       entries of the +x/+y/+z neighbour blocks (trilinear corners
//                            that cross a block face resolve with one L1-resident load)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace svr_dev {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;
constexpr uint32_t kFullBit = 0x80000000u;
constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int kRes = 8;        // block resolution
constexpr int kVox = 512;      // voxels per block
constexpr uint32_t kNoBrick = 0x80000000u;  // GridView::sbinfo: superblock without a brick
constexpr uint64_t kMaxBlocks = 1ull << 23;  // 32-bit voxel addresses: block * 512 + local
constexpr int32_t kCoordLim = 1 << 20;

struct __align__(16) HashSlot {
    unsigned long long key;
    uint32_t val;
    uint32_t pad;
};

__host__ __device__ inline bool packable(int32_t x, int32_t y, int32_t z) {
    return x >= -kCoordLim && x < kCoordLim && y >= -kCoordLim && y < kCoordLim &&
           z >= -kCoordLim && z < kCoordLim;
}
// (z, y, x) lexicographic order == numeric order of the packed key.
__host__ __device__ inline unsigned long long pack_key(int32_t x, int32_t y, int32_t z) {
    return (static_cast<unsigned long long>(z + kCoordLim) << 42) |
           (static_cast<unsigned long long>(y + kCoordLim) << 21) |
           static_cast<unsigned long long>(x + kCoordLim);
}
__host__ __device__ inline void unpack_key(unsigned long long k, int32_t& x, int32_t& y, int32_t& z) {
    const unsigned long long m = (1ull << 21) - 1;
    x = static_cast<int32_t>(k & m) - kCoordLim;
    y = static_cast<int32_t>((k >> 21) & m) - kCoordLim;
    z = static_cast<int32_t>((k >> 42) & m) - kCoordLim;
}
// splitmix64 finaliser: slot positions are not observable, only
// find() results are, so the device table uses its own mixer and a power-of-two size.
__host__ __device__ inline unsigned long long mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

struct GridView {
    const HashSlot* slots;
    unsigned long long slot_mask;
    const uint32_t* dense;
    const uint32_t* occ;
    const float4* pay;
    const uint32_t* vmask;
    const uint32_t* meta;
    const float* logits;
    const uint32_t* nbr;    // [A][8]: entry of block + (k&1, k>>1&1, k>>2), k = 0..7
    const uint8_t* bdist;   // dense mode: Chebyshev distance (blocks, capped) to the nearest
                            // allocated block per AABB cell; 0 = allocated
    const uint8_t* sbdist;  // hash mode: the same over 8^3-block superblocks (superblock units)
    int32_t sb_lo[3], sb_dim[3];
    const uint32_t* sbinfo; // hash mode: per superblock, its brick (superblock distance <= 1) or
                            // kNoBrick | superblock distance
    const uint8_t* bricks;  // [brick][512] block distances (capped at 9) of those superblocks
    float4* grad;
    uint8_t* active;
    uint8_t* touch;         // [A][8]: a valid sample with base block b and face-crossing mask k
                            // was scattered (k_backward*); k_touch_expand folds it into active
    int32_t lo[3], hi[3];   // block AABB (grid.hpp:222)
    int32_t dim[3];         // hi - lo + 1
    int use_dense;
    uint32_t n_blocks;
    int32_t C;
    double h, inv_h, L;
};

__device__ __forceinline__ uint32_t hash_find(const GridView& g, unsigned long long key) {
    unsigned long long i = mix64(key) & g.slot_mask;
    for (;;) {
        const HashSlot s = g.slots[i];
        if (s.key == key) return s.val;
        if (s.key == kEmptyKey) return kInvalid;
        i = (i + 1) & g.slot_mask;
    }
}

// Block index (| kFullBit when the block is fully observed) or kInvalid.
__device__ __forceinline__ uint32_t lookup_block(const GridView& g, int32_t bx, int32_t by,
                                                 int32_t bz) {
    const uint32_t x = static_cast<uint32_t>(bx - g.lo[0]);
    const uint32_t y = static_cast<uint32_t>(by - g.lo[1]);
    const uint32_t z = static_cast<uint32_t>(bz - g.lo[2]);
    if (x >= static_cast<uint32_t>(g.dim[0]) || y >= static_cast<uint32_t>(g.dim[1]) ||
        z >= static_cast<uint32_t>(g.dim[2]))
        return kInvalid;
    if (g.use_dense)
        return __ldg(g.dense + (static_cast<size_t>(z) * g.dim[1] + y) * g.dim[0] + x);
    const uint32_t idx = hash_find(g, pack_key(bx, by, bz));
    if (idx == kInvalid) return kInvalid;
    return idx | ((__ldg(g.meta + idx) & 1u) ? kFullBit : 0u);
}

// allocated? (DDA test, grid.cpp:317-318)
__device__ __forceinline__ bool block_allocated(const GridView& g, int32_t bx, int32_t by,
                                                int32_t bz) {
    const uint32_t x = static_cast<uint32_t>(bx - g.lo[0]);
    const uint32_t y = static_cast<uint32_t>(by - g.lo[1]);
    const uint32_t z = static_cast<uint32_t>(bz - g.lo[2]);
    if (x >= static_cast<uint32_t>(g.dim[0]) || y >= static_cast<uint32_t>(g.dim[1]) ||
        z >= static_cast<uint32_t>(g.dim[2]))
        return false;
    if (g.use_dense) {
        const size_t cell = (static_cast<size_t>(z) * g.dim[1] + y) * g.dim[0] + x;
        return (__ldg(g.occ + (cell >> 5)) >> (cell & 31)) & 1u;
    }
    return hash_find(g, pack_key(bx, by, bz)) != kInvalid;
}

__device__ __forceinline__ bool voxel_valid(const GridView& g, uint32_t entry, uint32_t local) {
    if (entry & kFullBit) return true;
    const uint32_t blk = entry & ~kFullBit;
    return (__ldg(g.vmask + blk * 16u + (local >> 5)) >> (local & 31)) & 1u;
}

// gather_impl over CornerCacheD (grid.cpp:112-155) in fp64 with the reference's operation
// order (explicit _rn so nothing is contracted): corner c takes bit a of c on axis a,
// w_c = (wx wy) wz, dw_c[a] = ((+-1 inv_h) w_other1) w_other2.  False when a corner's block
// is missing or its voxel unobserved.
__device__ __forceinline__ bool gather_fp64(const GridView& g, const double x[3], uint32_t gidx[8],
                                            double w[8], double dw[8][3]) {
    double fx[3];
    int base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double gg = __dmul_rn(x[a], g.inv_h);
        const double fl = floor(gg);
        base[a] = static_cast<int>(fl);
        fx[a] = __dsub_rn(gg, fl);
    }
    const double w0[3] = {__dsub_rn(1.0, fx[0]), __dsub_rn(1.0, fx[1]), __dsub_rn(1.0, fx[2])};
    if (g.n_blocks == 0) return false;
    int32_t lbx = INT32_MIN, lby = 0, lbz = 0;
    uint32_t le = kInvalid;
    for (int c = 0; c < 8; ++c) {
        const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
        const int vx = base[0] + cx, vy = base[1] + cy, vz = base[2] + cz;
        const int32_t bx = vx >> 3, by = vy >> 3, bz = vz >> 3;
        if (bx != lbx || by != lby || bz != lbz) {
            lbx = bx, lby = by, lbz = bz;
            le = lookup_block(g, bx, by, bz);
        }
        if (le == kInvalid) return false;
        const uint32_t local = (vx & 7) + 8 * ((vy & 7) + 8 * (vz & 7));
        if (!voxel_valid(g, le, local)) return false;
        gidx[c] = (le & ~kFullBit) * 512u + local;
        const double wx = cx ? fx[0] : w0[0];
        const double wy = cy ? fx[1] : w0[1];
        const double wz = cz ? fx[2] : w0[2];
        w[c] = __dmul_rn(__dmul_rn(wx, wy), wz);
        dw[c][0] = __dmul_rn(__dmul_rn(__dmul_rn(cx ? 1.0 : -1.0, g.inv_h), wy), wz);
        dw[c][1] = __dmul_rn(__dmul_rn(__dmul_rn(cy ? 1.0 : -1.0, g.inv_h), wx), wz);
        dw[c][2] = __dmul_rn(__dmul_rn(__dmul_rn(cz ? 1.0 : -1.0, g.inv_h), wx), wy);
    }
    return true;
}

// std::min / std::max argument semantics (ties and NaN return the first argument).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// ScaleField::lookup + value (scale_field.cpp:21-60) at integer pixel (x, y), fp64 with
// the reference's operation order.
__device__ __forceinline__ double scale_field_value(const double* grid, int rows, int cols, int W,
                                                    int H, int x, int y) {
    const double sx = __ddiv_rn(static_cast<double>(cols - 1), static_cast<double>(W - 1));
    const double sy = __ddiv_rn(static_cast<double>(rows - 1), static_cast<double>(H - 1));
    double gx = __dmul_rn(static_cast<double>(x), sx);
    double gy = __dmul_rn(static_cast<double>(y), sy);
    const double cmax = static_cast<double>(cols - 1), rmax = static_cast<double>(rows - 1);
    gx = gx < 0.0 ? 0.0 : (cmax < gx ? cmax : gx);
    gy = gy < 0.0 ? 0.0 : (rmax < gy ? rmax : gy);
    const int c0 = min(static_cast<int>(gx), cols - 2);
    const int r0 = min(static_cast<int>(gy), rows - 2);
    const double fx = __dsub_rn(gx, static_cast<double>(c0));
    const double fy = __dsub_rn(gy, static_cast<double>(r0));
    const int b = r0 * cols + c0;
    const double w[4] = {__dmul_rn(__dsub_rn(1.0, fx), __dsub_rn(1.0, fy)), __dmul_rn(fx, __dsub_rn(1.0, fy)),
                         __dmul_rn(__dsub_rn(1.0, fx), fy), __dmul_rn(fx, fy)};
    const int idx[4] = {b, b + 1, b + cols, b + cols + 1};
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v = __dadd_rn(v, __dmul_rn(w[k], __ldg(grid + idx[k])));
    return v;
}

// floor_div by 8 (grid.hpp:207-210) == arithmetic shift.
__device__ __forceinline__ int32_t fdiv8(int32_t v) { return v >> 3; }

}  // namespace svr_dev
