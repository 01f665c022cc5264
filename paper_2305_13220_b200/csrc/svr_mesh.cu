// sm_100a marching cubes over the sparse-dense grid (the reference's
// svr::marching_cubes, proj/src/core/meshing.cpp:168-273), same mesh word for word:
//   K14a k_mc_count   -- CTA per block, thread per cell: 8 corners through the neighbour
//                        table, case index, triangles per cell, per-block total
//   K14b k_mc_emit    -- CTA scan of the per-cell counts; every triangle corner gets its
//                        edge key (lower voxel, axis) and its fp64 position, in the
//                        reference's (block, z, y, x, triangle, corner) order
//   K14c dedup        -- stable radix sort of (key, slot): the first slot of each key run is
//                        the reference's first occurrence, vertex ids = scan over those
//   K14d k_mc_keep / k_mc_compact -- drop degenerate / zero-area triangles (meshing.cpp:243-250)
//   K14e k_mc_attrs   -- fp64 trilinear normal / colour / argmax label per vertex
// The 256-case table is built on the host from the same rules meshing.cpp:56-150 states
// (restated in build_table below) and lives in constant memory.
#include <algorithm>
#include <array>
#include <mutex>
#include <set>
#include <vector>

#include <cub/cub.cuh>

#include "svr_internal.h"

namespace svr_dev {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__constant__ uint8_t c_mc_count[256];
__constant__ uint8_t c_mc_tri[256][5][3];
__constant__ uint8_t c_edge_a[12], c_edge_b[12], c_edge_axis[12];

struct McView {
    GridView g;
    const int4* coords;
    const uint32_t* nbr;
    double iso;
    int32_t lo_vox[3];  // AABB min voxel, edge keys are relative to it
};

// Case index of cell v of block b, or -1 when a corner is unallocated / unobserved
// (meshing.cpp:175-184, 196-207).  s[] receives the corner sdfs as doubles.
__device__ __forceinline__ int cell_case(const McView& m, uint32_t b, int v, double s[8]) {
    const int lx = v & 7, ly = (v >> 3) & 7, lz = v >> 6;
    const uint32_t* nb = m.nbr + static_cast<size_t>(b) * 8;
    int cfg = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int x = lx + (c & 1), y = ly + ((c >> 1) & 1), z = lz + (c >> 2);
        const int o = (x >> 3) | ((y >> 3) << 1) | ((z >> 3) << 2);
        const uint32_t e = __ldg(nb + o);  // entry of block + (o&1, o>>1&1, o>>2)
        if (e == kInvalid) return -1;
        const uint32_t local = (x & 7) + 8 * (y & 7) + 64 * (z & 7);
        if (!voxel_valid(m.g, e, local)) return -1;
        s[c] = static_cast<double>(__ldg(m.g.pay + static_cast<size_t>(e & ~kFullBit) * kVox + local).x);
        if (s[c] < m.iso) cfg |= 1 << c;
    }
    return cfg;
}

__global__ void __launch_bounds__(512) k_mc_count(McView m, uint32_t* block_tris) {
    const uint32_t b = blockIdx.x;
    double s[8];
    const int cfg = cell_case(m, b, threadIdx.x, s);
    uint32_t n = cfg >= 0 ? c_mc_count[cfg] : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) n += __shfl_xor_sync(kFull, n, off);
    __shared__ uint32_t part[16];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 16; ++w) t += part[w];
        block_tris[b] = t;
    }
}

__global__ void __launch_bounds__(512) k_mc_emit(McView m, const uint32_t* __restrict__ block_tris,
                                                 const uint32_t* __restrict__ block_off,
                                                 unsigned long long* keys, uint32_t* slots, double* pos) {
    const uint32_t b = blockIdx.x;
    if (block_tris[b] == 0) return;
    using Scan = cub::BlockScan<uint32_t, 512>;
    __shared__ typename Scan::TempStorage tmp;
    const int v = threadIdx.x;
    double s[8];
    const int cfg = cell_case(m, b, v, s);
    const uint32_t n = cfg >= 0 ? c_mc_count[cfg] : 0u;
    uint32_t first;
    Scan(tmp).ExclusiveSum(n, first);
    if (!n) return;
    const int4 bc = m.coords[b];
    const int ax = bc.x * kRes + (v & 7), ay = bc.y * kRes + ((v >> 3) & 7), az = bc.z * kRes + (v >> 6);
    const uint64_t t0 = block_off[b] + first;
    for (uint32_t i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int e = c_mc_tri[cfg][i][k];
            const int ca = c_edge_a[e], cb = c_edge_b[e], axis = c_edge_axis[e];
            const int va[3] = {ax + (ca & 1), ay + ((ca >> 1) & 1), az + (ca >> 2)};
            // t = (iso - sa) / (sb - sa); p = voxel_to_world(va); p[axis] += t h (meshing.cpp:217-221)
            const double tt = __ddiv_rn(__dsub_rn(m.iso, s[ca]), __dsub_rn(s[cb], s[ca]));
            double p[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) p[a] = __dmul_rn(static_cast<double>(va[a]), m.g.h);
            p[axis] = __dadd_rn(p[axis], __dmul_rn(tt, m.g.h));
            const uint64_t slot = 3 * (t0 + i) + k;
            keys[slot] = static_cast<unsigned long long>(va[0] - m.lo_vox[0]) |
                         (static_cast<unsigned long long>(va[1] - m.lo_vox[1]) << 21) |
                         (static_cast<unsigned long long>(va[2] - m.lo_vox[2]) << 42) |
                         (static_cast<unsigned long long>(axis) << 62);
            slots[slot] = static_cast<uint32_t>(slot);
            pos[3 * slot] = p[0], pos[3 * slot + 1] = p[1], pos[3 * slot + 2] = p[2];
        }
    }
}

// Sorted run heads: first[slot] = 1 at the first (lowest) slot of every key; headpos = i at
// a head else 0 (a max-scan then gives each element its run head's sorted position).
__global__ void k_mc_heads(const unsigned long long* __restrict__ ks, const uint32_t* __restrict__ ss,
                           uint64_t n, uint32_t* first, uint32_t* headpos) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool head = i == 0 || ks[i] != ks[i - 1];
    first[ss[i]] = head;
    headpos[i] = head ? static_cast<uint32_t>(i) : 0u;
}

__global__ void k_mc_resolve(const uint32_t* __restrict__ ss, const uint32_t* __restrict__ headpos,
                             const uint32_t* __restrict__ vid, const double* __restrict__ pos, uint64_t n,
                             uint32_t* tri_idx, double* vout) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = ss[i], hp = headpos[i];
    const uint32_t hs = ss[hp];
    const uint32_t id = vid[hs];
    tri_idx[s] = id;
    if (hp == i) {  // first occurrence: its position is the vertex (meshing.cpp:237-238)
        vout[3 * static_cast<size_t>(id)] = pos[3 * static_cast<size_t>(s)];
        vout[3 * static_cast<size_t>(id) + 1] = pos[3 * static_cast<size_t>(s) + 1];
        vout[3 * static_cast<size_t>(id) + 2] = pos[3 * static_cast<size_t>(s) + 2];
    }
}

// meshing.cpp:243-250: distinct indices and 0.5 |e1 x e2| > 1e-12 (Eigen cross / norm order)
__global__ void k_mc_keep(const uint32_t* __restrict__ tri_idx, const double* __restrict__ v, uint64_t T,
                          uint32_t* keep) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const uint32_t i0 = tri_idx[3 * t], i1 = tri_idx[3 * t + 1], i2 = tri_idx[3 * t + 2];
    bool ok = i0 != i1 && i1 != i2 && i0 != i2;
    if (ok) {
        const double* a = v + 3 * static_cast<size_t>(i0);
        const double* b = v + 3 * static_cast<size_t>(i1);
        const double* c = v + 3 * static_cast<size_t>(i2);
        const double e1[3] = {__dsub_rn(b[0], a[0]), __dsub_rn(b[1], a[1]), __dsub_rn(b[2], a[2])};
        const double e2[3] = {__dsub_rn(c[0], a[0]), __dsub_rn(c[1], a[1]), __dsub_rn(c[2], a[2])};
        const double x = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
        const double y = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
        const double z = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
        const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
        ok = __dmul_rn(0.5, __dsqrt_rn(n2)) > 1e-12;
    }
    keep[t] = ok;
}

__global__ void k_mc_compact(const uint32_t* __restrict__ tri_idx, const uint32_t* __restrict__ keep,
                             const uint32_t* __restrict__ off, uint64_t T, int32_t* out) {
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= T || !keep[t]) return;
    const size_t o = 3 * static_cast<size_t>(off[t]);
    out[o] = static_cast<int32_t>(tri_idx[3 * t]);
    out[o + 1] = static_cast<int32_t>(tri_idx[3 * t + 1]);
    out[o + 2] = static_cast<int32_t>(tri_idx[3 * t + 2]);
}

// meshing.cpp:254-270: gather_corners (fp64) at the vertex; normal = normalized gradient when
// |g| > 1e-12 else +z; colour clamped to [0, 1]; label = first argmax of the logits.
__global__ void __launch_bounds__(256) k_mc_attrs(GridView g, const double* __restrict__ v, uint64_t nv,
                                                  double* nrm, double* col, int32_t* lab) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const double x[3] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    uint32_t gidx[8];
    double w[8], dw[8][3];
    double n[3] = {0.0, 0.0, 1.0}, c[3] = {0.0, 0.0, 0.0};
    int32_t label = 0;
    if (gather_fp64(g, x, gidx, w, dw)) {
        double gr[3] = {0.0, 0.0, 0.0}, cc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 p = __ldg(g.pay + gidx[k]);
            gr[0] = __dadd_rn(gr[0], __dmul_rn(dw[k][0], static_cast<double>(p.x)));
            gr[1] = __dadd_rn(gr[1], __dmul_rn(dw[k][1], static_cast<double>(p.x)));
            gr[2] = __dadd_rn(gr[2], __dmul_rn(dw[k][2], static_cast<double>(p.x)));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 p = __ldg(g.pay + gidx[k]);
            cc[0] = __dadd_rn(cc[0], __dmul_rn(w[k], static_cast<double>(p.y)));
            cc[1] = __dadd_rn(cc[1], __dmul_rn(w[k], static_cast<double>(p.z)));
            cc[2] = __dadd_rn(cc[2], __dmul_rn(w[k], static_cast<double>(p.w)));
        }
        const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(gr[0], gr[0]), __dmul_rn(gr[1], gr[1])),
                                    __dmul_rn(gr[2], gr[2]));
        const double len = __dsqrt_rn(n2);
        if (len > 1e-12) {
            n[0] = __ddiv_rn(gr[0], len), n[1] = __ddiv_rn(gr[1], len), n[2] = __ddiv_rn(gr[2], len);
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] = smin(smax(cc[a], 0.0), 1.0);
        double best = 0.0;
        for (int k = 0; k < g.C; ++k) {
            double acc = 0.0;
            for (int j = 0; j < 8; ++j)
                acc = __dadd_rn(acc, __dmul_rn(w[j], static_cast<double>(__ldg(g.logits + static_cast<size_t>(gidx[j]) * g.C + k))));
            if (k == 0 || best < acc) {  // std::max_element: first of the largest
                best = acc;
                label = k;
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        nrm[3 * i + a] = n[a];
        col[3 * i + a] = c[a];
    }
    lab[i] = label;
}

unsigned grid_for(uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

// The case table (meshing.cpp:56-150 rules, see svr_internal.h): edges = one-bit corner
// pairs, id = axis * 4 + rank of the lower corner; faces = cyclic quads (b, b+u, b+u+v, b+v);
// crossings pair up per face (4 crossings: each inside corner cut off by its two edges);
// segments chain into loops from the lowest edge, reversed when their midpoint normal
// points toward the inside corners, fan-triangulated.
struct Table {
    uint8_t count[256];
    uint8_t tri[256][5][3];
    uint8_t ea[12], eb[12], eaxis[12];
};

Table build_table() {
    Table t{};
    for (int a = 0; a < 3; ++a)
        for (int c = 0, r = 0; c < 8; ++c)
            if (!((c >> a) & 1)) {
                t.ea[a * 4 + r] = static_cast<uint8_t>(c);
                t.eb[a * 4 + r] = static_cast<uint8_t>(c | (1 << a));
                t.eaxis[a * 4 + r] = static_cast<uint8_t>(a);
                ++r;
            }
    auto edge = [&](int p, int q) {
        const int lo = std::min(p, q), hi = std::max(p, q);
        for (int e = 0; e < 12; ++e)
            if (t.ea[e] == lo && t.eb[e] == hi) return e;
        return -1;
    };
    std::array<std::array<int, 4>, 6> faces{};
    for (int a = 0, f = 0; a < 3; ++a) {
        const int u = a == 0 ? 1 : 0, w = a == 2 ? 1 : 2;
        for (int side = 0; side < 2; ++side, ++f) {
            const int base = side << a;
            faces[f] = {base, base | (1 << u), base | (1 << u) | (1 << w), base | (1 << w)};
        }
    }
    for (int cfg = 0; cfg < 256; ++cfg) {
        auto inside = [&](int c) { return (cfg >> c) & 1; };
        int link[12][2], deg[12] = {};
        auto pair = [&](int e, int f) {
            link[e][deg[e]++] = f;
            link[f][deg[f]++] = e;
        };
        for (const auto& q : faces) {
            int cut[4], n = 0;
            for (int i = 0; i < 4; ++i)
                if (inside(q[i]) != inside(q[(i + 1) % 4])) cut[n++] = edge(q[i], q[(i + 1) % 4]);
            if (n == 2) pair(cut[0], cut[1]);
            if (n == 4)
                for (int k = 0; k < 4; ++k)
                    if (inside(q[k])) pair(edge(q[(k + 3) % 4], q[k]), edge(q[k], q[(k + 1) % 4]));
        }
        bool used[12] = {};
        std::vector<std::array<int, 3>> tris;
        for (int s = 0; s < 12; ++s) {
            if (deg[s] != 2 || used[s]) continue;
            std::vector<int> loop;
            for (int cur = s, prev = -1;;) {
                loop.push_back(cur);
                used[cur] = true;
                const int nx = link[cur][0] == prev ? link[cur][1] : link[cur][0];
                prev = cur;
                cur = nx;
                if (cur == s) break;
            }
            if (loop.size() < 3) continue;
            auto mid = [&](int e, int a) { return 0.5 * (((t.ea[e] >> a) & 1) + ((t.eb[e] >> a) & 1)); };
            double nr[3] = {0, 0, 0};
            for (size_t i = 0; i < loop.size(); ++i) {
                const int e = loop[i], f = loop[(i + 1) % loop.size()];
                for (int a = 0; a < 3; ++a) {
                    const int a1 = (a + 1) % 3, a2 = (a + 2) % 3;
                    nr[a] += mid(e, a1) * mid(f, a2) - mid(e, a2) * mid(f, a1);
                }
            }
            double sin_[3] = {0, 0, 0}, sout[3] = {0, 0, 0};
            int nin = 0, nout = 0;
            for (int c = 0; c < 8; ++c) {
                for (int a = 0; a < 3; ++a) (inside(c) ? sin_ : sout)[a] += (c >> a) & 1;
                ++(inside(c) ? nin : nout);
            }
            double d = 0.0;
            for (int a = 0; a < 3; ++a) d += nr[a] * (sout[a] / std::max(nout, 1) - sin_[a] / std::max(nin, 1));
            if (d < 0.0) std::reverse(loop.begin(), loop.end());
            for (size_t i = 1; i + 1 < loop.size(); ++i) tris.push_back({loop[0], loop[i], loop[i + 1]});
        }
        t.count[cfg] = static_cast<uint8_t>(tris.size());
        for (size_t i = 0; i < tris.size() && i < 5; ++i)
            for (int k = 0; k < 3; ++k) t.tri[cfg][i][k] = static_cast<uint8_t>(tris[i][k]);
    }
    return t;
}

}  // namespace
}  // namespace svr_dev

namespace svr_internal {
using namespace svr_dev;

namespace {
struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    void* get(size_t bytes) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s) != cudaSuccess)
            throw Status{SVR_ERR_CUDA, "marching_cubes: out of device memory"};
        ptrs.push_back(p);
        return p;
    }
    template <typename T>
    T* as(size_t n) {
        return static_cast<T*>(get(n * sizeof(T)));
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Status{SVR_ERR_CUDA, std::string("marching_cubes: ") + what + ": " + cudaGetErrorString(e)};
}

std::mutex g_table_mu;
std::set<int> g_table_ready;  // devices whose constant-memory case table is loaded
}  // namespace

void MeshBufs::release() {
    for (void* p : {static_cast<void*>(v), static_cast<void*>(n), static_cast<void*>(c), static_cast<void*>(l),
                    static_cast<void*>(t)})
        if (p) cudaFree(p);
    v = n = c = nullptr;
    l = t = nullptr;
    cap_v = cap_t = nv = nt = 0;
}

void MeshBufs::reserve(uint64_t want_v, uint64_t want_t) {
    if (want_v > cap_v) {
        for (void* p : {static_cast<void*>(v), static_cast<void*>(n), static_cast<void*>(c), static_cast<void*>(l)})
            if (p) cudaFree(p);
        v = n = c = nullptr;
        l = nullptr;
        cap_v = 0;
        ck(cudaMalloc(&v, want_v * 24), "vertices");
        ck(cudaMalloc(&n, want_v * 24), "normals");
        ck(cudaMalloc(&c, want_v * 24), "colors");
        ck(cudaMalloc(&l, want_v * 4), "labels");
        cap_v = want_v;
    }
    if (want_t > cap_t) {
        if (t) cudaFree(t);
        t = nullptr;
        cap_t = 0;
        ck(cudaMalloc(&t, want_t * 12), "triangles");
        cap_t = want_t;
    }
}

void run_marching_cubes(const GridView& g, const int32_t* coords4, const uint32_t* nbr, const int32_t* lo_block,
                        double iso, MeshBufs& out, cudaStream_t s) {
    int dev = 0;
    ck(cudaGetDevice(&dev), "device");
    {
        std::lock_guard<std::mutex> lock(g_table_mu);
        if (!g_table_ready.count(dev)) {
        const Table t = build_table();
        ck(cudaMemcpyToSymbol(c_mc_count, t.count, sizeof(t.count)), "table");
        ck(cudaMemcpyToSymbol(c_mc_tri, t.tri, sizeof(t.tri)), "table");
        ck(cudaMemcpyToSymbol(c_edge_a, t.ea, 12), "table");
        ck(cudaMemcpyToSymbol(c_edge_b, t.eb, 12), "table");
        ck(cudaMemcpyToSymbol(c_edge_axis, t.eaxis, 12), "table");
        g_table_ready.insert(dev);
        }
    }
    out.nv = out.nt = 0;
    const uint32_t A = g.n_blocks;
    if (!A) return;
    McView m{g, reinterpret_cast<const int4*>(coords4), nbr, iso,
             {lo_block[0] * kRes, lo_block[1] * kRes, lo_block[2] * kRes}};
    Scratch sc{s, {}};
    uint32_t* btris = sc.as<uint32_t>(A);
    uint32_t* boff = sc.as<uint32_t>(A);
    k_mc_count<<<A, 512, 0, s>>>(m, btris);
    size_t tb = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, btris, boff, static_cast<int>(A), s), "scan / sort");
    void* tmp = sc.get(tb);
    ck(cub::DeviceScan::ExclusiveSum(tmp, tb, btris, boff, static_cast<int>(A), s), "scan / sort");
    uint32_t h2[2];
    ck(cudaMemcpyAsync(&h2[0], boff + A - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaMemcpyAsync(&h2[1], btris + A - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaStreamSynchronize(s), "count");
    const uint64_t T = static_cast<uint64_t>(h2[0]) + h2[1];
    if (T == 0) return;
    const uint64_t N = 3 * T;
    if (N >= (1ull << 31)) throw Status{SVR_ERR_CAPACITY, "marching_cubes: more than 2^31 triangle corners"};
    auto* keys = sc.as<unsigned long long>(N);
    auto* keys2 = sc.as<unsigned long long>(N);
    auto* slots = sc.as<uint32_t>(N);
    auto* slots2 = sc.as<uint32_t>(N);
    auto* pos = sc.as<double>(3 * N);
    k_mc_emit<<<A, 512, 0, s>>>(m, btris, boff, keys, slots, pos);
    // stable sort by edge key: within a key, slots stay ascending
    cub::DoubleBuffer<unsigned long long> kb(keys, keys2);
    cub::DoubleBuffer<uint32_t> vb(slots, slots2);
    tb = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, static_cast<int>(N), 0, 64, s), "scan / sort");
    tmp = sc.get(tb);
    ck(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, static_cast<int>(N), 0, 64, s), "scan / sort");
    auto* first = sc.as<uint32_t>(N);
    auto* headpos = sc.as<uint32_t>(N);
    auto* headmax = sc.as<uint32_t>(N);
    auto* vid = sc.as<uint32_t>(N);
    k_mc_heads<<<grid_for(N, 256), 256, 0, s>>>(kb.Current(), vb.Current(), N, first, headpos);
    tb = 0;
    ck(cub::DeviceScan::InclusiveScan(nullptr, tb, headpos, headmax, cub::Max(), static_cast<int>(N), s), "scan / sort");
    size_t tb2 = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb2, first, vid, static_cast<int>(N), s), "scan / sort");
    tmp = sc.get(std::max(tb, tb2));
    ck(cub::DeviceScan::InclusiveScan(tmp, tb, headpos, headmax, cub::Max(), static_cast<int>(N), s), "scan / sort");
    ck(cub::DeviceScan::ExclusiveSum(tmp, tb2, first, vid, static_cast<int>(N), s), "scan / sort");
    uint32_t hv[2];
    ck(cudaMemcpyAsync(&hv[0], vid + N - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaMemcpyAsync(&hv[1], first + N - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaStreamSynchronize(s), "count");
    const uint64_t nv = static_cast<uint64_t>(hv[0]) + hv[1];
    out.reserve(nv, T);
    auto* tri_idx = sc.as<uint32_t>(N);
    k_mc_resolve<<<grid_for(N, 256), 256, 0, s>>>(vb.Current(), headmax, vid, pos, N, tri_idx, out.v);
    auto* keep = sc.as<uint32_t>(T);
    auto* toff = sc.as<uint32_t>(T);
    k_mc_keep<<<grid_for(T, 256), 256, 0, s>>>(tri_idx, out.v, T, keep);
    tb = 0;
    ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, toff, static_cast<int>(T), s), "scan / sort");
    tmp = sc.get(tb);
    ck(cub::DeviceScan::ExclusiveSum(tmp, tb, keep, toff, static_cast<int>(T), s), "scan / sort");
    k_mc_compact<<<grid_for(T, 256), 256, 0, s>>>(tri_idx, keep, toff, T, out.t);
    k_mc_attrs<<<grid_for(nv, 256), 256, 0, s>>>(g, out.v, nv, out.n, out.c, out.l);
    ck(cudaMemcpyAsync(&hv[0], toff + T - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaMemcpyAsync(&hv[1], keep + T - 1, 4, cudaMemcpyDeviceToHost, s), "count");
    ck(cudaGetLastError(), "launch");
    ck(cudaStreamSynchronize(s), "count");
    out.nv = nv;
    out.nt = static_cast<uint64_t>(hv[0]) + hv[1];
}

}  // namespace svr_internal
