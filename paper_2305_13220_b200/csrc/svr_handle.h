// Internal host-side header of libsvr_b200.so: the svr_grid handle (one device + one stream,
// owner of all device memory) and the helpers every C-ABI translation unit shares --
// status exceptions, the guarded() ABI wrapper, host/device pointer staging.  The C-ABI
// itself is split over svr_grid.cu (handle, activation, payload, query, march, SDGV),
// svr_api_render.cu (render forward/backward, gradients, regularisers) and svr_api_more.cu
// (fusion, de-noising, losses / refinement batches, peer reduction, meshing).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "svr_internal.h"

namespace svr_host {
using namespace svr_dev;
using svr_internal::set_error;

struct Fail {
    int code;
    std::string msg;
};

#define SVR_CK(expr)                                                                        \
    do {                                                                                    \
        const cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess)                                                              \
            throw Fail{SVR_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)};   \
    } while (0)
#define SVR_LAUNCHED() SVR_CK(cudaGetLastError())

template <typename Fn>
inline int guarded(Fn&& fn) {
    try {
        fn();
        return SVR_OK;
    } catch (const Fail& f) {
        set_error(f.msg);
        return f.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return SVR_ERR_DATA;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SVR_ERR_DATA;
    }
}

inline bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        SVR_CK(cudaGetDevice(&prev));
        if (prev != dev) SVR_CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// Process-wide cache of device allocations (svr_grid.cu): blocks a handle gives back -- when
// it is destroyed or a buffer grows -- are kept mapped and handed to later requests of a
// similar size on the same device, instead of being returned with cudaFree and re-mapped by
// cudaMalloc (which costs ~0.3-1 ms per GB).  dev_alloc returns the block's true size;
// dev_release requires that no queued work still uses the block.  On cudaMalloc failure the
// device's cached blocks are freed and the allocation retried.
void* dev_alloc(size_t bytes, size_t* got);
void dev_release(void* p, size_t bytes, int device);

// Grow-only device buffer (on the caching allocator).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    void ensure(size_t need) {
        if (need <= bytes) return;
        release();
        SVR_CK(cudaGetDevice(&dev));
        p = dev_alloc(need, &bytes);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(dev, o.dev);
    }
    // as cudaFree did implicitly: the block's device is idle before the block is handed back
    void release() {
        if (!p) return;
        int cur = -1;
        cudaGetDevice(&cur);
        if (dev < 0) dev = cur;
        if (cur != dev) cudaSetDevice(dev);
        cudaDeviceSynchronize();
        if (cur != dev && cur >= 0) cudaSetDevice(cur);
        dev_release(p, bytes, dev);
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
};

// Host <-> device staging for one API call.  Device pointers pass through; host
// arrays are copied through stream-ordered temporaries, and the call synchronises
// before returning if any host array was involved.
struct Stage {
    cudaStream_t s;
    std::vector<void*> tmp;
    struct Out {
        void* host;
        void* dev;
        size_t bytes;
    };
    std::vector<Out> outs;
    bool host_involved = false;
    explicit Stage(cudaStream_t st) : s(st) {}
    void* alloc(size_t bytes) {
        void* d = nullptr;
        SVR_CK(cudaMallocAsync(&d, bytes, s));
        tmp.push_back(d);
        return d;
    }
    template <typename T>
    const T* in(const T* p, size_t n) {
        if (!p || n == 0 || is_device_ptr(p)) return p;
        host_involved = true;
        void* d = alloc(n * sizeof(T));
        SVR_CK(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, s));
        return static_cast<const T*>(d);
    }
    template <typename T>
    T* out(T* p, size_t n) {
        if (!p || n == 0 || is_device_ptr(p)) return p;
        host_involved = true;
        void* d = alloc(n * sizeof(T));
        outs.push_back({p, d, n * sizeof(T)});
        return static_cast<T*>(d);
    }
    void finish() {
        SVR_LAUNCHED();
        for (const Out& o : outs)
            SVR_CK(cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, s));
        outs.clear();
        for (void* p : tmp) cudaFreeAsync(p, s);
        tmp.clear();
        if (host_involved) SVR_CK(cudaStreamSynchronize(s));
    }
    ~Stage() {
        for (void* p : tmp) cudaFreeAsync(p, s);
    }
};

inline uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace svr_host

// internal header: the handle and the TUs that include it work in these namespaces
using namespace svr_dev;
using namespace svr_host;

struct svr_grid {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double h = 0, inv_h = 0, L = 0;
    int32_t C = 1;
    uint64_t capacity = 0;
    uint64_t nblk = 0;             // allocated blocks
    std::vector<int32_t> coords;   // host mirror, 3 per block: blocks [0, coords_synced) pulled
    uint64_t coords_synced = 0;
    void* pin = nullptr;           // pinned staging (host_coords, bounds)
    size_t pin_bytes = 0;
    DevBuf bounds_dev;
    int32_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};

    HashSlot* slots = nullptr;
    uint64_t nslots = 0;

    uint64_t cap_blocks = 0;  // rows allocated in the per-block arrays
    int32_t* coords4 = nullptr;
    float4* pay = nullptr;
    float* weight = nullptr;
    float* logits = nullptr;
    uint32_t* vmask = nullptr;
    uint32_t* meta = nullptr;
    float4* grad = nullptr;
    uint8_t* active = nullptr;
    uint8_t* touch = nullptr;  // [A][8] backward touch flags (GridView::touch), all zero between calls

    int lookup_pref = SVR_LOOKUP_AUTO;
    bool dense_dirty = true;
    int use_dense = 0;
    int32_t dim[3] = {0, 0, 0};
    DevBuf dense, occ, nbr, bdist, bdist_tmp;
    DevBuf sb_occ, sbdist, sbdist_tmp;  // hash mode: superblock occupancy + distance field
    DevBuf sb_info, brick_sb, brick_cnt, bricks, bricks_tmp;  // hash mode: block-distance bricks
    int use_sb = 0;
    uint32_t n_bricks = 0;
    int32_t sb_lo[3] = {0, 0, 0}, sb_dim[3] = {0, 0, 0};
    bool use_jump = true;   // march: exact empty-space jumps over the block-distance field

    // render context
    DevBuf ray_o, ray_d, counts, tbuf, nvalid;
    DevBuf ord_keys, ord_ids, ord_tmp;  // pre-march ray order (origin + direction keys)
    DevBuf ord_keys2, ord_ids2;         // post-march order (keys written by the march)
    DevBuf rec;                         // per-sample forward records for the backward
    bool ctx_rec = false;
    uint32_t* ctx_order = nullptr;
    // tuning knobs (svr_grid_set_tuning); none changes results
    // bit 1: order the march by origin + direction; bit 0: order forward/backward by the
    // block of each ray's first sample (3 = both)
    int ray_sort = 3;
    uint64_t sort_min_rays = 32768;  // smaller batches are rendered in caller order
    bool use_records = true;  // forward leaves 32 B/sample records; backward skips the re-gather
    bool bwd_pipe = true;     // persistent backward streaming records with cp.async.bulk
    int num_sms = 148;
    const double* ctx_o = nullptr;
    const double* ctx_d = nullptr;
    uint64_t ctx_n = 0;
    uint32_t ctx_S = 0;
    double ctx_step = 0, ctx_beta = 0;
    bool ctx_valid = false;

    DevBuf active_list, active_count;  // count: u64 + per-CTA scratch
    // multi-GPU reduction (svr_reduce.cu): union flags, its ascending list + device count,
    // the NCCL fallback's pack buffer, and the two interprocess-capable phase events
    DevBuf red_union, red_list, red_count, red_pack;
    cudaEvent_t red_done = nullptr, red_reduced = nullptr;
    DevBuf rms;                        // RMSProp state float4 [rms_blocks][512]
    uint64_t rms_blocks = 0;
    // fusion session: 32.32 fixed-point sums [fuse_blocks][4 + C][512] + counts [.][512]
    int fuse_flags = -1;
    uint64_t fuse_blocks = 0;
    uint32_t fuse_batch = 0;  // frames per k_fuse launch, 0 = auto
    DevBuf pay_spare, logits_spare;  // denoise output planes, swapped with pay / logits
    svr_internal::MeshBufs mesh;     // last svr_marching_cubes result
    DevBuf loss_acc;                 // svr_render_losses reduction scratch
    // "host_async" pipelined host I/O for render_forward / render_backward: pinned host arrays
    // move on two copy streams through double-buffered device slots, so the transfers of one
    // step overlap the kernels of the previous one; results are valid after synchronize.
    struct AsyncSlot {
        DevBuf o, d, up, out;
        cudaEvent_t in_ev = nullptr, up_ev = nullptr, fwd_ev = nullptr, out_ev = nullptr, free_ev = nullptr;
        bool used = false;
    };
    bool host_async = false;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    AsyncSlot aslot[2];
    int aslot_next = 0, ctx_aslot = -1;
    void ensure_async() {
        if (h2d) return;
        SVR_CK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        SVR_CK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (AsyncSlot& a : aslot)
            for (cudaEvent_t* e : {&a.in_ev, &a.up_ev, &a.fwd_ev, &a.out_ev, &a.free_ev})
                SVR_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    // Deferred zeroing ("zero_fused", default on): svr_grad_zero_active only compacts the
    // active list (device count) and leaves the zeroing pending; the next render_forward's
    // K5 warps store the zeros next to their ray work (the forward is latency bound, its DRAM
    // has room for the 1 GB of stores), and every other entry point runs the pending zeroing
    // kernel first (GridGuard).  Off: the zeroing kernel runs in order at once.
    bool zero_fused = true;
    bool zero_pending = false;
    void flush_zero() {
        if (!zero_pending) return;
        zero_pending = false;
        svr_internal::launch_grad_zero_active(grad, active, active_list.as<uint32_t>(),
                                              active_count.as<unsigned long long>(), static_cast<uint32_t>(n()),
                                              stream, 16u);
        SVR_LAUNCHED();
    }
    uint64_t spare_cap = 0;          // cap_blocks the spare pair was sized for
    DevBuf fuse_sum, fuse_cnt;
    DevBuf scratch_a, scratch_b, scratch_c, scratch_d, scratch_e, sort_tmp;

    uint64_t n() const { return nblk; }
    // host mirror of the block coordinates (x, y, z per block), pulled from coords4 lazily
    const std::vector<int32_t>& host_coords() {
        if (coords_synced < nblk) {
            const uint64_t cnt = nblk - coords_synced;
            int32_t* st = static_cast<int32_t*>(pinned(cnt * 16));
            SVR_CK(cudaMemcpyAsync(st, coords4 + coords_synced * 4, cnt * 16, cudaMemcpyDeviceToHost, stream));
            SVR_CK(cudaStreamSynchronize(stream));
            coords.resize(3 * nblk);
            int32_t* dst = coords.data() + 3 * coords_synced;
            for (uint64_t i = 0; i < cnt; ++i)
                dst[3 * i] = st[4 * i], dst[3 * i + 1] = st[4 * i + 1], dst[3 * i + 2] = st[4 * i + 2];
            coords_synced = nblk;
        }
        return coords;
    }
    // grow-only pinned host staging buffer
    void* pinned(size_t bytes) {
        if (bytes > pin_bytes) {
            if (pin) cudaFreeHost(pin);
            pin = nullptr;
            pin_bytes = 0;
            SVR_CK(cudaMallocHost(&pin, bytes));
            pin_bytes = bytes;
        }
        return pin;
    }

    ~svr_grid() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (cudaEvent_t e : {red_done, red_reduced})
            if (e) cudaEventDestroy(e);
        if (h2d) {
            cudaStreamSynchronize(h2d);
            cudaStreamSynchronize(d2h);
            for (AsyncSlot& a : aslot)
                for (cudaEvent_t e : {a.in_ev, a.up_ev, a.fwd_ev, a.out_ev, a.free_ev}) cudaEventDestroy(e);
            cudaStreamDestroy(h2d);
            cudaStreamDestroy(d2h);
        }
        if (slots) dev_release(slots, nslots * sizeof(HashSlot), device);
        const uint64_t cb = cap_blocks;
        const std::pair<void*, size_t> blocks[] = {
            {coords4, cb * 16}, {pay, cb * kVox * sizeof(float4)}, {weight, cb * kVox * 4},
            {logits, cb * kVox * 4 * static_cast<size_t>(C)}, {vmask, cb * 64}, {meta, cb * 4},
            {grad, cb * kVox * sizeof(float4)}, {active, cb}, {touch, cb * 8}};
        for (const auto& b : blocks)
            if (b.first) dev_release(b.first, b.second, device);
        if (pin) cudaFreeHost(pin);
        if (own_stream && stream) cudaStreamDestroy(stream);
        if (prev >= 0) cudaSetDevice(prev);
    }

    GridView view() {
        GridView v{};
        v.slots = slots;
        v.slot_mask = nslots - 1;
        v.dense = dense.as<uint32_t>();
        v.occ = occ.as<uint32_t>();
        v.pay = pay;
        v.vmask = vmask;
        v.meta = meta;
        v.logits = logits;
        v.nbr = nbr.as<uint32_t>();
        v.bdist = (use_dense && use_jump) ? bdist.as<uint8_t>() : nullptr;
        v.sbdist = (!use_dense && use_sb && use_jump) ? sbdist.as<uint8_t>() : nullptr;
        v.sbinfo = (v.sbdist && n_bricks) ? sb_info.as<uint32_t>() : nullptr;
        v.bricks = v.sbinfo ? bricks.as<uint8_t>() : nullptr;
        for (int a = 0; a < 3; ++a) v.sb_lo[a] = sb_lo[a], v.sb_dim[a] = sb_dim[a];
        v.grad = grad;
        v.active = active;
        v.touch = touch;
        for (int a = 0; a < 3; ++a) {
            v.lo[a] = lo[a];
            v.hi[a] = hi[a];
            v.dim[a] = n() ? hi[a] - lo[a] + 1 : 0;
        }
        v.use_dense = use_dense;
        v.n_blocks = static_cast<uint32_t>(n());
        v.C = C;
        v.h = h;
        v.inv_h = inv_h;
        v.L = L;
        return v;
    }

    // Grow the per-block arrays to hold `need` blocks (contents preserved).
    void ensure_blocks(uint64_t need) {
        if (need <= cap_blocks) return;
        uint64_t nc = std::max<uint64_t>(need, std::min<uint64_t>(capacity, cap_blocks * 2));
        nc = std::max<uint64_t>(nc, 64);
        nc = std::min<uint64_t>(std::max(nc, need), std::max<uint64_t>(capacity, need));
        if (cap_blocks) SVR_CK(cudaStreamSynchronize(stream));  // the old arrays go back to the cache
        auto grow = [&](auto*& ptr, size_t per_block) {
            using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
            size_t got = 0;
            T* np = static_cast<T*>(dev_alloc(nc * per_block * sizeof(T), &got));
            if (ptr) {
                SVR_CK(cudaMemcpyAsync(np, ptr, cap_blocks * per_block * sizeof(T),
                                       cudaMemcpyDeviceToDevice, stream));
                SVR_CK(cudaStreamSynchronize(stream));
                dev_release(ptr, cap_blocks * per_block * sizeof(T), device);
            }
            ptr = np;
        };
        grow(coords4, 4);
        grow(pay, kVox);
        grow(weight, kVox);
        grow(logits, static_cast<size_t>(kVox) * C);
        grow(vmask, 16);
        grow(meta, 1);
        grow(grad, kVox);
        grow(active, 1);
        grow(touch, 8);
        cap_blocks = nc;
    }

    // Zero-initialise blocks [first, first+count) (grid.cpp:69-75).
    void zero_blocks(uint64_t first, uint64_t count) {
        if (!count) return;
        SVR_CK(cudaMemsetAsync(pay + first * kVox, 0, count * kVox * sizeof(float4), stream));
        SVR_CK(cudaMemsetAsync(weight + first * kVox, 0, count * kVox * sizeof(float), stream));
        SVR_CK(cudaMemsetAsync(logits + first * kVox * C, 0, count * kVox * C * sizeof(float), stream));
        SVR_CK(cudaMemsetAsync(vmask + first * 16, 0, count * 16 * sizeof(uint32_t), stream));
        SVR_CK(cudaMemsetAsync(meta + first, 0, count * sizeof(uint32_t), stream));
        SVR_CK(cudaMemsetAsync(grad + first * kVox, 0, count * kVox * sizeof(float4), stream));
        SVR_CK(cudaMemsetAsync(active + first, 0, count, stream));
        SVR_CK(cudaMemsetAsync(touch + first * 8, 0, count * 8, stream));
    }

    // Blocks [first, first+count) got their coords in coords4: count them and extend the
    // AABB (grid.cpp:96-106) with a device min/max reduction (24 bytes read back); the host
    // coordinate mirror is pulled only when asked for (host_coords).
    void grew(uint64_t first, uint64_t count) {
        if (!count) return;
        int32_t* b = static_cast<int32_t*>(pinned(64));
        const int32_t init[6] = {first ? lo[0] : INT32_MAX, first ? lo[1] : INT32_MAX, first ? lo[2] : INT32_MAX,
                                 first ? hi[0] : INT32_MIN, first ? hi[1] : INT32_MIN, first ? hi[2] : INT32_MIN};
        std::memcpy(b, init, sizeof(init));
        bounds_dev.ensure(32);
        SVR_CK(cudaMemcpyAsync(bounds_dev.p, b, 24, cudaMemcpyHostToDevice, stream));
        svr_internal::launch_bounds(coords4 + first * 4, count, bounds_dev.as<int32_t>(), stream);
        SVR_LAUNCHED();
        SVR_CK(cudaMemcpyAsync(b, bounds_dev.p, 24, cudaMemcpyDeviceToHost, stream));
        SVR_CK(cudaStreamSynchronize(stream));
        for (int a = 0; a < 3; ++a) lo[a] = b[a], hi[a] = b[3 + a];
        nblk = first + count;
        dense_dirty = true;
    }

    // Lookup structures, rebuilt lazily after blocks or validity change: the dense AABB
    // index (when the AABB volume is modest) and the per-block neighbour table.
    void ensure_lookup() {
        if (!dense_dirty) return;
        dense_dirty = false;
        use_dense = 0;
        if (n() == 0) return;
        uint64_t cells = 1;
        for (int a = 0; a < 3; ++a) {
            dim[a] = hi[a] - lo[a] + 1;
            cells *= static_cast<uint64_t>(dim[a]);
        }
        const bool fits = cells <= (1ull << 28) && cells <= 64 * n() + (1ull << 22);
        if (lookup_pref == SVR_LOOKUP_DENSE && !fits)
            throw Fail{SVR_ERR_CONFIG, "lookup: block AABB too large for the dense index"};
        if (fits && lookup_pref != SVR_LOOKUP_HASH) {
            dense.ensure(cells * 4);
            occ.ensure(((cells + 31) / 32) * 4);
            SVR_CK(cudaMemsetAsync(dense.p, 0xFF, cells * 4, stream));
            SVR_CK(cudaMemsetAsync(occ.p, 0, ((cells + 31) / 32) * 4, stream));
            svr_internal::launch_dense_build(coords4, meta, static_cast<uint32_t>(n()), lo, dim,
                                             dense.as<uint32_t>(), occ.as<uint32_t>(), stream);
            SVR_LAUNCHED();
            bdist.ensure(cells);
            bdist_tmp.ensure(cells);
            svr_internal::launch_bdist(occ.as<uint32_t>(), dim, bdist.as<uint8_t>(), bdist_tmp.as<uint8_t>(), stream);
            SVR_LAUNCHED();
            use_dense = 1;
        }
        use_sb = 0;
        if (!use_dense) {  // hash mode: superblock (8^3 blocks) occupancy + distance field
            uint64_t sc = 1;
            for (int a = 0; a < 3; ++a) {
                sb_lo[a] = lo[a] >> 3;  // arithmetic shift = floor division
                sb_dim[a] = (hi[a] >> 3) - sb_lo[a] + 1;
                sc *= static_cast<uint64_t>(sb_dim[a]);
            }
            if (sc <= (1ull << 30)) {
                sb_occ.ensure(((sc + 31) / 32) * 4);
                SVR_CK(cudaMemsetAsync(sb_occ.p, 0, ((sc + 31) / 32) * 4, stream));
                svr_internal::launch_superblock_occ(coords4, static_cast<uint32_t>(n()), sb_lo, sb_dim,
                                                    sb_occ.as<uint32_t>(), stream);
                SVR_LAUNCHED();
                sbdist.ensure(sc);
                sbdist_tmp.ensure(sc);
                svr_internal::launch_bdist(sb_occ.as<uint32_t>(), sb_dim, sbdist.as<uint8_t>(),
                                           sbdist_tmp.as<uint8_t>(), stream);
                SVR_LAUNCHED();
                use_sb = 1;
                n_bricks = 0;
                if (sc <= (1ull << 26)) {  // block-distance bricks of the superblocks near blocks
                    // (at most 27 per occupied superblock, so <= 27 n of them)
                    const uint64_t max_b = std::min<uint64_t>(sc, 27ull * n());
                    sb_info.ensure(sc * 4);
                    brick_sb.ensure(max_b * 4);
                    brick_cnt.ensure(4);
                    const uint32_t nb = svr_internal::launch_brick_assign(
                        sb_dim, sbdist.as<uint8_t>(), sb_info.as<uint32_t>(), brick_sb.as<uint32_t>(),
                        brick_cnt.as<uint32_t>(), stream);
                    // 1 KB per brick (two buffers): built only while that stays small next to the
                    // blocks' own 26 KB (a grid of isolated blocks keeps the superblock field alone)
                    if (nb <= 2 * n() + 65536) {
                        bricks.ensure(static_cast<size_t>(nb) * 512);
                        bricks_tmp.ensure(static_cast<size_t>(nb) * 512);
                        svr_internal::launch_brick_fill(coords4, static_cast<uint32_t>(n()), sb_lo, sb_dim,
                                                        sb_info.as<uint32_t>(), brick_sb.as<uint32_t>(), nb,
                                                        bricks.as<uint8_t>(), bricks_tmp.as<uint8_t>(), stream);
                        SVR_LAUNCHED();
                        n_bricks = nb;
                    }
                }
            }
        }
        nbr.ensure(n() * 32);
        svr_internal::launch_nbr_build(view(), coords4, static_cast<uint32_t>(n()), nbr.as<uint32_t>(),
                                       stream);
        SVR_LAUNCHED();
    }

    // Insert `keys` (unique, absent) with indices n().. in order.
    void insert_new(const unsigned long long* d_keys, uint64_t count) {
        if (!count) return;
        const uint64_t first = n();
        ensure_blocks(first + count);
        zero_blocks(first, count);
        svr_internal::launch_hash_insert(slots, nslots - 1, d_keys, count, static_cast<uint32_t>(first),
                                         coords4, stream);
        SVR_LAUNCHED();
        grew(first, count);
    }

    // commit (allocation.cpp:19-43) on a device list of unique base keys.
    void commit(const unsigned long long* d_base, uint64_t nbase, int32_t R, svr_alloc_report& rep) {
        const uint64_t side = 2 * static_cast<uint64_t>(R) + 1;
        const uint64_t ncand = nbase * side * side * side;
        svr_internal::KeySet ks;
        const uint64_t slots_n = next_pow2(std::max<uint64_t>(2 * ncand, 1024));
        scratch_b.ensure(slots_n * 8 + ncand * 8 + 64);
        ks.slots = scratch_b.as<unsigned long long>();
        ks.mask = slots_n - 1;
        ks.list = ks.slots + slots_n;
        ks.cap = ncand;
        unsigned long long* counters = reinterpret_cast<unsigned long long*>(ks.list + ncand);
        SVR_CK(cudaMemsetAsync(counters, 0, 32, stream));
        svr_internal::launch_keyset_clear(ks, stream);
        uint32_t* flags = reinterpret_cast<uint32_t*>(counters + 3);
        svr_internal::launch_dilate(d_base, nbase, R, ks, counters, flags, stream);
        SVR_LAUNCHED();
        unsigned long long hc[4];
        SVR_CK(cudaMemcpyAsync(hc, counters, 32, cudaMemcpyDeviceToHost, stream));
        SVR_CK(cudaStreamSynchronize(stream));
        if (reinterpret_cast<uint32_t*>(&hc[3])[0] & 1u)
            throw Fail{SVR_ERR_CONFIG, "allocate: block coordinate outside +-2^20"};
        const uint64_t nwanted = hc[0];
        rep.blocks_requested = nwanted;
        // filter out the allocated ones
        scratch_c.ensure(nwanted * 8 + 64);
        unsigned long long* fresh = scratch_c.as<unsigned long long>();
        unsigned long long* nfresh_d = counters + 1;
        svr_internal::launch_filter_fresh(view(), ks.list, nwanted, fresh, nfresh_d, stream);
        SVR_LAUNCHED();
        unsigned long long nfresh = 0;
        SVR_CK(cudaMemcpyAsync(&nfresh, nfresh_d, 8, cudaMemcpyDeviceToHost, stream));
        SVR_CK(cudaStreamSynchronize(stream));
        if (nfresh > 1) {
            sort_tmp.ensure(svr_internal::sort_keys_tmp_bytes(nfresh));
            svr_internal::launch_sort_keys(fresh, nfresh, sort_tmp.p, stream);
        }
        SVR_LAUNCHED();
        const uint64_t room = capacity > n() ? capacity - n() : 0;
        const uint64_t take = std::min<uint64_t>(nfresh, room);
        insert_new(fresh, take);
        rep.blocks_added = take;
        rep.unallocated = nfresh - take;
        if (rep.unallocated > 0)
            throw Fail{SVR_ERR_CAPACITY, "allocate: grid capacity exceeded"};
    }

    void ensure_rays(uint64_t nr, uint32_t S) {
        counts.ensure(nr * 4);
        nvalid.ensure(8);  // valid-sample counter of the last forward
        tbuf.ensure(nr * S * 8);
    }
};

namespace svr_host {
// Entry-point guard: the handle's device, and any pending deferred zeroing run in order on the
// handle's stream -- every entry point except render_forward (which fuses it) uses it.
struct GridGuard : DeviceGuard {
    explicit GridGuard(svr_grid* g) : DeviceGuard(g->device) { g->flush_zero(); }
};
}  // namespace svr_host
