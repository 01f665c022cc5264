// Host C++ side of libsvr_b200.so: the svr_grid handle (one device + one stream) and
// every C-ABI entry point of include/svr.h.  It owns all device memory, stages host
// arrays, keeps the host mirror of block coordinates (grid.hpp:219-222) and rebuilds
// the dense AABB lookup index lazily.  There is no CPU compute fallback: every
// numerical result comes from the sm_100a kernels in svr_render.cu / svr_activate.cu /
// svr_grads.cu, and a missing or failing device surfaces as SVR_ERR_CUDA.
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
#include "svr_synth.h"

using namespace svr_dev;

namespace svr_internal {
thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace svr_internal

using svr_internal::set_error;

namespace {

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
int guarded(Fn&& fn) {
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

bool is_device_ptr(const void* p) {
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

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t need) {
        if (need <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        SVR_CK(cudaMalloc(&p, need));
        bytes = need;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
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

uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace

struct svr_grid {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double h = 0, inv_h = 0, L = 0;
    int32_t C = 1;
    uint64_t capacity = 0;
    std::vector<int32_t> coords;  // host mirror, 3 per block
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

    int lookup_pref = SVR_LOOKUP_AUTO;
    bool dense_dirty = true;
    int use_dense = 0;
    int32_t dim[3] = {0, 0, 0};
    DevBuf dense, occ, nbr, bdist, bdist_tmp;
    bool use_jump = true;  // march: exact empty-space jumps over the block-distance field

    // render context
    DevBuf ray_o, ray_d, counts, tbuf, nvalid;
    DevBuf ord_keys, ord_ids, ord_tmp;  // ray ordering (Morton key of the first sample block)
    DevBuf rec;                         // per-sample forward records for the backward
    bool ctx_rec = false;
    uint32_t* ctx_order = nullptr;
    // tuning knobs (svr_grid_set_tuning)
    // bit 1: order the march by origin + direction; bit 0: order forward/backward by the
    // block of each ray's first sample (3 = both)
    int ray_sort = 3;
    int sort_impl = 1;  // 1: CUB radix sort (default, best order), 0: in-house bucketed counting sort
    int fwd_min_blocks = 3;
    bool use_records = true;  // forward leaves 32 B/sample records; backward skips the re-gather
    bool bwd_pipe = true;     // persistent backward streaming records with cp.async.bulk
    bool fwd_pipe = false;    // persistent forward streaming t rows (measured slower: off)
    int fwd_pipe_min_blocks = 3;
    int pipe_min_blocks = 3;
    int num_sms = 148;
    int bwd_min_blocks = 3;
    bool warp_agg = true;  // backward scatter: hand a lane's first cell run to the previous lane
    const double* ctx_o = nullptr;
    const double* ctx_d = nullptr;
    uint64_t ctx_n = 0;
    uint32_t ctx_S = 0;
    double ctx_step = 0, ctx_beta = 0;
    bool ctx_valid = false;

    DevBuf active_list, active_count;  // count: u64 + per-CTA scratch
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
    uint64_t spare_cap = 0;          // cap_blocks the spare pair was sized for
    DevBuf fuse_sum, fuse_cnt;
    DevBuf scratch_a, scratch_b, scratch_c, sort_tmp;
    void* sort_tmp_p = nullptr;
    size_t sort_tmp_bytes = 0;

    uint64_t n() const { return coords.size() / 3; }

    ~svr_grid() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (h2d) {
            cudaStreamSynchronize(h2d);
            cudaStreamSynchronize(d2h);
            for (AsyncSlot& a : aslot)
                for (cudaEvent_t e : {a.in_ev, a.up_ev, a.fwd_ev, a.out_ev, a.free_ev}) cudaEventDestroy(e);
            cudaStreamDestroy(h2d);
            cudaStreamDestroy(d2h);
        }
        for (void* p : {static_cast<void*>(slots), static_cast<void*>(coords4), static_cast<void*>(pay),
                        static_cast<void*>(weight), static_cast<void*>(logits), static_cast<void*>(vmask),
                        static_cast<void*>(meta), static_cast<void*>(grad), static_cast<void*>(active),
                        sort_tmp_p})
            if (p) cudaFree(p);
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
        v.grad = grad;
        v.active = active;
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
        auto grow = [&](auto*& ptr, size_t per_block) {
            using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
            T* np = nullptr;
            SVR_CK(cudaMalloc(&np, nc * per_block * sizeof(T)));
            if (ptr) {
                SVR_CK(cudaMemcpyAsync(np, ptr, cap_blocks * per_block * sizeof(T),
                                       cudaMemcpyDeviceToDevice, stream));
                SVR_CK(cudaStreamSynchronize(stream));
                cudaFree(ptr);
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
    }

    // Host mirror + AABB after blocks [first, first+count) got coords (grid.cpp:96-106).
    void pull_coords(uint64_t first, uint64_t count) {
        std::vector<int32_t> c4(count * 4);
        SVR_CK(cudaMemcpyAsync(c4.data(), coords4 + first * 4, count * 16, cudaMemcpyDeviceToHost, stream));
        SVR_CK(cudaStreamSynchronize(stream));
        for (uint64_t i = 0; i < count; ++i) push_coord(c4[4 * i], c4[4 * i + 1], c4[4 * i + 2]);
    }
    void push_coord(int32_t x, int32_t y, int32_t z) {
        if (coords.empty()) {
            lo[0] = hi[0] = x, lo[1] = hi[1] = y, lo[2] = hi[2] = z;
        } else {
            lo[0] = std::min(lo[0], x), lo[1] = std::min(lo[1], y), lo[2] = std::min(lo[2], z);
            hi[0] = std::max(hi[0], x), hi[1] = std::max(hi[1], y), hi[2] = std::max(hi[2], z);
        }
        coords.push_back(x), coords.push_back(y), coords.push_back(z);
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
        pull_coords(first, count);
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
        svr_internal::launch_sort_keys(fresh, nfresh, &sort_tmp_p, &sort_tmp_bytes, stream);
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
        nvalid.ensure(nr * 4);
        tbuf.ensure(nr * S * 8);
    }
};

namespace {

svr_grid* make_grid(double h, int32_t B, int32_t C, uint64_t capacity, int32_t device) {
    if (!(h > 0.0)) throw Fail{SVR_ERR_CONFIG, "grid: voxel_size must be positive"};  // grid.cpp:83
    if (B < 2) throw Fail{SVR_ERR_CONFIG, "grid: block_res must be >= 2"};
    if (B != kRes) throw Fail{SVR_ERR_CONFIG, "grid: this build specialises block_res = 8"};
    if (C < 1) throw Fail{SVR_ERR_CONFIG, "grid: label_channels must be >= 1"};
    int ndev = 0;
    SVR_CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw Fail{SVR_ERR_CUDA, "grid: no such CUDA device"};
    DeviceGuard dg(device);
    auto g = std::make_unique<svr_grid>();
    g->device = device;
    g->h = h;
    g->inv_h = 1.0 / h;  // grid.cpp:116
    g->L = h * kRes;     // grid.hpp:112
    g->C = C;
    g->capacity = capacity ? capacity : (1ull << 21);  // grid.hpp:107
    SVR_CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->own_stream = true;
    if (const char* e = std::getenv("SVR_RAY_SORT")) g->ray_sort = std::atoi(e);
    SVR_CK(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
    {  // host-array staging uses stream-ordered temporaries: keep freed pool memory mapped
        // across synchronisations instead of returning it to the OS (threshold 0 default)
        cudaMemPool_t pool;
        SVR_CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = ~0ull;
        SVR_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    g->nslots = next_pow2(std::max<uint64_t>(2 * g->capacity, 1024));
    SVR_CK(cudaMalloc(&g->slots, g->nslots * sizeof(HashSlot)));
    SVR_CK(cudaMemsetAsync(g->slots, 0xFF, g->nslots * sizeof(HashSlot), g->stream));
    SVR_CK(cudaStreamSynchronize(g->stream));
    return g.release();
}

}  // namespace

extern "C" {

const char* svr_last_error(void) { return svr_internal::g_err.c_str(); }
int svr_abi_version(void) { return SVR_ABI_VERSION; }

int svr_device_count(int32_t* n) {
    return guarded([&] {
        int c = 0;
        SVR_CK(cudaGetDeviceCount(&c));
        *n = c;
    });
}

int svr_grid_create(double voxel_size, int32_t block_res, int32_t label_channels, uint64_t capacity,
                    int32_t device, svr_grid** out) {
    return guarded([&] { *out = make_grid(voxel_size, block_res, label_channels, capacity, device); });
}

int svr_grid_destroy(svr_grid* g) {
    delete g;
    return SVR_OK;
}

int svr_grid_set_stream(svr_grid* g, void* s) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        SVR_CK(cudaStreamSynchronize(g->stream));
        if (g->own_stream) cudaStreamDestroy(g->stream);
        g->stream = static_cast<cudaStream_t>(s);
        g->own_stream = false;
        if (!s) {
            SVR_CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
            g->own_stream = true;
        }
    });
}

int svr_grid_synchronize(svr_grid* g) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        SVR_CK(cudaStreamSynchronize(g->stream));
        if (g->h2d) {
            SVR_CK(cudaStreamSynchronize(g->h2d));
            SVR_CK(cudaStreamSynchronize(g->d2h));
        }
    });
}

int svr_grid_get_info(svr_grid* g, svr_grid_info* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        g->ensure_lookup();
        svr_grid_info i{};
        i.voxel_size = g->h;
        i.block_res = kRes;
        i.label_channels = g->C;
        i.capacity = g->capacity;
        i.block_count = g->n();
        i.hash_slots = g->nslots;
        for (int a = 0; a < 3; ++a) i.bounds_lo[a] = g->lo[a], i.bounds_hi[a] = g->hi[a];
        i.lookup_mode = g->use_dense ? SVR_LOOKUP_DENSE : SVR_LOOKUP_HASH;
        i.device = g->device;
        const uint64_t per_block = 16 + kVox * (16 + 4 + 4ull * g->C + 16) + 64 + 4 + 1;
        i.device_bytes = g->nslots * sizeof(HashSlot) + g->cap_blocks * per_block + g->dense.bytes +
                         g->occ.bytes + g->tbuf.bytes + g->counts.bytes + g->nvalid.bytes;
        *out = i;
    });
}

int svr_grid_set_tuning(svr_grid* g, const char* key, int64_t value) {
    return guarded([&] {
        const std::string k = key ? key : "";
        if (k == "ray_sort") {
            if (value < 0 || value > 3) throw Fail{SVR_ERR_CONFIG, "tuning: ray_sort is 0..3"};
            g->ray_sort = static_cast<int>(value);
        } else if (k == "fwd_min_blocks") {
            g->fwd_min_blocks = static_cast<int>(value);
        } else if (k == "sort_impl") {
            g->sort_impl = static_cast<int>(value);
        } else if (k == "fwd_pipe") {
            g->fwd_pipe = value != 0;
        } else if (k == "fwd_pipe_min_blocks") {
            g->fwd_pipe_min_blocks = static_cast<int>(value);
        } else if (k == "bwd_pipe") {
            g->bwd_pipe = value != 0;
        } else if (k == "pipe_min_blocks") {
            g->pipe_min_blocks = static_cast<int>(value);
        } else if (k == "records") {
            g->use_records = value != 0;
        } else if (k == "bwd_min_blocks") {
            g->bwd_min_blocks = static_cast<int>(value);
        } else if (k == "march_jump") {
            g->use_jump = value != 0;
        } else if (k == "warp_agg") {
            g->warp_agg = value != 0;
        } else if (k == "host_async") {
            SVR_CK(cudaStreamSynchronize(g->stream));
            if (g->h2d) {
                SVR_CK(cudaStreamSynchronize(g->h2d));
                SVR_CK(cudaStreamSynchronize(g->d2h));
            }
            g->host_async = value != 0;
        } else if (k == "fuse_batch") {
            if (value < 0) throw Fail{SVR_ERR_CONFIG, "tuning: fuse_batch >= 0"};
            g->fuse_batch = static_cast<uint32_t>(value);
        } else {
            throw Fail{SVR_ERR_CONFIG, "tuning: unknown key " + k};
        }
    });
}

int svr_grid_set_lookup(svr_grid* g, int32_t mode) {
    return guarded([&] {
        if (mode < SVR_LOOKUP_AUTO || mode > SVR_LOOKUP_DENSE)
            throw Fail{SVR_ERR_CONFIG, "lookup: unknown mode"};
        DeviceGuard dg(g->device);
        g->lookup_pref = mode;
        g->dense_dirty = true;
        g->ensure_lookup();
    });
}

int svr_grid_allocate_blocks(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        if (n == 0) return;
        std::vector<int32_t> hc(3 * n);
        if (is_device_ptr(coords)) {
            SVR_CK(cudaMemcpy(hc.data(), coords, 12 * n, cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(hc.data(), coords, 12 * n);
        }
        std::vector<uint32_t> existing(n, kInvalid);
        if (g->n()) {
            Stage st(g->stream);
            const int32_t* dc = st.in(hc.data(), 3 * n);
            uint32_t* dout = st.out(existing.data(), n);
            svr_internal::launch_hash_find(g->slots, g->nslots - 1, dc, n, dout, g->stream);
            st.finish();
        }
        std::unordered_map<unsigned long long, uint32_t> fresh_idx;
        std::vector<unsigned long long> fresh;
        std::vector<uint32_t> idx(n, kInvalid);
        int code = SVR_OK;
        std::string msg;
        for (uint64_t i = 0; i < n; ++i) {
            const int32_t x = hc[3 * i], y = hc[3 * i + 1], z = hc[3 * i + 2];
            if (existing[i] != kInvalid) {
                idx[i] = existing[i];
                continue;
            }
            if (!packable(x, y, z)) {
                code = SVR_ERR_CONFIG;
                msg = "grid: block coordinate outside +-2^20";
                break;
            }
            const unsigned long long k = pack_key(x, y, z);
            auto it = fresh_idx.find(k);
            if (it != fresh_idx.end()) {
                idx[i] = it->second;
                continue;
            }
            if (g->n() + fresh.size() >= g->capacity) {  // grid.cpp:91-92
                code = SVR_ERR_CAPACITY;
                msg = "grid: block capacity exceeded";
                break;
            }
            const uint32_t v = static_cast<uint32_t>(g->n() + fresh.size());
            fresh_idx.emplace(k, v);
            fresh.push_back(k);
            idx[i] = v;
        }
        if (!fresh.empty()) {
            g->scratch_a.ensure(fresh.size() * 8);
            SVR_CK(cudaMemcpyAsync(g->scratch_a.p, fresh.data(), fresh.size() * 8,
                                   cudaMemcpyHostToDevice, g->stream));
            g->insert_new(g->scratch_a.as<unsigned long long>(), fresh.size());
        }
        if (idx_out) {
            if (is_device_ptr(idx_out)) {
                SVR_CK(cudaMemcpy(idx_out, idx.data(), 4 * n, cudaMemcpyHostToDevice));
            } else {
                std::memcpy(idx_out, idx.data(), 4 * n);
            }
        }
        if (code != SVR_OK) throw Fail{code, msg};
    });
}

int svr_grid_activate_points(svr_grid* g, const double* xyz, uint64_t n, int32_t dilation,
                             svr_alloc_report* report) {
    svr_alloc_report rep{};
    const int st = guarded([&] {
        if (dilation < 0) throw Fail{SVR_ERR_CONFIG, "allocate: dilation must be >= 0"};
        DeviceGuard dg(g->device);
        Stage stg(g->stream);
        const double* dx = stg.in(xyz, 3 * n);
        svr_internal::KeySet ks;
        const uint64_t slots_n = next_pow2(std::max<uint64_t>(2 * n, 1024));
        g->scratch_a.ensure(slots_n * 8 + n * 8 + 64);
        ks.slots = g->scratch_a.as<unsigned long long>();
        ks.mask = slots_n - 1;
        ks.list = ks.slots + slots_n;
        ks.cap = n;
        unsigned long long* counters = ks.list + n;
        SVR_CK(cudaMemsetAsync(counters, 0, 16, g->stream));
        svr_internal::launch_keyset_clear(ks, g->stream);
        svr_internal::launch_points_to_keys(dx, n, g->L, ks, counters,
                                            reinterpret_cast<uint32_t*>(counters + 1), g->stream);
        stg.finish();
        unsigned long long hc[2];
        SVR_CK(cudaMemcpyAsync(hc, counters, 16, cudaMemcpyDeviceToHost, g->stream));
        SVR_CK(cudaStreamSynchronize(g->stream));
        if (reinterpret_cast<uint32_t*>(&hc[1])[0] & 1u)
            throw Fail{SVR_ERR_CONFIG, "allocate: block coordinate outside +-2^20"};
        rep.pixels_used = n;  // allocation.cpp:85
        g->commit(ks.list, hc[0], dilation, rep);
    });
    if (report) *report = rep;
    return st;
}

int svr_grid_activate_depth(svr_grid* g, const float* depth, const svr_camera* cams,
                            uint32_t n_frames, const double* scales, int32_t sf_rows,
                            int32_t sf_cols, int32_t dilation, svr_alloc_report* report) {
    svr_alloc_report rep{};
    const int st = guarded([&] {
        if (dilation < 0) throw Fail{SVR_ERR_CONFIG, "allocate: dilation must be >= 0"};
        DeviceGuard dg(g->device);
        if (n_frames == 0) {
            g->commit(nullptr, 0, dilation, rep);
            return;
        }
        std::vector<svr_camera> hcams(n_frames);
        if (is_device_ptr(cams)) {
            SVR_CK(cudaMemcpy(hcams.data(), cams, n_frames * sizeof(svr_camera), cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(hcams.data(), cams, n_frames * sizeof(svr_camera));
        }
        const int32_t W = hcams[0].width, H = hcams[0].height;
        for (uint32_t f = 0; f < n_frames; ++f)
            if (hcams[f].width != W || hcams[f].height != H)
                throw Fail{SVR_ERR_CONFIG, "allocate: all frames must share one size"};
        if (scales && (sf_rows < 2 || sf_cols < 2))
            throw Fail{SVR_ERR_CONFIG, "scale field needs at least a 2x2 grid"};
        if (W < 1 || H < 1) throw Fail{SVR_ERR_CONFIG, "allocate: empty frames"};
        const uint64_t npx = static_cast<uint64_t>(W) * H * n_frames;
        Stage stg(g->stream);
        const float* dd = stg.in(depth, npx);
        const svr_camera* dc = stg.in(hcams.data(), n_frames);
        const double* ds = scales ? stg.in(scales, static_cast<uint64_t>(n_frames) * sf_rows * sf_cols)
                                  : nullptr;
        // base-key set: start at 2^22 slots and double on overflow
        uint64_t slots_n = 1ull << 22;
        unsigned long long hc[3];
        svr_internal::KeySet ks;
        for (;;) {
            const uint64_t cap = slots_n / 2;
            g->scratch_a.ensure(slots_n * 8 + cap * 8 + 64);
            ks.slots = g->scratch_a.as<unsigned long long>();
            ks.mask = slots_n - 1;
            ks.list = ks.slots + slots_n;
            ks.cap = cap;
            unsigned long long* counters = ks.list + cap;
            SVR_CK(cudaMemsetAsync(counters, 0, 24, g->stream));
            svr_internal::launch_keyset_clear(ks, g->stream);
            svr_internal::launch_depth_to_keys(dd, dc, n_frames, W, H, ds, sf_rows, sf_cols, g->L, ks,
                                               counters, counters + 1,
                                               reinterpret_cast<uint32_t*>(counters + 2), g->stream);
            SVR_LAUNCHED();
            SVR_CK(cudaMemcpyAsync(hc, counters, 24, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            if (hc[0] <= cap) break;
            slots_n *= 2;
        }
        stg.finish();
        if (reinterpret_cast<uint32_t*>(&hc[2])[0] & 1u)
            throw Fail{SVR_ERR_CONFIG, "allocate: block coordinate outside +-2^20"};
        rep.pixels_used = hc[1];
        // keep the base list alive while commit reuses scratch_a? copy it out first
        DevBuf base;
        base.ensure(std::max<uint64_t>(hc[0], 1) * 8);
        SVR_CK(cudaMemcpyAsync(base.p, ks.list, hc[0] * 8, cudaMemcpyDeviceToDevice, g->stream));
        g->commit(base.as<unsigned long long>(), hc[0], dilation, rep);
        SVR_CK(cudaStreamSynchronize(g->stream));
    });
    if (report) *report = rep;
    return st;
}

int svr_grid_find(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        if (!n) return;
        Stage st(g->stream);
        const int32_t* dc = st.in(coords, 3 * n);
        uint32_t* dout = st.out(idx_out, n);
        svr_internal::launch_hash_find(g->slots, g->nslots - 1, dc, n, dout, g->stream);
        st.finish();
    });
}

int svr_grid_coords(svr_grid* g, int32_t* out) {
    return guarded([&] {
        if (g->coords.empty()) return;
        if (is_device_ptr(out)) {
            DeviceGuard dg(g->device);
            SVR_CK(cudaMemcpy(out, g->coords.data(), g->coords.size() * 4, cudaMemcpyHostToDevice));
        } else {
            std::memcpy(out, g->coords.data(), g->coords.size() * 4);
        }
    });
}

int svr_grid_set_payload(svr_grid* g, uint32_t first, uint32_t n, const float* sdf,
                         const float* weight, const float* rgb, const float* logits) {
    return guarded([&] {
        if (static_cast<uint64_t>(first) + n > g->n())
            throw Fail{SVR_ERR_DATA, "payload: block range out of bounds"};
        if (!n) return;
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        const uint64_t V = static_cast<uint64_t>(n) * kVox;
        const float* a = st.in(sdf, V);
        const float* b = st.in(weight, V);
        const float* c = st.in(rgb, 3 * V);
        const float* d = st.in(logits, V * g->C);
        svr_internal::launch_payload_in(g->pay, g->weight, g->logits, g->vmask, g->meta, first, n,
                                        g->C, a, b, c, d, g->stream);
        st.finish();
        if (weight) g->dense_dirty = true;
    });
}

int svr_grid_get_payload(svr_grid* g, uint32_t first, uint32_t n, float* sdf, float* weight,
                         float* rgb, float* logits) {
    return guarded([&] {
        if (static_cast<uint64_t>(first) + n > g->n())
            throw Fail{SVR_ERR_DATA, "payload: block range out of bounds"};
        if (!n) return;
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        const uint64_t V = static_cast<uint64_t>(n) * kVox;
        float* a = st.out(sdf, V);
        float* b = st.out(weight, V);
        float* c = st.out(rgb, 3 * V);
        float* d = st.out(logits, V * g->C);
        svr_internal::launch_payload_out(g->pay, g->weight, g->logits, first, n, g->C, a, b, c, d,
                                         g->stream);
        st.finish();
    });
}

int svr_query(svr_grid* g, const double* x, uint64_t n, double* sdf, double* grad, double* rgb,
              double* logits, uint8_t* valid) {
    return guarded([&] {
        if (!n) return;
        DeviceGuard dg(g->device);
        g->ensure_lookup();
        Stage st(g->stream);
        const double* dx = st.in(x, 3 * n);
        double* a = st.out(sdf, n);
        double* b = st.out(grad, 3 * n);
        double* c = st.out(rgb, 3 * n);
        double* d = st.out(logits, n * g->C);
        uint8_t* e = st.out(valid, n);
        svr_internal::launch_query(g->view(), dx, n, a, b, c, d, e, g->stream);
        st.finish();
    });
}

int svr_march(svr_grid* g, const double* o, const double* d, uint64_t n, double step,
              uint32_t max_samples, uint32_t* counts, double* t, double* delta) {
    return guarded([&] {
        if (!(step > 0.0)) throw Fail{SVR_ERR_CONFIG, "march: step must be positive"};
        if (!n) return;
        DeviceGuard dg(g->device);
        g->ensure_lookup();
        Stage st(g->stream);
        const double* dO = st.in(o, 3 * n);
        const double* dD = st.in(d, 3 * n);
        uint32_t* dc = st.out(counts, n);
        if (!dc) dc = static_cast<uint32_t*>(st.alloc(4 * n));
        const uint64_t nt = n * static_cast<uint64_t>(max_samples);
        double* dt = st.out(t, nt);
        if (!dt && nt) dt = static_cast<double*>(st.alloc(8 * nt));
        double* dl = st.out(delta, nt);
        svr_internal::launch_march(g->view(), dO, dD, n, nullptr, step, max_samples, dc, dt, dl, g->stream);
        st.finish();
    });
}

namespace {
bool is_pinned_host(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// The forward kernels on g->stream: optional pre-march ray order, K4 march, optional
// post-march order, K5 forward (+ records).  dO / dD / outputs are device pointers.
void forward_kernels(svr_grid* g, const double* dO, const double* dD, uint64_t n, double step,
                     uint32_t max_samples, double beta, float* a, float* b, float* c, float* e) {
    g->ensure_rays(std::max<uint64_t>(n, 1), max_samples);
    const GridView v = g->view();
    g->ctx_order = nullptr;
    const bool sort = g->ray_sort != 0 && n > 1;
    const bool cub_sort = sort && g->sort_impl == 1;
    if (cub_sort) {
        g->ord_keys.ensure(8 * n);
        g->ord_ids.ensure(8 * n);
        g->ord_tmp.ensure(std::max<size_t>(svr_internal::ray_order_tmp_bytes(n), 16));
    } else if (sort) {
        g->ord_ids.ensure(4 * svr_internal::ray_order_scratch_words(n));
    }
    uint32_t* k = g->ord_keys.as<uint32_t>();
    uint32_t* id = g->ord_ids.as<uint32_t>();
    auto order_rays = [&](bool post_march) {
        const uint32_t* cnt = post_march ? g->counts.as<uint32_t>() : nullptr;
        const double* tt = post_march ? g->tbuf.as<double>() : nullptr;
        if (cub_sort) {
            svr_internal::launch_ray_order(v, dO, dD, n, cnt, tt, max_samples, k, id, k + n, id + n,
                                           g->ord_tmp.p, g->ord_tmp.bytes, &g->ctx_order, g->stream);
        } else {
            svr_internal::launch_ray_bucket_order(v, dO, dD, n, cnt, tt, max_samples, id, g->stream);
            g->ctx_order = id;
        }
    };
    if (sort && (g->ray_sort & 2)) order_rays(false);  // pre-march: origin + direction
    svr_internal::launch_march(v, dO, dD, n, g->ctx_order, step, max_samples, g->counts.as<uint32_t>(),
                               g->tbuf.as<double>(), nullptr, g->stream);
    if (sort && (g->ray_sort & 1)) order_rays(true);   // post-march: first-sample block
    g->ctx_rec = g->use_records;
    if (g->ctx_rec) g->rec.ensure(n * max_samples * 32);
    float4* recp = g->ctx_rec ? g->rec.as<float4>() : nullptr;
    const bool piped =
        g->fwd_pipe && svr_internal::launch_render_forward_pipe(v, dO, dD, n, g->ctx_order, g->counts.as<uint32_t>(),
                                                                g->tbuf.as<double>(), max_samples, step, beta, a, b,
                                                                c, e, recp, g->stream, g->fwd_pipe_min_blocks,
                                                                g->num_sms);
    if (!piped)
        svr_internal::launch_render_forward(v, dO, dD, n, g->ctx_order, g->counts.as<uint32_t>(),
                                            g->tbuf.as<double>(), max_samples, step, beta, a, b, c, e, nullptr,
                                            recp, g->stream, g->fwd_min_blocks);
}

void backward_kernels(svr_grid* g, const float* a, const float* b, const float* c) {
    const uint64_t n = g->ctx_n;
    const bool piped =
        g->bwd_pipe && g->ctx_rec &&
        svr_internal::launch_render_backward_pipe(g->view(), g->ctx_o, g->ctx_d, n, g->ctx_order,
                                                  g->counts.as<uint32_t>(), g->tbuf.as<double>(), g->ctx_S,
                                                  g->ctx_step, g->ctx_beta, a, b, c, g->rec.as<float4>(),
                                                  g->stream, g->pipe_min_blocks, g->num_sms, g->warp_agg);
    if (!piped)
        svr_internal::launch_render_backward(g->view(), g->ctx_o, g->ctx_d, n, g->ctx_order,
                                             g->counts.as<uint32_t>(), g->tbuf.as<double>(), g->ctx_S,
                                             g->ctx_step, g->ctx_beta, a, b, c,
                                             g->ctx_rec ? g->rec.as<float4>() : nullptr, g->stream,
                                             g->bwd_min_blocks, g->warp_agg);
}
}  // namespace

int svr_render_forward(svr_grid* g, const double* o, const double* d, uint64_t n, double step,
                       uint32_t max_samples, double beta, float* rgb, float* depth, float* normal,
                       float* wsum, uint32_t* n_samples) {
    return guarded([&] {
        if (!(beta > 0.0)) throw Fail{SVR_ERR_CONFIG, "render: beta must be positive"};
        if (!(step > 0.0)) throw Fail{SVR_ERR_CONFIG, "render: step must be positive"};
        if (max_samples < 1 || max_samples > 2048)
            throw Fail{SVR_ERR_CONFIG, "render: max_samples must be in [1, 2048]"};
        DeviceGuard dg(g->device);
        g->ensure_lookup();
        g->ctx_valid = false;
        g->ctx_aslot = -1;
        // host_async: every host array pinned -> transfers on the copy streams, no host sync
        const void* arrs[7] = {o, d, rgb, depth, normal, wsum, n_samples};
        bool async = g->host_async && n > 0, any_host = false;
        for (const void* p : arrs) {
            if (!p || is_device_ptr(p)) continue;
            any_host = true;
            async = async && is_pinned_host(p);
        }
        if (async && any_host) {
            g->ensure_async();
            const int si = g->aslot_next;
            g->aslot_next ^= 1;
            svr_grid::AsyncSlot& sl = g->aslot[si];
            sl.o.ensure(24 * n);
            sl.d.ensure(24 * n);
            sl.out.ensure(36 * n);
            if (sl.used) SVR_CK(cudaStreamWaitEvent(g->h2d, sl.free_ev, 0));  // slot's last backward done
            const double* dO = o;
            const double* dD = d;
            if (!is_device_ptr(o)) {
                SVR_CK(cudaMemcpyAsync(sl.o.p, o, 24 * n, cudaMemcpyHostToDevice, g->h2d));
                dO = sl.o.as<double>();
            }
            if (!is_device_ptr(d)) {
                SVR_CK(cudaMemcpyAsync(sl.d.p, d, 24 * n, cudaMemcpyHostToDevice, g->h2d));
                dD = sl.d.as<double>();
            }
            SVR_CK(cudaEventRecord(sl.in_ev, g->h2d));
            SVR_CK(cudaStreamWaitEvent(g->stream, sl.in_ev, 0));
            if (sl.used) SVR_CK(cudaStreamWaitEvent(g->stream, sl.out_ev, 0));  // slot outputs drained
            float* so = sl.out.as<float>();
            struct O {
                float* host;
                float* dev;
                size_t bytes;
            } outs[4] = {{rgb, so, 12 * n}, {depth, so + 3 * n, 4 * n}, {normal, so + 4 * n, 12 * n},
                         {wsum, so + 7 * n, 4 * n}};
            float* dev_out[4];
            for (int i = 0; i < 4; ++i)
                dev_out[i] = (!outs[i].host || is_device_ptr(outs[i].host)) ? outs[i].host : outs[i].dev;
            forward_kernels(g, dO, dD, n, step, max_samples, beta, dev_out[0], dev_out[1], dev_out[2], dev_out[3]);
            uint32_t* ns_dev = reinterpret_cast<uint32_t*>(so + 8 * n);
            if (n_samples)
                SVR_CK(cudaMemcpyAsync(is_device_ptr(n_samples) ? n_samples : ns_dev, g->counts.p, 4 * n,
                                       cudaMemcpyDeviceToDevice, g->stream));
            SVR_LAUNCHED();
            SVR_CK(cudaEventRecord(sl.fwd_ev, g->stream));
            SVR_CK(cudaStreamWaitEvent(g->d2h, sl.fwd_ev, 0));
            for (int i = 0; i < 4; ++i)
                if (dev_out[i] == outs[i].dev)
                    SVR_CK(cudaMemcpyAsync(outs[i].host, outs[i].dev, outs[i].bytes, cudaMemcpyDeviceToHost, g->d2h));
            if (n_samples && !is_device_ptr(n_samples))
                SVR_CK(cudaMemcpyAsync(n_samples, ns_dev, 4 * n, cudaMemcpyDeviceToHost, g->d2h));
            SVR_CK(cudaEventRecord(sl.out_ev, g->d2h));
            // until this slot's backward runs, free_ev must not report it free
            SVR_CK(cudaEventRecord(sl.free_ev, g->stream));
            sl.used = true;
            g->ctx_aslot = si;
            g->ctx_o = dO;
            g->ctx_d = dD;
        } else {
            Stage st(g->stream);
            // retain rays for the backward pass: device arrays by pointer, host arrays copied
            const double* dO = o;
            const double* dD = d;
            if (n && !is_device_ptr(o)) {
                g->ray_o.ensure(24 * n);
                SVR_CK(cudaMemcpyAsync(g->ray_o.p, o, 24 * n, cudaMemcpyHostToDevice, g->stream));
                dO = g->ray_o.as<double>();
                st.host_involved = true;
            }
            if (n && !is_device_ptr(d)) {
                g->ray_d.ensure(24 * n);
                SVR_CK(cudaMemcpyAsync(g->ray_d.p, d, 24 * n, cudaMemcpyHostToDevice, g->stream));
                dD = g->ray_d.as<double>();
                st.host_involved = true;
            }
            g->ensure_rays(std::max<uint64_t>(n, 1), max_samples);
            float* a = st.out(rgb, 3 * n);
            float* b = st.out(depth, n);
            float* c = st.out(normal, 3 * n);
            float* e = st.out(wsum, n);
            if (n) {
                forward_kernels(g, dO, dD, n, step, max_samples, beta, a, b, c, e);
                if (n_samples) {
                    uint32_t* ns = st.out(n_samples, n);
                    SVR_CK(cudaMemcpyAsync(ns, g->counts.p, 4 * n, cudaMemcpyDeviceToDevice, g->stream));
                }
            }
            st.finish();
            g->ctx_o = dO;
            g->ctx_d = dD;
        }
        g->ctx_n = n;
        g->ctx_S = max_samples;
        g->ctx_step = step;
        g->ctx_beta = beta;
        g->ctx_valid = true;
    });
}

int svr_render_backward(svr_grid* g, const float* d_rgb, const float* d_depth, const float* d_normal) {
    return guarded([&] {
        if (!g->ctx_valid) throw Fail{SVR_ERR_DATA, "render_backward: no retained forward context"};
        if (!d_rgb || !d_depth || !d_normal)
            throw Fail{SVR_ERR_DATA, "render_backward: upstream gradients required"};
        DeviceGuard dg(g->device);
        const uint64_t n = g->ctx_n;
        if (!n) return;
        if (g->ctx_aslot >= 0) {  // pipelined host I/O (the forward ran through a slot)
            svr_grid::AsyncSlot& sl = g->aslot[g->ctx_aslot];
            const float* up[3] = {d_rgb, d_depth, d_normal};
            const size_t cnt[3] = {3 * n, n, 3 * n};
            bool ok = true;
            for (const float* p : up) ok = ok && (is_device_ptr(p) || is_pinned_host(p));
            if (ok) {
                sl.up.ensure(28 * n);
                const float* dev[3];
                size_t off = 0;
                for (int i = 0; i < 3; ++i) {
                    if (is_device_ptr(up[i])) {
                        dev[i] = up[i];
                    } else {
                        float* dst = sl.up.as<float>() + off;
                        SVR_CK(cudaMemcpyAsync(dst, up[i], 4 * cnt[i], cudaMemcpyHostToDevice, g->h2d));
                        dev[i] = dst;
                    }
                    off += cnt[i];
                }
                SVR_CK(cudaEventRecord(sl.up_ev, g->h2d));
                SVR_CK(cudaStreamWaitEvent(g->stream, sl.up_ev, 0));
                backward_kernels(g, dev[0], dev[1], dev[2]);
                SVR_LAUNCHED();
                SVR_CK(cudaEventRecord(sl.free_ev, g->stream));
                return;
            }
        }
        Stage st(g->stream);
        const float* a = st.in(d_rgb, 3 * n);
        const float* b = st.in(d_depth, n);
        const float* c = st.in(d_normal, 3 * n);
        backward_kernels(g, a, b, c);
        st.finish();
        if (g->ctx_aslot >= 0) SVR_CK(cudaEventRecord(g->aslot[g->ctx_aslot].free_ev, g->stream));
    });
}

int svr_render_get_stats(svr_grid* g, svr_render_stats* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        svr_render_stats s{};
        s.rays = g->ctx_valid ? g->ctx_n : 0;
        if (g->ctx_valid && g->ctx_n) {
            // re-run the forward's validity count on the retained context (not on the hot path)
            std::vector<uint32_t> cnt(g->ctx_n);
            SVR_CK(cudaMemcpyAsync(cnt.data(), g->counts.p, 4 * g->ctx_n, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            for (uint32_t c : cnt) s.samples += c;
            DevBuf vc;
            vc.ensure(8);
            SVR_CK(cudaMemsetAsync(vc.p, 0, 8, g->stream));
            svr_internal::launch_render_forward(g->view(), g->ctx_o, g->ctx_d, g->ctx_n, g->ctx_order,
                                                g->counts.as<uint32_t>(), g->tbuf.as<double>(),
                                                g->ctx_S, g->ctx_step, g->ctx_beta, nullptr, nullptr,
                                                nullptr, nullptr, vc.as<unsigned long long>(), nullptr,
                                                g->stream, g->fwd_min_blocks);
            SVR_LAUNCHED();
            unsigned long long v = 0;
            SVR_CK(cudaMemcpyAsync(&v, vc.p, 8, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            s.valid_samples = v;
        }
        *out = s;
    });
}

int svr_grad_zero(svr_grid* g) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        if (!g->n()) return;
        SVR_CK(cudaMemsetAsync(g->grad, 0, g->n() * kVox * sizeof(float4), g->stream));
        SVR_CK(cudaMemsetAsync(g->active, 0, g->n(), g->stream));
    });
}

int svr_grad_get(svr_grid* g, float* g_sdf, float* g_rgb) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        if (!g->n()) return;
        Stage st(g->stream);
        const uint64_t V = g->n() * kVox;
        float* a = st.out(g_sdf, V);
        float* b = st.out(g_rgb, 3 * V);
        svr_internal::launch_grad_out(g->grad, static_cast<uint32_t>(g->n()), a, b, g->stream);
        st.finish();
    });
}

int svr_active_blocks(svr_grid* g, uint8_t* mask, uint32_t* list, uint64_t* count) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        Stage st(g->stream);
        if (mask && nb) {
            uint8_t* m = st.out(mask, nb);
            SVR_CK(cudaMemcpyAsync(m, g->active, nb, cudaMemcpyDeviceToDevice, g->stream));
        }
        if (list || count) {
            g->active_list.ensure(std::max<uint32_t>(nb, 1) * 4);
            g->active_count.ensure(8 + 4 * ((nb + 1023) / 1024 + 2));
            auto* dcount = g->active_count.as<unsigned long long>();
            svr_internal::launch_active_list(g->active, nb, g->active_list.as<uint32_t>(), dcount, g->stream);
            SVR_LAUNCHED();
            unsigned long long c = 0;
            SVR_CK(cudaMemcpyAsync(&c, dcount, 8, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            if (count) {
                if (is_device_ptr(count)) {
                    SVR_CK(cudaMemcpyAsync(count, dcount, 8, cudaMemcpyDeviceToDevice, g->stream));
                } else {
                    *count = c;
                }
            }
            if (list && c) {
                uint32_t* l = st.out(list, c);
                SVR_CK(cudaMemcpyAsync(l, g->active_list.p, 4 * c, cudaMemcpyDeviceToDevice, g->stream));
            }
        }
        st.finish();
    });
}

int svr_active_set_mask(svr_grid* g, const uint8_t* mask) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        Stage st(g->stream);
        const uint8_t* m = st.in(mask, nb);
        svr_internal::launch_set_active(g->active, m, nb, g->stream);
        st.finish();
    });
}

int svr_grad_pack(svr_grid* g, const uint32_t* blocks, uint64_t n, float* out) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        const uint32_t* b = st.in(blocks, n);
        float* o = st.out(out, n * kVox * 4);
        svr_internal::launch_grad_pack(g->grad, b, n, reinterpret_cast<float4*>(o), g->stream);
        st.finish();
    });
}

int svr_grad_unpack(svr_grid* g, const uint32_t* blocks, uint64_t n, const float* in) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        const uint32_t* b = st.in(blocks, n);
        const float* i = st.in(in, n * kVox * 4);
        svr_internal::launch_grad_unpack(g->grad, b, n, reinterpret_cast<const float4*>(i), g->stream);
        st.finish();
    });
}

int svr_grad_zero_active(svr_grid* g) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        if (!nb) return;
        g->active_list.ensure(nb * 4);
        g->active_count.ensure(8 + 4 * ((nb + 1023) / 1024 + 2));
        auto* dcount = g->active_count.as<unsigned long long>();
        svr_internal::launch_active_list(g->active, nb, g->active_list.as<uint32_t>(), dcount, g->stream);
        svr_internal::launch_grad_zero_active(g->grad, g->active, g->active_list.as<uint32_t>(), dcount,
                                              nb, g->stream);
        SVR_LAUNCHED();
    });
}

int svr_sample_uniform(svr_grid* g, uint64_t n, uint64_t seed, double* out) {
    return guarded([&] {
        if (g->n() == 0) throw Fail{SVR_ERR_DATA, "sample_uniform: empty grid"};  // grid.cpp:358
        if (!n) return;
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        double* o = st.out(out, 3 * n);
        svr_internal::launch_sample_uniform(g->coords4, static_cast<uint32_t>(g->n()), g->L, n, seed, o,
                                            g->stream);
        st.finish();
    });
}

int svr_eikonal(svr_grid* g, const double* x, uint64_t n, double scale, double* loss, uint64_t* n_valid) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        double sums[2] = {0.0, 0.0};
        if (n && g->n()) {
            g->ensure_lookup();
            Stage st(g->stream);
            const double* dx = st.in(x, 3 * n);
            double* dsum = static_cast<double*>(st.alloc(16));
            SVR_CK(cudaMemsetAsync(dsum, 0, 16, g->stream));
            const GridView v = g->view();
            svr_internal::launch_eikonal_stats(v, dx, n, dsum, g->stream);
            SVR_LAUNCHED();
            SVR_CK(cudaMemcpyAsync(sums, dsum, 16, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            if (sums[1] > 0.0 && scale != 0.0)
                svr_internal::launch_eikonal_scatter(v, dx, n, 2.0 * scale / sums[1], g->stream);
            st.finish();
        }
        if (loss) *loss = sums[1] > 0.0 ? sums[0] / sums[1] : 0.0;
        if (n_valid) *n_valid = static_cast<uint64_t>(sums[1]);
    });
}

int svr_rmsprop_step(svr_grid* g, float lr, float alpha, float eps) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        if (!nb) return;
        if (g->rms_blocks < nb) {  // grow the state, new rows start at zero
            DevBuf fresh;
            fresh.ensure(static_cast<size_t>(nb) * kVox * sizeof(float4));
            SVR_CK(cudaMemsetAsync(fresh.p, 0, static_cast<size_t>(nb) * kVox * sizeof(float4), g->stream));
            if (g->rms_blocks)
                SVR_CK(cudaMemcpyAsync(fresh.p, g->rms.p, g->rms_blocks * kVox * sizeof(float4),
                                       cudaMemcpyDeviceToDevice, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            std::swap(g->rms.p, fresh.p);
            std::swap(g->rms.bytes, fresh.bytes);
            g->rms_blocks = nb;
        }
        g->active_list.ensure(nb * 4);
        g->active_count.ensure(8 + 4 * ((nb + 1023) / 1024 + 2));
        auto* dcount = g->active_count.as<unsigned long long>();
        svr_internal::launch_active_list(g->active, nb, g->active_list.as<uint32_t>(), dcount, g->stream);
        svr_internal::launch_rmsprop(g->pay, g->grad, g->rms.as<float4>(), g->active,
                                     g->active_list.as<uint32_t>(), dcount, nb, lr, alpha, eps, g->stream);
        SVR_LAUNCHED();
    });
}

// ---------------------------------------------------------------------------
// Fusion + de-noising, kernels K12/K13 in svr_fusion.cu.
// ---------------------------------------------------------------------------
namespace {
// Grow the session's sums to the current block count (new rows zero).  The buffers stay
// cached in the handle between sessions (re-zeroed by svr_fuse_begin).
void fuse_grow(svr_grid* g) {
    const uint64_t nb = g->n();
    if (g->fuse_blocks >= nb) return;
    const size_t per_sum = static_cast<size_t>(4 + g->C) * kVox * sizeof(long long);
    const size_t per_cnt = kVox * sizeof(uint32_t);
    if (g->fuse_sum.bytes < nb * per_sum || g->fuse_cnt.bytes < nb * per_cnt) {
        DevBuf s2, c2;
        const uint64_t rows = std::max<uint64_t>(nb, g->cap_blocks);
        s2.ensure(rows * per_sum);
        c2.ensure(rows * per_cnt);
        if (g->fuse_blocks) {
            SVR_CK(cudaMemcpyAsync(s2.p, g->fuse_sum.p, g->fuse_blocks * per_sum, cudaMemcpyDeviceToDevice, g->stream));
            SVR_CK(cudaMemcpyAsync(c2.p, g->fuse_cnt.p, g->fuse_blocks * per_cnt, cudaMemcpyDeviceToDevice, g->stream));
        }
        SVR_CK(cudaStreamSynchronize(g->stream));
        std::swap(g->fuse_sum.p, s2.p);
        std::swap(g->fuse_sum.bytes, s2.bytes);
        std::swap(g->fuse_cnt.p, c2.p);
        std::swap(g->fuse_cnt.bytes, c2.bytes);
    }
    const uint64_t f = g->fuse_blocks;
    SVR_CK(cudaMemsetAsync(static_cast<char*>(g->fuse_sum.p) + f * per_sum, 0, (nb - f) * per_sum, g->stream));
    SVR_CK(cudaMemsetAsync(static_cast<char*>(g->fuse_cnt.p) + f * per_cnt, 0, (nb - f) * per_cnt, g->stream));
    g->fuse_blocks = nb;
}
}  // namespace

int svr_fuse_begin(svr_grid* g, int32_t flags) {
    return guarded([&] {
        if (flags & ~(SVR_FUSE_COLOR | SVR_FUSE_SEMANTIC)) throw Fail{SVR_ERR_CONFIG, "fuse_begin: unknown flags"};
        DeviceGuard dg(g->device);
        g->fuse_flags = -1;
        g->fuse_blocks = 0;
        fuse_grow(g);
        g->fuse_flags = flags;
    });
}

int svr_fuse_frames(svr_grid* g, const float* depth, const float* rgb, const float* semantic,
                    const svr_camera* cams, uint32_t n_frames, const double* scales, int32_t sf_rows,
                    int32_t sf_cols, double mu, svr_fuse_report* report) {
    svr_fuse_report rep{};
    const int st = guarded([&] {
        if (g->fuse_flags < 0) throw Fail{SVR_ERR_CONFIG, "fuse: no session (svr_fuse_begin)"};
        if (!(mu > 0.0) || !(mu < 524288.0)) throw Fail{SVR_ERR_CONFIG, "fuse: mu must be in (0, 2^19)"};
        if (((g->fuse_flags & SVR_FUSE_COLOR) != 0) != (rgb != nullptr) ||
            ((g->fuse_flags & SVR_FUSE_SEMANTIC) != 0) != (semantic != nullptr))
            throw Fail{SVR_ERR_CONFIG, "fuse: channels differ from the session's flags"};
        if (scales && (sf_rows < 2 || sf_cols < 2))
            throw Fail{SVR_ERR_CONFIG, "scale field needs at least a 2x2 grid"};
        if (n_frames == 0) return;
        if (!depth || !cams) throw Fail{SVR_ERR_DATA, "fuse: depth and cameras are required"};
        std::vector<svr_camera> hc(n_frames);
        if (is_device_ptr(cams))
            SVR_CK(cudaMemcpy(hc.data(), cams, n_frames * sizeof(svr_camera), cudaMemcpyDeviceToHost));
        else
            std::memcpy(hc.data(), cams, n_frames * sizeof(svr_camera));
        const int32_t W = hc[0].width, H = hc[0].height;
        for (const svr_camera& c : hc)
            if (c.width != W || c.height != H) throw Fail{SVR_ERR_CONFIG, "fuse: all frames must share one size"};
        if (W < 1 || H < 1) throw Fail{SVR_ERR_CONFIG, "fuse: empty image"};
        if (scales && (W < 2 || H < 2)) throw Fail{SVR_ERR_CONFIG, "scale field image size too small"};
        DeviceGuard dg(g->device);
        fuse_grow(g);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        const size_t npx = static_cast<size_t>(W) * H;
        const size_t sf = scales ? static_cast<size_t>(sf_rows) * sf_cols : 0;
        // frames per launch: every launch streams the running sums once (~(8 (4 + C) + 4) B per
        // voxel each way), so a launch takes as many frames as possible -- all of them when the
        // images are device-resident, else what 1 GB of staging holds.
        const size_t per_frame = npx * (4 + (rgb ? 12 : 0) + (semantic ? 4 * g->C : 0)) + sf * 8;
        const bool resident = is_device_ptr(depth) && (!rgb || is_device_ptr(rgb)) &&
                              (!semantic || is_device_ptr(semantic)) && (!scales || is_device_ptr(scales));
        const uint32_t batch = g->fuse_batch ? std::min(g->fuse_batch, n_frames)
                               : resident ? n_frames
                                        : static_cast<uint32_t>(std::max<size_t>(
                                              1, std::min<size_t>(n_frames, (1ull << 30) / per_frame)));
        Stage st(g->stream);
        auto* counters = static_cast<unsigned long long*>(st.alloc(16));
        SVR_CK(cudaMemsetAsync(counters, 0, 16, g->stream));
        const svr_camera* dcams = st.in(cams, n_frames);
        for (uint32_t f0 = 0; f0 < n_frames; f0 += batch) {
            const uint32_t nf = std::min(batch, n_frames - f0);
            Stage sb(g->stream);
            const float* dd = sb.in(depth + f0 * npx, nf * npx);
            const float* dr = sb.in(rgb ? rgb + 3 * f0 * npx : nullptr, 3 * nf * npx);
            const float* ds = sb.in(semantic ? semantic + static_cast<size_t>(g->C) * f0 * npx : nullptr,
                                    static_cast<size_t>(g->C) * nf * npx);
            const double* dsc = sb.in(scales ? scales + f0 * sf : nullptr, nf * sf);
            svr_internal::launch_fuse(g->coords4, nb, dcams + f0, nf, W, H, g->C, dd, dr, ds, dsc, sf_rows,
                                      sf_cols, g->h, mu, g->fuse_sum.as<long long>(), g->fuse_cnt.as<uint32_t>(),
                                      counters, g->stream);
            sb.finish();
        }
        unsigned long long hcnt[2] = {0, 0};
        SVR_CK(cudaMemcpyAsync(hcnt, counters, 16, cudaMemcpyDeviceToHost, g->stream));
        st.finish();
        SVR_CK(cudaStreamSynchronize(g->stream));
        rep.frames = n_frames;
        rep.in_view = hcnt[0];
        rep.rejected = hcnt[1];
        rep.integrated = hcnt[0] - hcnt[1];
    });
    if (report) *report = rep;
    return st;
}

int svr_fuse_finalize(svr_grid* g) {
    return guarded([&] {
        if (g->fuse_flags < 0) throw Fail{SVR_ERR_CONFIG, "fuse: no session (svr_fuse_begin)"};
        DeviceGuard dg(g->device);
        fuse_grow(g);
        svr_internal::launch_fuse_finalize(g->fuse_sum.as<long long>(), g->fuse_cnt.as<uint32_t>(),
                                           static_cast<uint32_t>(g->n()), g->C, g->fuse_flags, g->pay, g->weight,
                                           g->logits, g->vmask, g->meta, g->stream);
        SVR_LAUNCHED();
        SVR_CK(cudaStreamSynchronize(g->stream));
        g->dense_dirty = true;
        g->fuse_flags = -1;
        g->fuse_blocks = 0;
    });
}

int svr_denoise(svr_grid* g, double sigma_vox, int32_t radius) {
    return guarded([&] {
        if (!(sigma_vox > 0.0)) throw Fail{SVR_ERR_CONFIG, "denoise: sigma must be positive"};
        if (radius < 0 || radius > 4) throw Fail{SVR_ERR_CONFIG, "denoise: radius must be in [0, 4]"};
        DeviceGuard dg(g->device);
        const uint64_t nb = g->n();
        if (!nb) return;
        g->ensure_lookup();
        double gw[9];
        for (int d = -radius; d <= radius; ++d)
            gw[d + radius] = std::exp(-static_cast<double>(d * d) / (2.0 * sigma_vox * sigma_vox));
        // output planes: the spare pair left by the previous denoise (same row capacity)
        if (g->spare_cap != g->cap_blocks) {
            g->pay_spare.bytes = 0;
            g->logits_spare.bytes = 0;
        }
        g->pay_spare.ensure(g->cap_blocks * kVox * sizeof(float4));
        g->logits_spare.ensure(g->cap_blocks * kVox * g->C * sizeof(float));
        g->spare_cap = g->cap_blocks;
        svr_internal::launch_denoise(g->view(), g->coords4, g->pay_spare.as<float4>(), g->logits_spare.as<float>(),
                                     radius, gw, g->stream);
        SVR_LAUNCHED();
        // the new planes become the payload; the old ones the next call's spare pair
        float4* old_pay = g->pay;
        float* old_lg = g->logits;
        g->pay = g->pay_spare.as<float4>();
        g->logits = g->logits_spare.as<float>();
        g->pay_spare.p = old_pay;
        g->logits_spare.p = old_lg;
    });
}

// ---------------------------------------------------------------------------
// Peer-memory gradient all-reduce (K8p in svr_grads.cu).
// ---------------------------------------------------------------------------
int svr_grad_ipc_handle(svr_grid* g, void* handle_out, uint64_t* plane_bytes) {
    return guarded([&] {
        if (!handle_out) throw Fail{SVR_ERR_DATA, "grad_ipc_handle: output required"};
        DeviceGuard dg(g->device);
        if (!g->grad) throw Fail{SVR_ERR_DATA, "grad_ipc_handle: the grid has no blocks yet"};
        cudaIpcMemHandle_t h;
        SVR_CK(cudaIpcGetMemHandle(&h, g->grad));
        static_assert(sizeof(h) == SVR_IPC_HANDLE_BYTES, "IPC handle size");
        std::memcpy(handle_out, &h, sizeof(h));
        if (plane_bytes) *plane_bytes = g->cap_blocks * kVox * sizeof(float4);
    });
}

int svr_grad_plane(svr_grid* g, void** ptr_out, uint64_t* plane_bytes) {
    return guarded([&] {
        if (ptr_out) *ptr_out = g->grad;
        if (plane_bytes) *plane_bytes = g->cap_blocks * kVox * sizeof(float4);
    });
}

int svr_ipc_open(const void* handle, int32_t device, void** ptr_out) {
    return guarded([&] {
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        SVR_CK(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int svr_ipc_close(void* ptr) {
    return guarded([&] { SVR_CK(cudaIpcCloseMemHandle(ptr)); });
}

int svr_grad_peer_allreduce(svr_grid* g, void* const* peer_planes, uint32_t world, uint32_t rank,
                            const uint32_t* rows, uint64_t n_rows) {
    return guarded([&] {
        if (world < 1 || world > 8 || rank >= world) throw Fail{SVR_ERR_CONFIG, "peer_allreduce: 1 <= world <= 8"};
        DeviceGuard dg(g->device);
        float4* planes[8];
        for (uint32_t q = 0; q < world; ++q) {
            planes[q] = static_cast<float4*>(peer_planes ? peer_planes[q] : nullptr);
            if (q == rank && !planes[q]) planes[q] = g->grad;
            if (!planes[q]) throw Fail{SVR_ERR_DATA, "peer_allreduce: missing peer plane"};
        }
        Stage st(g->stream);
        const uint32_t* r = st.in(rows, n_rows);
        svr_internal::launch_peer_allreduce(planes, world, rank, r, n_rows, g->stream);
        st.finish();
    });
}

// ---------------------------------------------------------------------------
// Refinement losses, K15 in svr_losses.cu.
// ---------------------------------------------------------------------------
int svr_render_losses(svr_grid* g, uint64_t n, const float* rgb, const float* depth, const float* normal,
                      const float* wsum, const float* tgt_rgb, const float* prior_depth,
                      const float* prior_normal, const uint32_t* cam_idx, const svr_camera* cams,
                      uint32_t n_cams, double lambda_d, double lambda_n, float* d_rgb, float* d_depth,
                      float* d_normal, svr_loss_stats* stats) {
    return guarded([&] {
        if (!rgb || !depth || !normal || !wsum || !tgt_rgb || !d_rgb || !d_depth || !d_normal)
            throw Fail{SVR_ERR_DATA, "render_losses: rendered outputs, colour targets and gradients required"};
        if (prior_normal && (!cam_idx || !cams || !n_cams))
            throw Fail{SVR_ERR_DATA, "render_losses: the normal term needs cameras and per-ray camera indices"};
        if (!(lambda_d >= 0.0) || !(lambda_n >= 0.0)) throw Fail{SVR_ERR_CONFIG, "render_losses: negative weight"};
        DeviceGuard dg(g->device);
        g->loss_acc.ensure(16 * sizeof(double));
        Stage st(g->stream);
        const float* a = st.in(rgb, 3 * n);
        const float* b = st.in(depth, n);
        const float* c = st.in(normal, 3 * n);
        const float* w = st.in(wsum, n);
        const float* t = st.in(tgt_rgb, 3 * n);
        const float* pd = st.in(prior_depth, n);
        const float* pn = st.in(prior_normal, 3 * n);
        const uint32_t* ci = st.in(cam_idx, prior_normal ? n : 0);
        const svr_camera* cm = st.in(cams, prior_normal ? n_cams : 0);
        float* gc = st.out(d_rgb, 3 * n);
        float* gd = st.out(d_depth, n);
        float* gn = st.out(d_normal, 3 * n);
        double* acc = g->loss_acc.as<double>();
        svr_internal::launch_render_losses(n, a, b, c, w, t, pd, pn, ci, cm, lambda_d, lambda_n, gc, gd, gn, acc,
                                           g->stream);
        double h[16] = {0};
        if (stats) SVR_CK(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
        st.finish();
        if (stats) {
            SVR_CK(cudaStreamSynchronize(g->stream));
            svr_loss_stats o{};
            o.n_c = static_cast<uint64_t>(h[5]);
            o.n_d = static_cast<uint64_t>(h[0]);
            o.n_n = static_cast<uint64_t>(h[6]);
            o.L_c = o.n_c ? h[10] / h[5] : 0.0;
            o.L_d = o.n_d ? h[11] / h[0] : 0.0;
            o.L_n = o.n_n ? h[12] / h[6] : 0.0;
            o.total = o.L_c + lambda_d * o.L_d + lambda_n * o.L_n;
            o.a = h[7];
            o.b = h[8];
            o.singular = h[9] != 0.0 ? 1 : 0;
            *stats = o;
        }
    });
}

int svr_sample_frame_rays(svr_grid* g, const svr_camera* cams, uint32_t n_frames, const float* rgb,
                          const float* depth, const float* normal, uint32_t images_per_batch,
                          uint32_t rays_per_image, uint64_t seed, double* o, double* d, float* tgt_rgb,
                          float* prior_depth, float* prior_normal, uint32_t* cam_idx, uint32_t* pixel) {
    return guarded([&] {
        if (!n_frames || !cams) throw Fail{SVR_ERR_DATA, "sample_frame_rays: no frames"};
        if (!o || !d) throw Fail{SVR_ERR_DATA, "sample_frame_rays: ray outputs required"};
        if (tgt_rgb && !rgb) throw Fail{SVR_ERR_DATA, "sample_frame_rays: colour targets need the rgb frames"};
        std::vector<svr_camera> hc(n_frames);
        if (is_device_ptr(cams))
            SVR_CK(cudaMemcpy(hc.data(), cams, n_frames * sizeof(svr_camera), cudaMemcpyDeviceToHost));
        else
            std::memcpy(hc.data(), cams, n_frames * sizeof(svr_camera));
        const int32_t W = hc[0].width, H = hc[0].height;
        for (const svr_camera& c : hc)
            if (c.width != W || c.height != H) throw Fail{SVR_ERR_CONFIG, "sample_frame_rays: frames differ in size"};
        const uint64_t n = static_cast<uint64_t>(images_per_batch) * rays_per_image;
        if (!n) return;
        if (static_cast<uint64_t>(n_frames) * W * H >= (1ull << 32))
            throw Fail{SVR_ERR_CONFIG, "sample_frame_rays: more than 2^32 frame pixels"};
        DeviceGuard dg(g->device);
        Stage st(g->stream);
        const size_t npx = static_cast<size_t>(n_frames) * W * H;
        const svr_camera* dc = st.in(cams, n_frames);
        const float* ri = st.in(rgb, 3 * npx);
        const float* di = st.in(depth, npx);
        const float* ni = st.in(normal, 3 * npx);
        double* a = st.out(o, 3 * n);
        double* b = st.out(d, 3 * n);
        float* t = st.out(tgt_rgb, 3 * n);
        float* pd = st.out(prior_depth, n);
        float* pn = st.out(prior_normal, 3 * n);
        uint32_t* ci = st.out(cam_idx, n);
        uint32_t* px = st.out(pixel, n);
        svr_internal::launch_sample_frame_rays(dc, n_frames, W, H, rays_per_image, n, seed, ri, di, ni, a, b, t, pd, pn,
                                               ci, px, g->stream);
        st.finish();
    });
}

int svr_band_points(svr_grid* g, double band, uint64_t cap, double* out, uint64_t* n_out) {
    return guarded([&] {
        if (!g->ctx_valid) throw Fail{SVR_ERR_DATA, "band_points: no retained forward context"};
        if (!g->ctx_rec) throw Fail{SVR_ERR_CONFIG, "band_points: needs the forward records (tuning records = 1)"};
        DeviceGuard dg(g->device);
        const uint64_t n = g->ctx_n;
        uint64_t total = 0;
        if (n) {
            g->scratch_a.ensure(8 * n + 16);
            const size_t tb = std::max<size_t>(svr_internal::band_points_tmp_bytes(n), 16);
            g->scratch_c.ensure(tb);
            Stage st(g->stream);
            double* pts = out ? st.out(out, 3 * cap) : nullptr;
            total = svr_internal::band_points(g->ctx_o, g->ctx_d, g->counts.as<uint32_t>(), g->tbuf.as<double>(),
                                              g->rec.as<float4>(), n, g->ctx_S, static_cast<float>(band),
                                              g->scratch_a.as<uint32_t>(), g->scratch_c.p, tb, cap, pts, g->stream);
            st.finish();
        }
        if (n_out) *n_out = total;
    });
}

// ---------------------------------------------------------------------------
// Marching cubes (meshing.cpp:168-273) and the PLY writer (mesh_io.cpp:30-68).
// ---------------------------------------------------------------------------
int svr_marching_cubes(svr_grid* g, double iso, uint64_t* n_vertices, uint64_t* n_triangles) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        g->mesh.nv = g->mesh.nt = 0;
        if (g->n()) {
            // edge keys: voxel coordinates relative to the AABB in 21 / 21 / 20 bits
            const int64_t ex = (static_cast<int64_t>(g->hi[0]) - g->lo[0] + 1) * kRes;
            const int64_t ey = (static_cast<int64_t>(g->hi[1]) - g->lo[1] + 1) * kRes;
            const int64_t ez = (static_cast<int64_t>(g->hi[2]) - g->lo[2] + 1) * kRes;
            if (ex >= (1 << 21) || ey >= (1 << 21) || ez >= (1 << 20))
                throw Fail{SVR_ERR_CONFIG, "marching_cubes: block AABB wider than 2^18 x 2^18 x 2^17 blocks"};
            g->ensure_lookup();
            try {
                svr_internal::run_marching_cubes(g->view(), g->coords4, g->nbr.as<uint32_t>(), g->lo, iso, g->mesh,
                                                 g->stream);
            } catch (const svr_internal::Status& e) {
                throw Fail{e.code, e.msg};
            }
        }
        if (n_vertices) *n_vertices = g->mesh.nv;
        if (n_triangles) *n_triangles = g->mesh.nt;
    });
}

int svr_mesh_get(svr_grid* g, double* vertices, double* normals, double* colors, int32_t* labels,
                 int32_t* triangles) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint64_t nv = g->mesh.nv, nt = g->mesh.nt;
        auto copy = [&](void* dst, const void* src, size_t bytes) {
            if (!dst || !bytes) return;
            SVR_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, g->stream));
        };
        copy(vertices, g->mesh.v, nv * 24);
        copy(normals, g->mesh.n, nv * 24);
        copy(colors, g->mesh.c, nv * 24);
        copy(labels, g->mesh.l, nv * 4);
        copy(triangles, g->mesh.t, nt * 12);
        SVR_CK(cudaStreamSynchronize(g->stream));
    });
}

int svr_mesh_save_ply(svr_grid* g, const char* path) {
    return guarded([&] {
        DeviceGuard dg(g->device);
        const uint64_t nv = g->mesh.nv, nt = g->mesh.nt;
        std::vector<double> v(3 * nv), n(3 * nv), c(3 * nv);
        std::vector<int32_t> l(nv), t(3 * nt);
        if (nv) {
            SVR_CK(cudaMemcpyAsync(v.data(), g->mesh.v, nv * 24, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaMemcpyAsync(n.data(), g->mesh.n, nv * 24, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaMemcpyAsync(c.data(), g->mesh.c, nv * 24, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaMemcpyAsync(l.data(), g->mesh.l, nv * 4, cudaMemcpyDeviceToHost, g->stream));
        }
        if (nt) SVR_CK(cudaMemcpyAsync(t.data(), g->mesh.t, nt * 12, cudaMemcpyDeviceToHost, g->stream));
        SVR_CK(cudaStreamSynchronize(g->stream));
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Fail{SVR_ERR_DATA, std::string("export_ply: cannot open ") + path};
        // header of export_ply: positions, normals, uchar colours, int label, triangle lists
        os << "ply\nformat binary_little_endian 1.0\n"
           << "element vertex " << nv << "\n"
           << "property float x\nproperty float y\nproperty float z\n"
           << "property float nx\nproperty float ny\nproperty float nz\n"
           << "property uchar red\nproperty uchar green\nproperty uchar blue\n"
           << "property int label\n"
           << "element face " << nt << "\n"
           << "property list uchar int vertex_indices\n"
           << "end_header\n";
        const size_t rec = 12 + 12 + 3 + 4;
        std::vector<char> body(nv * rec + nt * 13);
        char* o = body.data();
        auto put = [&](const void* p, size_t k) {
            std::memcpy(o, p, k);
            o += k;
        };
        for (uint64_t i = 0; i < nv; ++i) {
            for (int a = 0; a < 3; ++a) {
                const float f = static_cast<float>(v[3 * i + a]);
                put(&f, 4);
            }
            for (int a = 0; a < 3; ++a) {
                const float f = static_cast<float>(n[3 * i + a]);
                put(&f, 4);
            }
            for (int a = 0; a < 3; ++a) {  // lround(clamp(c, 0, 1) * 255)
                const double cl = std::min(std::max(c[3 * i + a], 0.0), 1.0);
                const uint8_t u = static_cast<uint8_t>(std::lround(cl * 255.0));
                put(&u, 1);
            }
            put(&l[i], 4);
        }
        for (uint64_t i = 0; i < nt; ++i) {
            const uint8_t three = 3;
            put(&three, 1);
            put(&t[3 * i], 12);
        }
        os.write(body.data(), static_cast<std::streamsize>(body.size()));
        if (!os) throw Fail{SVR_ERR_DATA, std::string("export_ply: write failed for ") + path};
    });
}

// ---------------------------------------------------------------------------
// SDGV v1 snapshots (grid_io.cpp:37-97), streamed in chunks of blocks.
// ---------------------------------------------------------------------------
int svr_grid_save_sdgv(svr_grid* g, const char* path) {
    return guarded([&] {
        std::ofstream os(path, std::ios::binary);
        if (!os) throw Fail{SVR_ERR_DATA, std::string("save_grid: cannot open ") + path};
        const uint32_t ver = 1, B = kRes, C = static_cast<uint32_t>(g->C);
        const uint64_t nb = g->n();
        os.write("SDGV", 4);
        os.write(reinterpret_cast<const char*>(&ver), 4);
        os.write(reinterpret_cast<const char*>(&g->h), 8);
        os.write(reinterpret_cast<const char*>(&B), 4);
        os.write(reinterpret_cast<const char*>(&nb), 8);
        os.write(reinterpret_cast<const char*>(&C), 4);
        const uint32_t chunk = 4096;
        std::vector<float> sdf, w, rgb, lg;
        for (uint64_t f = 0; f < nb; f += chunk) {
            const uint32_t m = static_cast<uint32_t>(std::min<uint64_t>(chunk, nb - f));
            sdf.resize(static_cast<size_t>(m) * kVox);
            w.resize(static_cast<size_t>(m) * kVox);
            rgb.resize(static_cast<size_t>(m) * kVox * 3);
            lg.resize(static_cast<size_t>(m) * kVox * C);
            const int st = svr_grid_get_payload(g, static_cast<uint32_t>(f), m, sdf.data(), w.data(),
                                                rgb.data(), lg.data());
            if (st) throw Fail{st, svr_internal::g_err};
            for (uint32_t i = 0; i < m; ++i) {
                os.write(reinterpret_cast<const char*>(&g->coords[3 * (f + i)]), 12);
                os.write(reinterpret_cast<const char*>(&sdf[static_cast<size_t>(i) * kVox]), kVox * 4);
                os.write(reinterpret_cast<const char*>(&w[static_cast<size_t>(i) * kVox]), kVox * 4);
                os.write(reinterpret_cast<const char*>(&rgb[static_cast<size_t>(i) * kVox * 3]), kVox * 12);
                os.write(reinterpret_cast<const char*>(&lg[static_cast<size_t>(i) * kVox * C]),
                         static_cast<std::streamsize>(kVox) * 4 * C);
            }
        }
        if (!os) throw Fail{SVR_ERR_DATA, std::string("save_grid: write failed for ") + path};
    });
}

int svr_grid_load_sdgv(const char* path, int32_t device, svr_grid** out) {
    return guarded([&] {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw Fail{SVR_ERR_DATA, std::string("load_grid: cannot open ") + path};
        char magic[4];
        is.read(magic, 4);
        if (!is || std::memcmp(magic, "SDGV", 4) != 0) throw Fail{SVR_ERR_DATA, "load_grid: bad magic"};
        uint32_t ver = 0, B = 0, C = 0;
        double h = 0;
        uint64_t nb = 0;
        is.read(reinterpret_cast<char*>(&ver), 4);
        if (ver != 1) throw Fail{SVR_ERR_DATA, "load_grid: unsupported version"};
        is.read(reinterpret_cast<char*>(&h), 8);
        is.read(reinterpret_cast<char*>(&B), 4);
        is.read(reinterpret_cast<char*>(&nb), 8);
        is.read(reinterpret_cast<char*>(&C), 4);
        if (!is) throw Fail{SVR_ERR_DATA, "load_grid: truncated header"};
        std::unique_ptr<svr_grid> g(make_grid(h, static_cast<int32_t>(B), static_cast<int32_t>(C),
                                              std::max<uint64_t>(1ull << 21, nb), device));
        const uint32_t chunk = 4096;
        std::vector<int32_t> cc;
        std::vector<float> sdf, w, rgb, lg;
        std::vector<uint32_t> idx;
        for (uint64_t f = 0; f < nb; f += chunk) {
            const uint32_t m = static_cast<uint32_t>(std::min<uint64_t>(chunk, nb - f));
            cc.resize(3 * m);
            sdf.resize(static_cast<size_t>(m) * kVox);
            w.resize(sdf.size());
            rgb.resize(sdf.size() * 3);
            lg.resize(sdf.size() * C);
            for (uint32_t i = 0; i < m; ++i) {
                is.read(reinterpret_cast<char*>(&cc[3 * i]), 12);
                is.read(reinterpret_cast<char*>(&sdf[static_cast<size_t>(i) * kVox]), kVox * 4);
                is.read(reinterpret_cast<char*>(&w[static_cast<size_t>(i) * kVox]), kVox * 4);
                is.read(reinterpret_cast<char*>(&rgb[static_cast<size_t>(i) * kVox * 3]), kVox * 12);
                is.read(reinterpret_cast<char*>(&lg[static_cast<size_t>(i) * kVox * C]),
                        static_cast<std::streamsize>(kVox) * 4 * C);
                if (!is) throw Fail{SVR_ERR_DATA, "load_grid: truncated block data"};
            }
            idx.resize(m);
            int st = svr_grid_allocate_blocks(g.get(), cc.data(), m, idx.data());
            if (st) throw Fail{st, svr_internal::g_err};
            bool contiguous = true;
            for (uint32_t i = 0; i < m; ++i) contiguous = contiguous && idx[i] == idx[0] + i;
            if (contiguous) {
                st = svr_grid_set_payload(g.get(), idx[0], m, sdf.data(), w.data(), rgb.data(), lg.data());
                if (st) throw Fail{st, svr_internal::g_err};
            } else {  // duplicate records: later records overwrite (grid_io.cpp:90-95)
                for (uint32_t i = 0; i < m; ++i) {
                    const size_t o = static_cast<size_t>(i) * kVox;
                    st = svr_grid_set_payload(g.get(), idx[i], 1, &sdf[o], &w[o], &rgb[3 * o], &lg[C * o]);
                    if (st) throw Fail{st, svr_internal::g_err};
                }
            }
        }
        *out = g.release();
    });
}

}  // extern "C"
