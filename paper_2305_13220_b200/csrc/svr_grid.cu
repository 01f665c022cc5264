// Host C++ side of libsvr_b200.so, part 1 of the C-ABI (include/svr.h): the svr_grid handle
// lifecycle, tuning, activation, payload, query, march and SDGV I/O.  It owns all device memory, stages host
// arrays, keeps the host mirror of block coordinates (grid.hpp:219-222) and rebuilds
// the dense AABB lookup index lazily.  There is no CPU compute fallback: every
// numerical result comes from the sm_100a kernels in svr_render.cu / svr_activate.cu /
// svr_grads.cu, and a missing or failing device surfaces as SVR_ERR_CUDA.
#include <map>
#include <mutex>

#include "svr_handle.h"

using namespace svr_dev;
using namespace svr_host;

namespace svr_internal {
thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace svr_internal

namespace svr_host {
namespace {
std::mutex g_cache_mu;
std::map<int, std::multimap<size_t, void*>> g_cache;  // device -> (true size, block)
}  // namespace

void* dev_alloc(size_t bytes, size_t* got) {
    bytes = std::max<size_t>(bytes, 256);
    int dev = 0;
    SVR_CK(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto& m = g_cache[dev];
        auto it = m.lower_bound(bytes);  // smallest cached block that fits, if not much larger
        if (it != m.end() && it->first <= bytes + bytes / 8 + (2u << 20)) {
            void* p = it->second;
            *got = it->first;
            m.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {  // give the cached blocks of this device back, retry
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(g_cache_mu);
        cudaDeviceSynchronize();
        for (auto& kv : g_cache[dev]) cudaFree(kv.second);
        g_cache[dev].clear();
        e = cudaMalloc(&p, bytes);
    }
    SVR_CK(e);
    *got = bytes;
    return p;
}

void dev_release(void* p, size_t bytes, int device) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache[device].emplace(bytes, p);
}
}  // namespace svr_host

namespace svr_internal {
unsigned sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    SVR_LCK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) SVR_LCK(cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev));
    return static_cast<unsigned>(cache[dev]);
}
void throw_cuda(cudaError_t e, const char* what) {
    throw svr_host::Fail{SVR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
}  // namespace svr_internal

namespace {

svr_grid* make_grid(double h, int32_t B, int32_t C, uint64_t capacity, int32_t device) {
    if (!(h > 0.0)) throw Fail{SVR_ERR_CONFIG, "grid: voxel_size must be positive"};  // grid.cpp:83
    if (B < 2) throw Fail{SVR_ERR_CONFIG, "grid: block_res must be >= 2"};
    if (B != kRes) throw Fail{SVR_ERR_CONFIG, "grid: this build specialises block_res = 8"};
    if (C < 1) throw Fail{SVR_ERR_CONFIG, "grid: label_channels must be >= 1"};
    // voxel addresses are 32-bit (block * 512 + local): at most 2^23 blocks (a 2^23-block grid
    // with C = 4 is ~250 GB, beyond one B200's 180 GB anyway)
    if (capacity > kMaxBlocks) throw Fail{SVR_ERR_CONFIG, "grid: capacity above 2^23 blocks"};
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
    size_t got = 0;
    g->slots = static_cast<HashSlot*>(dev_alloc(g->nslots * sizeof(HashSlot), &got));
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
    delete g;  // ~svr_grid synchronises the handle's stream, the side stream and the copy streams
    return SVR_OK;
}

int svr_grid_set_stream(svr_grid* g, void* s) {
    return guarded([&] {
        GridGuard dg(g);
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
        GridGuard dg(g);
        SVR_CK(cudaStreamSynchronize(g->stream));  // joined with the side stream (GridGuard)
        if (g->h2d) {
            SVR_CK(cudaStreamSynchronize(g->h2d));
            SVR_CK(cudaStreamSynchronize(g->d2h));
        }
    });
}

int svr_grid_join(svr_grid* g) {
    return guarded([&] { GridGuard dg(g); });
}

int svr_grid_get_info(svr_grid* g, svr_grid_info* out) {
    return guarded([&] {
        GridGuard dg(g);
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
        } else if (k == "sort_min_rays") {
            if (value < 0) throw Fail{SVR_ERR_CONFIG, "tuning: sort_min_rays must be >= 0"};
            g->sort_min_rays = static_cast<uint64_t>(value);
        } else if (k == "records") {
            g->use_records = value != 0;
        } else if (k == "bwd_pipe") {
            g->bwd_pipe = value != 0;
        } else if (k == "march_jump") {
            g->use_jump = value != 0;
        } else if (k == "zero_fused") {
            GridGuard dg(g);
            g->zero_fused = value != 0;
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
        GridGuard dg(g);
        g->lookup_pref = mode;
        g->dense_dirty = true;
        g->ensure_lookup();
    });
}

int svr_grid_allocate_blocks(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out) {
    return guarded([&] {
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
            g->scratch_e.ensure(static_cast<size_t>(n_frames) * (W + H) * sizeof(double));
            svr_internal::launch_depth_to_keys(dd, dc, n_frames, W, H, ds, sf_rows, sf_cols, g->L, ks,
                                               counters, counters + 1,
                                               reinterpret_cast<uint32_t*>(counters + 2),
                                               g->scratch_e.as<double>(), g->stream);
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
        g->scratch_d.ensure(std::max<uint64_t>(hc[0], 1) * 8);
        SVR_CK(cudaMemcpyAsync(g->scratch_d.p, ks.list, hc[0] * 8, cudaMemcpyDeviceToDevice, g->stream));
        g->commit(g->scratch_d.as<unsigned long long>(), hc[0], dilation, rep);
        SVR_CK(cudaStreamSynchronize(g->stream));
    });
    if (report) *report = rep;
    return st;
}

int svr_grid_find(svr_grid* g, const int32_t* coords, uint64_t n, uint32_t* idx_out) {
    return guarded([&] {
        GridGuard dg(g);
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
        if (!g->n()) return;
        GridGuard dg(g);
        const std::vector<int32_t>& hc = g->host_coords();
        if (is_device_ptr(out)) {
            SVR_CK(cudaMemcpy(out, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice));
        } else {
            std::memcpy(out, hc.data(), hc.size() * 4);
        }
    });
}

int svr_grid_set_payload(svr_grid* g, uint32_t first, uint32_t n, const float* sdf,
                         const float* weight, const float* rgb, const float* logits) {
    return guarded([&] {
        if (static_cast<uint64_t>(first) + n > g->n())
            throw Fail{SVR_ERR_DATA, "payload: block range out of bounds"};
        if (!n) return;
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        // the renderer's march kernel (march_variant), so the march parity tests cover it
        svr_internal::launch_march(g->view(), dO, dD, n, nullptr, step, max_samples, dc, dt, dl, g->stream);
        st.finish();
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
        const std::vector<int32_t>* hc = nullptr;
        {
            GridGuard dg(g);
            hc = &g->host_coords();
        }
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
                os.write(reinterpret_cast<const char*>(&(*hc)[3 * (f + i)]), 12);
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
