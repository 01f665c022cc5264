// K8r: the multi-GPU active-block gradient all-reduce without host synchronisation
// (the reference only states the contract: rays are independent and the
// voxel gradients of all workers are summed, proj/src/core/parallel.cpp:35-63).
//
// Every rank holds a replica of the grid and the gradients of its own ray shard.  One
// reduction = three stream-ordered phases per rank, separated by cross-rank event waits:
//   publish  record done[r] after the backward
//   sum      wait done[q] of every rank q; u = OR_q active_q (peer reads of the u8 flags);
//            ascending compaction of u (device-side count, identical on every rank); over its
//            1/W slice of that list each rank sums the rows of the W gradient planes in rank
//            order and stores the sum into all W planes (reduce-scatter + all-gather in one
//            pass over NVLink peer memory); record reduced[r]
//   adopt    wait reduced[q] of every rank; active = u
// No phase reads a count or a flag on the host.  Single process (svr_reduce_grads: one
// handle per device, peer access between the devices) runs the phases back to back with
// in-process events; multi-process (svr_peer_group_*, CUDA IPC handles for the planes, the
// flag arrays and the interprocess events) needs a host-side rendezvous between the phases
// so that every rank has *recorded* its event before another one waits on it -- a CPU
// barrier, not a device synchronisation.  svr_reduce_grads falls back to NCCL
// (ncclCommInitAll + grouped ncclAllReduce, dlopen'ed) when the devices cannot reach each
// other's memory; that path reads the union count on the host once.
#include <dlfcn.h>

#include <map>
#include <mutex>
#include <set>

#include <nccl.h>

#include "svr_handle.h"

namespace svr_dev {
namespace {

constexpr int kMaxRanks = 8;
struct RankPtrs {
    float4* grad[kMaxRanks];
    const uint8_t* act[kMaxRanks];
};

// u[b] = OR over ranks of active_q[b]; four flags per thread.
__global__ void k_mask_union(RankPtrs rp, uint32_t world, uint32_t n, uint8_t* u) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    if (i + 4 <= n) {
        uint32_t v = 0;
        for (uint32_t q = 0; q < world; ++q) v |= *reinterpret_cast<const uint32_t*>(rp.act[q] + i);
        *reinterpret_cast<uint32_t*>(u + i) = v;
    } else {
        for (uint32_t b = i; b < n; ++b) {
            uint8_t v = 0;
            for (uint32_t q = 0; q < world; ++q) v |= rp.act[q][b];
            u[b] = v;
        }
    }
}

// Rank `rank` of `world` owns rows [c rank / W, c (rank + 1) / W) of the ascending list (c read
// on the device).  Thread v of a CTA handles voxel v of one row: the W values are summed in
// rank order (the same bits on every rank) and stored into every plane.
__global__ void __launch_bounds__(512) k_peer_allreduce_dev(RankPtrs rp, uint32_t world, uint32_t rank,
                                                            const uint32_t* __restrict__ rows,
                                                            const unsigned long long* __restrict__ count) {
    const unsigned long long c = *count;
    const unsigned long long first = c * rank / world, last = c * (rank + 1) / world;
    for (unsigned long long j = first + blockIdx.x; j < last; j += gridDim.x) {
        const size_t v = static_cast<size_t>(rows[j]) * kVox + threadIdx.x;
        float4 acc = rp.grad[0][v];
        for (uint32_t q = 1; q < world; ++q) {
            const float4 x = rp.grad[q][v];
            acc.x += x.x, acc.y += x.y, acc.z += x.z, acc.w += x.w;
        }
        for (uint32_t q = 0; q < world; ++q) rp.grad[q][v] = acc;
    }
}

// pack / unpack of the rows of a device-count list (NCCL fallback)
__global__ void __launch_bounds__(128) k_pack_rows(const float4* __restrict__ grad, const uint32_t* __restrict__ rows,
                                                   const unsigned long long* __restrict__ count, float4* out) {
    const unsigned long long c = *count;
    for (unsigned long long j = blockIdx.x; j < c; j += gridDim.x) {
        const size_t src = static_cast<size_t>(rows[j]) * kVox, dst = j * kVox;
#pragma unroll
        for (int k = 0; k < 4; ++k) out[dst + threadIdx.x + 128 * k] = grad[src + threadIdx.x + 128 * k];
    }
}
__global__ void __launch_bounds__(128) k_unpack_rows(float4* grad, const uint32_t* __restrict__ rows,
                                                     const unsigned long long* __restrict__ count,
                                                     const float4* __restrict__ in) {
    const unsigned long long c = *count;
    for (unsigned long long j = blockIdx.x; j < c; j += gridDim.x) {
        const size_t dst = static_cast<size_t>(rows[j]) * kVox, src = j * kVox;
#pragma unroll
        for (int k = 0; k < 4; ++k) grad[dst + threadIdx.x + 128 * k] = in[src + threadIdx.x + 128 * k];
    }
}

}  // namespace
}  // namespace svr_dev

namespace {

// The per-grid reduction state lives in the handle (red_*); this makes sure it exists.
void ensure_red_state(svr_grid* g) {
    const uint32_t nb = static_cast<uint32_t>(g->n());
    g->red_union.ensure(std::max<uint32_t>(nb, 4) + 16);
    g->red_list.ensure(std::max<uint32_t>(nb, 1) * 4);
    g->red_count.ensure(8 + 4 * ((nb + 1023) / 1024 + 2));
    for (cudaEvent_t* e : {&g->red_done, &g->red_reduced})
        if (!*e) SVR_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming | cudaEventInterprocess));
}

unsigned sum_grid(int num_sms) { return static_cast<unsigned>(num_sms) * 4u; }

// phase "sum" on one rank: union -> compaction -> own slice of the peer all-reduce
void launch_sum(svr_grid* g, const RankPtrs& rp, uint32_t world, uint32_t rank) {
    const uint32_t nb = static_cast<uint32_t>(g->n());
    uint8_t* u = g->red_union.as<uint8_t>();
    auto* dcount = g->red_count.as<unsigned long long>();
    const unsigned threads = 256, flags_per_cta = threads * 4;
    if (nb) svr_dev::k_mask_union<<<(nb + flags_per_cta - 1) / flags_per_cta, threads, 0, g->stream>>>(rp, world, nb, u);
    svr_internal::launch_active_list(u, nb, g->red_list.as<uint32_t>(), dcount, g->stream);
    if (nb)
        svr_dev::k_peer_allreduce_dev<<<std::min<unsigned>(nb, sum_grid(g->num_sms)), 512, 0, g->stream>>>(
            rp, world, rank, g->red_list.as<uint32_t>(), dcount);
    SVR_LAUNCHED();
}

void launch_adopt(svr_grid* g) {
    const uint32_t nb = static_cast<uint32_t>(g->n());
    if (nb) SVR_CK(cudaMemcpyAsync(g->active, g->red_union.p, nb, cudaMemcpyDeviceToDevice, g->stream));
}

// ---- NCCL, loaded on first use (the product library does not link it) -------------------
struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("NCCL not found: ") + dlerror();
            return;
        }
        api.commInitAll = reinterpret_cast<decltype(api.commInitAll)>(dlsym(h, "ncclCommInitAll"));
        api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
        api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
        api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
        api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.commInitAll && api.allReduce && api.groupStart && api.groupEnd && api.errStr;
        if (!api.ok) api.why = "NCCL library lacks an entry point";
    });
    return api;
}
#define SVR_NCCL(expr)                                                                          \
    do {                                                                                        \
        const ncclResult_t r_ = (expr);                                                         \
        if (r_ != ncclSuccess) throw Fail{SVR_ERR_CUDA, std::string(#expr) + ": " + nccl().errStr(r_)}; \
    } while (0)

// communicators per device list, created once per process
std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;
std::vector<ncclComm_t>& comms_for(const std::vector<int>& devs) {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comms.find(devs);
    if (it != g_comms.end()) return it->second;
    std::vector<ncclComm_t> c(devs.size());
    SVR_NCCL(nccl().commInitAll(c.data(), static_cast<int>(devs.size()), devs.data()));
    return g_comms.emplace(devs, std::move(c)).first->second;
}

std::mutex g_peer_mu;
std::set<std::pair<int, int>> g_peer_enabled;
// true when every ordered pair of distinct devices can (and now does) access peer memory
bool enable_peer_access(const std::vector<int>& devs) {
    for (int a : devs)
        for (int b : devs) {
            if (a == b) continue;
            int can = 0;
            SVR_CK(cudaDeviceCanAccessPeer(&can, a, b));
            if (!can) return false;
        }
    std::lock_guard<std::mutex> lk(g_peer_mu);
    for (int a : devs)
        for (int b : devs) {
            if (a == b || g_peer_enabled.count({a, b})) continue;
            DeviceGuard dg(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SVR_CK(e);
            cudaGetLastError();
            g_peer_enabled.insert({a, b});
        }
    return true;
}

void reduce_nccl(svr_grid* const* grids, uint32_t n) {
    if (!nccl().ok) throw Fail{SVR_ERR_CUDA, "reduce_grads (nccl): " + nccl().why};
    std::vector<int> devs(n);
    for (uint32_t i = 0; i < n; ++i) devs[i] = grids[i]->device;
    if (std::set<int>(devs.begin(), devs.end()).size() != n)
        throw Fail{SVR_ERR_CONFIG, "reduce_grads (nccl): one handle per device"};
    auto& comms = comms_for(devs);
    const uint32_t nb = static_cast<uint32_t>(grids[0]->n());
    // 1. union of the active flags
    SVR_NCCL(nccl().groupStart());
    for (uint32_t i = 0; i < n; ++i) {
        DeviceGuard dg(devs[i]);
        SVR_NCCL(nccl().allReduce(grids[i]->active, grids[i]->red_union.p, nb, ncclUint8, ncclMax, comms[i],
                                  grids[i]->stream));
    }
    SVR_NCCL(nccl().groupEnd());
    // 2. compaction (device count), one host read of the count (identical on every rank)
    for (uint32_t i = 0; i < n; ++i) {
        DeviceGuard dg(devs[i]);
        svr_internal::launch_active_list(grids[i]->red_union.as<uint8_t>(), nb, grids[i]->red_list.as<uint32_t>(),
                                         grids[i]->red_count.as<unsigned long long>(), grids[i]->stream);
        SVR_LAUNCHED();
    }
    unsigned long long c = 0;
    {
        DeviceGuard dg(devs[0]);
        SVR_CK(cudaMemcpyAsync(&c, grids[0]->red_count.p, 8, cudaMemcpyDeviceToHost, grids[0]->stream));
        SVR_CK(cudaStreamSynchronize(grids[0]->stream));
    }
    // 3. pack -> grouped all-reduce(SUM) -> unpack, then adopt the union
    for (uint32_t i = 0; i < n; ++i) {
        svr_grid* g = grids[i];
        DeviceGuard dg(devs[i]);
        g->red_pack.ensure(std::max<unsigned long long>(c, 1) * kVox * sizeof(float4));
        if (c)
            svr_dev::k_pack_rows<<<std::min<unsigned long long>(c, sum_grid(g->num_sms)), 128, 0, g->stream>>>(
                g->grad, g->red_list.as<uint32_t>(), g->red_count.as<unsigned long long>(), g->red_pack.as<float4>());
        SVR_LAUNCHED();
    }
    if (c) {
        SVR_NCCL(nccl().groupStart());
        for (uint32_t i = 0; i < n; ++i) {
            DeviceGuard dg(devs[i]);
            SVR_NCCL(nccl().allReduce(grids[i]->red_pack.p, grids[i]->red_pack.p, c * kVox * 4, ncclFloat32, ncclSum,
                                      comms[i], grids[i]->stream));
        }
        SVR_NCCL(nccl().groupEnd());
    }
    for (uint32_t i = 0; i < n; ++i) {
        svr_grid* g = grids[i];
        DeviceGuard dg(devs[i]);
        if (c)
            svr_dev::k_unpack_rows<<<std::min<unsigned long long>(c, sum_grid(g->num_sms)), 128, 0, g->stream>>>(
                g->grad, g->red_list.as<uint32_t>(), g->red_count.as<unsigned long long>(), g->red_pack.as<float4>());
        SVR_LAUNCHED();
        launch_adopt(g);
    }
}

void reduce_peer(svr_grid* const* grids, uint32_t n) {
    RankPtrs rp{};
    for (uint32_t q = 0; q < n; ++q) rp.grad[q] = grids[q]->grad, rp.act[q] = grids[q]->active;
    for (uint32_t i = 0; i < n; ++i) {  // publish
        DeviceGuard dg(grids[i]->device);
        SVR_CK(cudaEventRecord(grids[i]->red_done, grids[i]->stream));
    }
    for (uint32_t i = 0; i < n; ++i) {  // sum
        DeviceGuard dg(grids[i]->device);
        for (uint32_t q = 0; q < n; ++q)
            if (q != i) SVR_CK(cudaStreamWaitEvent(grids[i]->stream, grids[q]->red_done, 0));
        launch_sum(grids[i], rp, n, i);
        SVR_CK(cudaEventRecord(grids[i]->red_reduced, grids[i]->stream));
    }
    for (uint32_t i = 0; i < n; ++i) {  // adopt
        DeviceGuard dg(grids[i]->device);
        for (uint32_t q = 0; q < n; ++q)
            if (q != i) SVR_CK(cudaStreamWaitEvent(grids[i]->stream, grids[q]->red_reduced, 0));
        launch_adopt(grids[i]);
    }
}

}  // namespace

// multi-process peer group (one per rank)
struct svr_peer_group {
    svr_grid* g = nullptr;
    uint32_t world = 0, rank = 0;
    RankPtrs rp{};
    cudaEvent_t done[kMaxRanks] = {}, reduced[kMaxRanks] = {};
    std::vector<void*> opened_mem;
    std::vector<cudaEvent_t> opened_ev;
};

extern "C" {

int svr_reduce_grads_ex(svr_grid* const* grids, uint32_t n, int32_t mode) {
    return guarded([&] {
        if (!grids || n < 1 || n > kMaxRanks) throw Fail{SVR_ERR_CONFIG, "reduce_grads: 1 <= n <= 8 handles"};
        if (mode < SVR_REDUCE_AUTO || mode > SVR_REDUCE_NCCL) throw Fail{SVR_ERR_CONFIG, "reduce_grads: unknown mode"};
        const uint64_t nb = grids[0]->n();
        for (uint32_t i = 0; i < n; ++i) {
            if (!grids[i]) throw Fail{SVR_ERR_CONFIG, "reduce_grads: null handle"};
            if (grids[i]->n() != nb) throw Fail{SVR_ERR_DATA, "reduce_grads: the replicas differ in block count"};
            GridGuard dg(grids[i]);
            ensure_red_state(grids[i]);
        }
        if (nb == 0 || (n == 1 && mode != SVR_REDUCE_NCCL)) return;  // one handle: already the sum
        std::vector<int> devs(n);
        for (uint32_t i = 0; i < n; ++i) devs[i] = grids[i]->device;
        const bool peer = mode != SVR_REDUCE_NCCL && enable_peer_access(devs);
        if (mode == SVR_REDUCE_PEER && !peer) throw Fail{SVR_ERR_CUDA, "reduce_grads: no peer access between the devices"};
        if (peer) reduce_peer(grids, n);
        else reduce_nccl(grids, n);
    });
}

int svr_reduce_grads(svr_grid* const* grids, uint32_t n) { return svr_reduce_grads_ex(grids, n, SVR_REDUCE_AUTO); }

int svr_peer_export_get(svr_grid* g, svr_peer_export* out) {
    return guarded([&] {
        if (!out) throw Fail{SVR_ERR_DATA, "peer_export: output required"};
        GridGuard dg(g);
        if (!g->grad || !g->n()) throw Fail{SVR_ERR_DATA, "peer_export: the grid has no blocks yet"};
        ensure_red_state(g);
        static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(out->grad), "IPC handle size");
        static_assert(sizeof(cudaIpcEventHandle_t) == sizeof(out->ev_done), "IPC event handle size");
        cudaIpcMemHandle_t hg, ha;
        cudaIpcEventHandle_t he, hr;
        SVR_CK(cudaIpcGetMemHandle(&hg, g->grad));
        SVR_CK(cudaIpcGetMemHandle(&ha, g->active));
        SVR_CK(cudaIpcGetEventHandle(&he, g->red_done));
        SVR_CK(cudaIpcGetEventHandle(&hr, g->red_reduced));
        std::memcpy(out->grad, &hg, sizeof(hg));
        std::memcpy(out->active, &ha, sizeof(ha));
        std::memcpy(out->ev_done, &he, sizeof(he));
        std::memcpy(out->ev_reduced, &hr, sizeof(hr));
        out->n_blocks = g->n();
        out->device = g->device;
        out->reserved = 0;
    });
}

int svr_peer_group_open(svr_grid* g, const svr_peer_export* all, uint32_t world, uint32_t rank,
                        svr_peer_group** out) {
    return guarded([&] {
        if (!out || !all) throw Fail{SVR_ERR_DATA, "peer_group_open: arguments required"};
        if (world < 1 || world > kMaxRanks || rank >= world) throw Fail{SVR_ERR_CONFIG, "peer_group_open: 1 <= world <= 8"};
        GridGuard dg(g);
        ensure_red_state(g);
        auto pg = std::make_unique<svr_peer_group>();
        pg->g = g, pg->world = world, pg->rank = rank;
        try {
            for (uint32_t q = 0; q < world; ++q) {
                if (all[q].n_blocks != g->n()) throw Fail{SVR_ERR_DATA, "peer_group_open: the replicas differ in block count"};
                if (q == rank) {
                    pg->rp.grad[q] = g->grad, pg->rp.act[q] = g->active;
                    pg->done[q] = g->red_done, pg->reduced[q] = g->red_reduced;
                    continue;
                }
                cudaIpcMemHandle_t hg, ha;
                cudaIpcEventHandle_t he, hr;
                std::memcpy(&hg, all[q].grad, sizeof(hg));
                std::memcpy(&ha, all[q].active, sizeof(ha));
                std::memcpy(&he, all[q].ev_done, sizeof(he));
                std::memcpy(&hr, all[q].ev_reduced, sizeof(hr));
                void *pgrad = nullptr, *pact = nullptr;
                SVR_CK(cudaIpcOpenMemHandle(&pgrad, hg, cudaIpcMemLazyEnablePeerAccess));
                pg->opened_mem.push_back(pgrad);
                SVR_CK(cudaIpcOpenMemHandle(&pact, ha, cudaIpcMemLazyEnablePeerAccess));
                pg->opened_mem.push_back(pact);
                SVR_CK(cudaIpcOpenEventHandle(&pg->done[q], he));
                pg->opened_ev.push_back(pg->done[q]);
                SVR_CK(cudaIpcOpenEventHandle(&pg->reduced[q], hr));
                pg->opened_ev.push_back(pg->reduced[q]);
                pg->rp.grad[q] = static_cast<float4*>(pgrad);
                pg->rp.act[q] = static_cast<const uint8_t*>(pact);
            }
        } catch (...) {
            for (void* p : pg->opened_mem) cudaIpcCloseMemHandle(p);
            for (cudaEvent_t e : pg->opened_ev) cudaEventDestroy(e);
            throw;
        }
        *out = pg.release();
    });
}

int svr_peer_reduce_phase(svr_peer_group* pg, int32_t phase) {
    return guarded([&] {
        if (!pg) throw Fail{SVR_ERR_DATA, "peer_reduce_phase: null group"};
        svr_grid* g = pg->g;
        GridGuard dg(g);
        if (g->grad != pg->rp.grad[pg->rank] || g->active != pg->rp.act[pg->rank])
            throw Fail{SVR_ERR_DATA, "peer_reduce_phase: the grid grew since the group was opened"};
        switch (phase) {
            case SVR_REDUCE_PUBLISH:
                SVR_CK(cudaEventRecord(g->red_done, g->stream));
                break;
            case SVR_REDUCE_SUM:
                for (uint32_t q = 0; q < pg->world; ++q)
                    if (q != pg->rank) SVR_CK(cudaStreamWaitEvent(g->stream, pg->done[q], 0));
                launch_sum(g, pg->rp, pg->world, pg->rank);
                SVR_CK(cudaEventRecord(g->red_reduced, g->stream));
                break;
            case SVR_REDUCE_ADOPT:
                for (uint32_t q = 0; q < pg->world; ++q)
                    if (q != pg->rank) SVR_CK(cudaStreamWaitEvent(g->stream, pg->reduced[q], 0));
                launch_adopt(g);
                break;
            default:
                throw Fail{SVR_ERR_CONFIG, "peer_reduce_phase: phase is 0 (publish), 1 (sum) or 2 (adopt)"};
        }
    });
}

int svr_peer_group_close(svr_peer_group* pg) {
    return guarded([&] {
        if (!pg) return;
        {
            DeviceGuard dg(pg->g->device);
            SVR_CK(cudaStreamSynchronize(pg->g->stream));
            for (void* p : pg->opened_mem) cudaIpcCloseMemHandle(p);
            for (cudaEvent_t e : pg->opened_ev) cudaEventDestroy(e);
        }
        delete pg;
    });
}

}  // extern "C"
