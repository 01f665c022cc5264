// Host C++ side of libsvr_b200.so, part 2 of the C-ABI (include/svr.h): render forward /
// backward (incl. the host_async pipelined host I/O), gradient planes, the active-block
// reduction plumbing, uniform sampling, Eikonal and RMSProp.
#include "svr_handle.h"

using namespace svr_dev;
using namespace svr_host;

extern "C" {

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

// The forward kernels on g->stream: optional pre-march ray order, K4 march (which also writes
// the post-march sort keys), optional post-march order, K5 forward (+ records).  dO / dD /
// outputs are device pointers.
void forward_kernels(svr_grid* g, const double* dO, const double* dD, uint64_t n, double step,
                     uint32_t max_samples, double beta, float* a, float* b, float* c, float* e) {
    g->ensure_rays(std::max<uint64_t>(n, 1), max_samples);
    const GridView v = g->view();
    g->ctx_order = nullptr;
    // below sort_min_rays the two ordering sorts cost more than the coherence they buy
    const bool sort = g->ray_sort != 0 && n > 1 && n >= g->sort_min_rays;
    const bool pre = sort && (g->ray_sort & 2), post = sort && (g->ray_sort & 1);
    if (sort) g->ord_tmp.ensure(std::max<size_t>(svr_internal::ray_order_tmp_bytes(n), 16));
    if (pre) {  // pre-march: origin + direction
        g->ord_keys.ensure(8 * n);
        g->ord_ids.ensure(8 * n);
        uint32_t* k = g->ord_keys.as<uint32_t>();
        uint32_t* id = g->ord_ids.as<uint32_t>();
        svr_internal::launch_ray_order(dO, dD, n, v, false, k, id, k + n, id + n, g->ord_tmp.p, g->ord_tmp.bytes,
                                       &g->ctx_order, g->stream);
    }
    uint32_t* k2 = nullptr;
    uint32_t* id2 = nullptr;
    if (post) {
        g->ord_keys2.ensure(8 * n);
        g->ord_ids2.ensure(8 * n);
        k2 = g->ord_keys2.as<uint32_t>();
        id2 = g->ord_ids2.as<uint32_t>();
    }
    svr_internal::launch_march(v, dO, dD, n, g->ctx_order, step, max_samples, g->counts.as<uint32_t>(),
                               g->tbuf.as<double>(), nullptr, g->stream, k2, id2, g->nvalid.as<unsigned long long>());
    if (post)  // post-march: first-sample block, keys written by the march
        svr_internal::launch_ray_order(dO, dD, n, v, true, k2, id2, k2 + n, id2 + n, g->ord_tmp.p, g->ord_tmp.bytes,
                                       &g->ctx_order, g->stream);
    g->ctx_rec = g->use_records;
    if (g->ctx_rec) g->rec.ensure(n * max_samples * 32);
    float4* recp = g->ctx_rec ? g->rec.as<float4>() : nullptr;
    // a pending svr_grad_zero_active rides along when each warp gets at most 8 row chunks
    // (512 B stores); otherwise it runs as its own kernel first
    const bool fuse_zero = g->zero_pending && n && g->n() * (kVox / 32) <= 8 * n;
    if (g->zero_pending && !fuse_zero) g->flush_zero();
    g->zero_pending = false;
    svr_internal::launch_render_forward(v, dO, dD, n, g->ctx_order, g->counts.as<uint32_t>(), g->tbuf.as<double>(),
                                        max_samples, step, beta, a, b, c, e, g->nvalid.as<unsigned long long>(),
                                        recp, g->stream, fuse_zero ? g->grad : nullptr, fuse_zero ? g->active : nullptr,
                                        fuse_zero ? g->active_list.as<uint32_t>() : nullptr,
                                        fuse_zero ? g->active_count.as<unsigned long long>() : nullptr);
}

void backward_kernels(svr_grid* g, const float* a, const float* b, const float* c) {
    const uint64_t n = g->ctx_n;
    const bool piped =
        g->bwd_pipe && g->ctx_rec &&
        svr_internal::launch_render_backward_pipe(g->view(), g->ctx_o, g->ctx_d, n, g->ctx_order,
                                                  g->counts.as<uint32_t>(), g->tbuf.as<double>(), g->ctx_S,
                                                  g->ctx_step, g->ctx_beta, a, b, c, g->rec.as<float4>(),
                                                  g->stream, g->num_sms);
    if (!piped)
        svr_internal::launch_render_backward(g->view(), g->ctx_o, g->ctx_d, n, g->ctx_order,
                                             g->counts.as<uint32_t>(), g->tbuf.as<double>(), g->ctx_S,
                                             g->ctx_step, g->ctx_beta, a, b, c,
                                             g->ctx_rec ? g->rec.as<float4>() : nullptr, g->stream);
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
        DeviceGuard dg(g->device);  // no flush: the forward kernel fuses a pending zeroing
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
        GridGuard dg(g);
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
        GridGuard dg(g);
        svr_render_stats s{};
        s.rays = g->ctx_valid ? g->ctx_n : 0;
        if (g->ctx_valid && g->ctx_n) {
            // marched samples from the counts; valid samples as counted by the last forward
            std::vector<uint32_t> cnt(g->ctx_n);
            unsigned long long v = 0;
            SVR_CK(cudaMemcpyAsync(cnt.data(), g->counts.p, 4 * g->ctx_n, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaMemcpyAsync(&v, g->nvalid.p, 8, cudaMemcpyDeviceToHost, g->stream));
            SVR_CK(cudaStreamSynchronize(g->stream));
            for (uint32_t c : cnt) s.samples += c;
            s.valid_samples = v;
        }
        *out = s;
    });
}

int svr_grad_zero(svr_grid* g) {
    return guarded([&] {
        GridGuard dg(g);
        if (!g->n()) return;
        SVR_CK(cudaMemsetAsync(g->grad, 0, g->n() * kVox * sizeof(float4), g->stream));
        SVR_CK(cudaMemsetAsync(g->active, 0, g->n(), g->stream));
    });
}

int svr_grad_get(svr_grid* g, float* g_sdf, float* g_rgb) {
    return guarded([&] {
        GridGuard dg(g);
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
        GridGuard dg(g);
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
            if ((!count || is_device_ptr(count)) && (!list || is_device_ptr(list))) {
                // device outputs: stream-ordered, no host read of the count (the list gets
                // all nb slots; entries past *count are unspecified)
                if (count) SVR_CK(cudaMemcpyAsync(count, dcount, 8, cudaMemcpyDeviceToDevice, g->stream));
                if (list && nb)
                    SVR_CK(cudaMemcpyAsync(list, g->active_list.p, 4ull * nb, cudaMemcpyDeviceToDevice, g->stream));
                st.finish();
                return;
            }
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
        GridGuard dg(g);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        Stage st(g->stream);
        const uint8_t* m = st.in(mask, nb);
        svr_internal::launch_set_active(g->active, m, nb, g->stream);
        st.finish();
    });
}

int svr_grad_pack(svr_grid* g, const uint32_t* blocks, uint64_t n, float* out) {
    return guarded([&] {
        GridGuard dg(g);
        Stage st(g->stream);
        const uint32_t* b = st.in(blocks, n);
        float* o = st.out(out, n * kVox * 4);
        svr_internal::launch_grad_pack(g->grad, b, n, reinterpret_cast<float4*>(o), g->stream);
        st.finish();
    });
}

int svr_grad_unpack(svr_grid* g, const uint32_t* blocks, uint64_t n, const float* in) {
    return guarded([&] {
        GridGuard dg(g);
        Stage st(g->stream);
        const uint32_t* b = st.in(blocks, n);
        const float* i = st.in(in, n * kVox * 4);
        svr_internal::launch_grad_unpack(g->grad, b, n, reinterpret_cast<const float4*>(i), g->stream);
        st.finish();
    });
}

int svr_grad_zero_active(svr_grid* g) {
    return guarded([&] {
        GridGuard dg(g);
        const uint32_t nb = static_cast<uint32_t>(g->n());
        if (!nb) return;
        g->active_list.ensure(nb * 4);
        g->active_count.ensure(8 + 4 * ((nb + 1023) / 1024 + 2));
        auto* dcount = g->active_count.as<unsigned long long>();
        svr_internal::launch_active_list(g->active, nb, g->active_list.as<uint32_t>(), dcount, g->stream);
        SVR_LAUNCHED();
        g->zero_pending = true;  // the next render_forward stores the zeros (zero_fused), or
        if (!g->zero_fused) g->flush_zero();  // now, in order
    });
}

int svr_sample_uniform(svr_grid* g, uint64_t n, uint64_t seed, double* out) {
    return guarded([&] {
        if (g->n() == 0) throw Fail{SVR_ERR_DATA, "sample_uniform: empty grid"};  // grid.cpp:358
        if (!n) return;
        GridGuard dg(g);
        Stage st(g->stream);
        double* o = st.out(out, 3 * n);
        svr_internal::launch_sample_uniform(g->coords4, static_cast<uint32_t>(g->n()), g->L, n, seed, o,
                                            g->stream);
        st.finish();
    });
}

int svr_eikonal(svr_grid* g, const double* x, uint64_t n, double scale, double* loss, uint64_t* n_valid) {
    return guarded([&] {
        GridGuard dg(g);
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
        GridGuard dg(g);
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
            g->rms.swap(fresh);
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

}  // extern "C"
