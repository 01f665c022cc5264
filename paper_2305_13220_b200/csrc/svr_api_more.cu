// Host C++ side of libsvr_b200.so, part 3 of the C-ABI (include/svr.h): fusion and
// de-noising, the peer-memory gradient reduction, refinement losses and batches, marching
// cubes and the PLY writer.
#include "svr_handle.h"

using namespace svr_dev;
using namespace svr_host;

extern "C" {

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
        g->fuse_sum.swap(s2);
        g->fuse_cnt.swap(c2);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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
        GridGuard dg(g);
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

int svr_mesh_save_obj(svr_grid* g, const char* path) {
    return guarded([&] {
        GridGuard dg(g);
        const uint64_t nv = g->mesh.nv, nt = g->mesh.nt;
        std::vector<double> v(3 * nv);
        std::vector<int32_t> t(3 * nt);
        if (nv) SVR_CK(cudaMemcpyAsync(v.data(), g->mesh.v, nv * 24, cudaMemcpyDeviceToHost, g->stream));
        if (nt) SVR_CK(cudaMemcpyAsync(t.data(), g->mesh.t, nt * 12, cudaMemcpyDeviceToHost, g->stream));
        SVR_CK(cudaStreamSynchronize(g->stream));
        std::ofstream os(path);
        if (!os) throw Fail{SVR_ERR_DATA, std::string("export_obj: cannot open ") + path};
        os.precision(9);  // export_obj (mesh_io.cpp:155-164): "v x y z", 1-based "f i j k"
        for (uint64_t i = 0; i < nv; ++i) os << "v " << v[3 * i] << " " << v[3 * i + 1] << " " << v[3 * i + 2] << "\n";
        for (uint64_t i = 0; i < nt; ++i)
            os << "f " << t[3 * i] + 1 << " " << t[3 * i + 1] + 1 << " " << t[3 * i + 2] + 1 << "\n";
        if (!os) throw Fail{SVR_ERR_DATA, std::string("export_obj: write failed for ") + path};
    });
}

int svr_mesh_save_ply(svr_grid* g, const char* path) {
    return guarded([&] {
        GridGuard dg(g);
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

}  // extern "C"
