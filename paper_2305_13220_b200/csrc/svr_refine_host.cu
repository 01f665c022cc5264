// Host C++ side of libsvr_b200.so, part 4 of the C-ABI (include/svr.h): the native refine
// loop -- the same composition as paper_2305_13220_b200/refine.py, with
// the frames and every per-step buffer owned on the device by an svr_refiner handle:
// K17 batch -> K4/K5 forward -> K15 losses -> K6 backward -> K16 band + K9 uniform points ->
// K10 Eikonal -> K11 RMSProp (lr decayed exponentially to lr * gamma over the run).
#include "svr_handle.h"

using namespace svr_dev;
using namespace svr_host;

struct svr_refiner {
    svr_grid* g = nullptr;
    svr_refine_config cfg{};
    uint32_t n_frames = 0;
    uint64_t n = 0;
    DevBuf cams, rgb, depth, normal;           // device copies of the frames
    DevBuf o, d, tgt, pd, pn, ci;              // the batch
    DevBuf out_rgb, out_depth, out_normal, out_wsum;
    DevBuf g_rgb, g_depth, g_normal;
    DevBuf pts;
    std::vector<svr_camera> host_cams;
};

namespace {
void upload(DevBuf& dst, const void* src, size_t bytes, cudaStream_t s) {
    dst.ensure(std::max<size_t>(bytes, 16));
    if (src) SVR_CK(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyDefault, s));
}
void ck(int st) {
    if (st) throw Fail{st, svr_last_error()};
}
}  // namespace

extern "C" {

void svr_refine_config_default(svr_refine_config* c) {
    *c = svr_refine_config{};
    c->rays_per_image = 1024;  // RenderConfig
    c->images_per_batch = 64;
    c->lambda_d = 0.1;
    c->lambda_n = 0.05;
    c->lambda_eik = 0.1;
    c->lr = 1e-3;
    c->gamma = 0.1;
    c->alpha = 0.99;
    c->eps = 1e-8;
    c->max_samples = 64;
    c->uniform_points = 16384;
    c->band_cap = 65536;
    c->seed = 0;
}

int svr_refiner_create(svr_grid* g, const svr_camera* cams, uint32_t n_frames, const float* rgb,
                       const float* depth, const float* normal, const svr_refine_config* cfg,
                       svr_refiner** out) {
    return guarded([&] {
        if (!cfg || !out || !cams || !rgb || !n_frames) throw Fail{SVR_ERR_DATA, "refiner: frames and config required"};
        if (!(cfg->step > 0.0) || !(cfg->beta > 0.0) || !(cfg->mu > 0.0))
            throw Fail{SVR_ERR_CONFIG, "refiner: step, beta and mu must be positive"};
        GridGuard dg(g);
        auto r = std::make_unique<svr_refiner>();
        r->g = g;
        r->cfg = *cfg;
        r->n_frames = n_frames;
        r->host_cams.resize(n_frames);
        if (is_device_ptr(cams))
            SVR_CK(cudaMemcpy(r->host_cams.data(), cams, n_frames * sizeof(svr_camera), cudaMemcpyDeviceToHost));
        else
            std::memcpy(r->host_cams.data(), cams, n_frames * sizeof(svr_camera));
        const size_t npx = static_cast<size_t>(n_frames) * r->host_cams[0].width * r->host_cams[0].height;
        cudaStream_t s = g->stream;
        upload(r->cams, r->host_cams.data(), n_frames * sizeof(svr_camera), s);
        upload(r->rgb, rgb, npx * 12, s);
        if (depth) upload(r->depth, depth, npx * 4, s);
        if (normal) upload(r->normal, normal, npx * 12, s);
        const uint64_t n = static_cast<uint64_t>(cfg->rays_per_image) * cfg->images_per_batch;
        r->n = n;
        for (DevBuf* b : {&r->o, &r->d}) b->ensure(24 * n);
        for (DevBuf* b : {&r->tgt, &r->pn, &r->out_rgb, &r->out_normal, &r->g_rgb, &r->g_normal}) b->ensure(12 * n);
        for (DevBuf* b : {&r->pd, &r->ci, &r->out_depth, &r->out_wsum, &r->g_depth}) b->ensure(4 * n);
        r->pts.ensure(24 * (static_cast<size_t>(cfg->band_cap) + cfg->uniform_points) + 24);
        SVR_CK(cudaStreamSynchronize(s));
        *out = r.release();
    });
}

int svr_refiner_step(svr_refiner* r, uint32_t i, uint32_t steps, svr_loss_stats* stats, double* eik_loss) {
    return guarded([&] {
        svr_grid* g = r->g;
        const svr_refine_config& c = r->cfg;
        GridGuard dg(g);
        const bool has_d = r->depth.p != nullptr, has_n = r->normal.p != nullptr;
        // seeds as paper_2305_13220_b200/refine.py (rank 0)
        ck(svr_sample_frame_rays(g, r->cams.as<svr_camera>(), r->n_frames, r->rgb.as<float>(),
                                 has_d ? r->depth.as<float>() : nullptr, has_n ? r->normal.as<float>() : nullptr,
                                 c.images_per_batch, c.rays_per_image, (c.seed * 1000003ull + i) * 65599ull,
                                 r->o.as<double>(), r->d.as<double>(), r->tgt.as<float>(), r->pd.as<float>(),
                                 r->pn.as<float>(), r->ci.as<uint32_t>(), nullptr));
        ck(svr_render_forward(g, r->o.as<double>(), r->d.as<double>(), r->n, c.step, c.max_samples, c.beta,
                              r->out_rgb.as<float>(), r->out_depth.as<float>(), r->out_normal.as<float>(),
                              r->out_wsum.as<float>(), nullptr));
        ck(svr_render_losses(g, r->n, r->out_rgb.as<float>(), r->out_depth.as<float>(), r->out_normal.as<float>(),
                             r->out_wsum.as<float>(), r->tgt.as<float>(), has_d ? r->pd.as<float>() : nullptr,
                             has_n ? r->pn.as<float>() : nullptr, r->ci.as<uint32_t>(), r->host_cams.data(),
                             r->n_frames, c.lambda_d, c.lambda_n, r->g_rgb.as<float>(), r->g_depth.as<float>(),
                             r->g_normal.as<float>(), stats));
        ck(svr_render_backward(g, r->g_rgb.as<float>(), r->g_depth.as<float>(), r->g_normal.as<float>()));
        uint64_t nb = 0;
        ck(svr_band_points(g, 0.5 * c.mu, c.band_cap, r->pts.as<double>(), &nb));
        uint64_t m = std::min<uint64_t>(nb, c.band_cap);
        if (c.uniform_points) {
            ck(svr_sample_uniform(g, c.uniform_points, (c.seed * 7919ull + i) * 65599ull, r->pts.as<double>() + 3 * m));
            m += c.uniform_points;
        }
        double el = 0.0;
        uint64_t nv = 0;
        if (m && c.lambda_eik > 0.0) ck(svr_eikonal(g, r->pts.as<double>(), m, c.lambda_eik, &el, &nv));
        if (eik_loss) *eik_loss = el;
        const double lr = c.lr * std::pow(c.gamma, static_cast<double>(i) / std::max<uint32_t>(steps - 1, 1));
        ck(svr_rmsprop_step(g, static_cast<float>(lr), static_cast<float>(c.alpha), static_cast<float>(c.eps)));
        if (stats) stats->total += c.lambda_eik * el;
    });
}

int svr_refiner_destroy(svr_refiner* r) {
    return guarded([&] {
        if (!r) return;
        GridGuard dg(r->g);
        SVR_CK(cudaStreamSynchronize(r->g->stream));
        delete r;
    });
}

}  // extern "C"
