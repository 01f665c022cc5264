// Synthetic analytic-SDF scene fixtures (host C++, fixtures/libsvr_fixture.so -- NOT part of
// the product library).  Restates the reference generator proj/src/core/synthetic.cpp:42-192
// (scene, sdf, color, raycast, ring cameras) without Eigen, plus the payload / ray / gradient
// recipes of SURVEY.md 8(d).  Inputs only: nothing here runs inside the rendering hot path.
// Pinned bit for bit to the reference's own SyntheticScene compiled verbatim into
// oracle/_ref (tests/test_synthetic.py::test_fixture_equals_reference_generator).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "svr_synth.h"

namespace svr_internal {  // this library's own last-error slot (svr_fixture_last_error)
thread_local std::string g_fixture_err;
void set_error(const std::string& msg) { g_fixture_err = msg; }
}

namespace {

constexpr int kLabelWall = 0, kLabelFloor = 1, kLabelSphere = 2, kLabelBox = 3;
// synthetic.cpp:26-31
const double kBaseColor[4][3] = {
    {0.72, 0.70, 0.62}, {0.48, 0.36, 0.26}, {0.20, 0.45, 0.72}, {0.72, 0.30, 0.24}};

struct V3 {
    double x, y, z;
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double sqnorm(V3 a) { return (a.x * a.x + a.y * a.y) + a.z * a.z; }
double norm(V3 a) { return std::sqrt(sqnorm(a)); }
V3 scale(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
V3 normalized(V3 a) {
    const double z = sqnorm(a);
    return z > 0.0 ? scale(a, std::sqrt(z)) : a;
}
V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }

struct Object {
    bool is_sphere;
    V3 center;
    V3 half;
    int label;
};

// box_sdf (synthetic.cpp:33-38)
double box_sdf(V3 p, V3 half) {
    const double q[3] = {std::abs(p.x) - half.x, std::abs(p.y) - half.y, std::abs(p.z) - half.z};
    const V3 outside{std::max(q[0], 0.0), std::max(q[1], 0.0), std::max(q[2], 0.0)};
    const double inside = std::min(std::max(std::max(q[0], q[1]), q[2]), 0.0);
    return norm(outside) + inside;
}

int n_threads(int requested) {
    if (requested > 0) return requested;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

template <typename F>
void parallel_range(uint64_t n, int threads, F&& fn) {
    const int w = static_cast<int>(std::min<uint64_t>(std::max(1, threads), std::max<uint64_t>(n, 1)));
    if (w <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    const uint64_t chunk = (n + w - 1) / w;
    std::vector<std::thread> pool;
    for (int i = 0; i < w; ++i) {
        const uint64_t b = i * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& t : pool) t.join();
}

}  // namespace

struct svr_scene {
    svr_scene_spec spec;
    V3 room_half;
    std::vector<Object> objects;

    // SyntheticScene::sdf (synthetic.cpp:71-80)
    double sdf(V3 x) const {
        double d = std::min(std::min(room_half.x - std::abs(x.x), room_half.y - std::abs(x.y)),
                            room_half.z - std::abs(x.z));
        for (const Object& o : objects) {
            const double od = o.is_sphere ? norm(sub(x, o.center)) - o.half.x
                                          : box_sdf(sub(x, o.center), o.half);
            d = std::min(d, od);
        }
        return d;
    }
    // class of the surface nearest to x (fixture label for rgb / logits)
    int label(V3 x) const {
        const double dw[3] = {room_half.x - std::abs(x.x), room_half.y - std::abs(x.y),
                              room_half.z - std::abs(x.z)};
        int axis = 0;
        for (int a = 1; a < 3; ++a)
            if (dw[a] < dw[axis]) axis = a;
        double best = dw[axis];
        int lab = (axis == 2 && x.z < 0.0) ? kLabelFloor : kLabelWall;
        for (const Object& o : objects) {
            const double od = o.is_sphere ? norm(sub(x, o.center)) - o.half.x
                                          : box_sdf(sub(x, o.center), o.half);
            if (od < best) {
                best = od;
                lab = o.label;
            }
        }
        return lab;
    }
    // SyntheticScene::color (synthetic.cpp:82-87)
    void color(V3 x, int label, double* rgb) const {
        const double f = spec.texture_frequency;
        const double m = 1.0 + spec.texture_amplitude * std::sin(f * x.x + 1.3) *
                                   std::sin(f * x.y + 2.1) * std::sin(f * x.z + 0.7);
        for (int c = 0; c < 3; ++c) rgb[c] = std::min(std::max(kBaseColor[label][c] * m, 0.0), 1.0);
    }
    // SyntheticScene::raycast (synthetic.cpp:89-162): returns z-depth (camera-z unit dir)
    bool raycast(const svr_camera& cam, double u, double v, double& depth, int* label = nullptr,
                 V3* point = nullptr, V3* normal = nullptr) const {
        const double dc[3] = {(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, 1.0};
        V3 d;
        double dd[3];
        for (int i = 0; i < 3; ++i)
            dd[i] = (cam.R[3 * i] * dc[0] + cam.R[3 * i + 1] * dc[1]) + cam.R[3 * i + 2] * dc[2];
        d = {dd[0], dd[1], dd[2]};
        const V3 o{cam.t[0], cam.t[1], cam.t[2]};
        double best_t = std::numeric_limits<double>::max();
        bool hit = false;
        int best_label = -1;
        V3 best_n{0.0, 0.0, 1.0};
        const double rh[3] = {room_half.x, room_half.y, room_half.z};
        for (int a = 0; a < 3; ++a) {
            if (d[a] == 0.0) continue;
            const double plane = d[a] > 0.0 ? rh[a] : -rh[a];
            const double t = (plane - o[a]) / d[a];
            if (t > 1e-9 && t < best_t) {
                best_t = t;
                hit = true;
                best_label = (a == 2 && d[a] < 0.0) ? kLabelFloor : kLabelWall;
                const double nv = d[a] > 0.0 ? -1.0 : 1.0;  // synthetic.cpp:104-106
                best_n = {a == 0 ? nv : 0.0, a == 1 ? nv : 0.0, a == 2 ? nv : 0.0};
            }
        }
        for (const Object& obj : objects) {
            if (obj.is_sphere) {
                const V3 oc = sub(o, obj.center);
                const double A = sqnorm(d);
                const double B = 2.0 * dot(d, oc);
                const double C = sqnorm(oc) - obj.half.x * obj.half.x;
                const double disc = B * B - 4 * A * C;
                if (disc < 0.0) continue;
                const double t = (-B - std::sqrt(disc)) / (2 * A);
                if (t > 1e-9 && t < best_t) {
                    best_t = t;
                    hit = true;
                    best_label = obj.label;
                    // (o + t d - c).normalized() (synthetic.cpp:120)
                    const V3 q{o.x + t * d.x - obj.center.x, o.y + t * d.y - obj.center.y,
                               o.z + t * d.z - obj.center.z};
                    const double qn = std::sqrt(sqnorm(q));
                    best_n = {q.x / qn, q.y / qn, q.z / qn};
                }
            } else {
                double t0 = -std::numeric_limits<double>::max();
                double t1 = std::numeric_limits<double>::max();
                int enter_axis = -1;
                bool ok = true;
                for (int a = 0; a < 3 && ok; ++a) {
                    const double lo = obj.center[a] - obj.half[a];
                    const double hi = obj.center[a] + obj.half[a];
                    if (d[a] == 0.0) {
                        ok = o[a] > lo && o[a] < hi;
                        continue;
                    }
                    double ta = (lo - o[a]) / d[a];
                    double tb = (hi - o[a]) / d[a];
                    if (ta > tb) std::swap(ta, tb);
                    if (ta > t0) {
                        t0 = ta;
                        enter_axis = a;
                    }
                    t1 = std::min(t1, tb);
                }
                if (ok && t0 < t1 && t0 > 1e-9 && t0 < best_t && enter_axis >= 0) {
                    best_t = t0;
                    hit = true;
                    best_label = obj.label;
                    const double nv = d[enter_axis] > 0.0 ? -1.0 : 1.0;  // synthetic.cpp:147-149
                    best_n = {enter_axis == 0 ? nv : 0.0, enter_axis == 1 ? nv : 0.0, enter_axis == 2 ? nv : 0.0};
                }
            }
        }
        depth = best_t;
        if (label) *label = best_label;
        if (point) *point = {o.x + best_t * d.x, o.y + best_t * d.y, o.z + best_t * d.z};  // synthetic.cpp:158
        if (normal) *normal = best_n;
        return hit;
    }
    // SyntheticScene::camera_for_frame (synthetic.cpp:164-192)
    svr_camera camera(int frame) const {
        svr_camera cam{};
        cam.width = spec.width;
        cam.height = spec.height;
        cam.fx = (spec.width / 2.0) / std::tan(spec.fov_deg * M_PI / 360.0);
        cam.fy = cam.fx;
        cam.cx = (spec.width - 1) / 2.0;
        cam.cy = (spec.height - 1) / 2.0;
        const double theta = 2 * M_PI * frame / spec.n_frames;
        const double ring = 0.72 * std::min(room_half.x, room_half.y);
        const V3 eye{ring * std::cos(theta), ring * std::sin(theta),
                     0.35 * room_half.z * std::sin(2 * theta) + 0.05};
        const V3 target{0.25 * ring * std::cos(theta + 2.2), 0.25 * ring * std::sin(theta + 2.2),
                        0.5 * room_half.z * std::sin(3 * theta + 0.8)};
        const V3 forward = normalized(sub(target, eye));
        const V3 up{0.0, 0.0, 1.0};
        const V3 right = normalized(cross(forward, up));
        const V3 down = cross(forward, right);
        const V3 cols[3] = {right, down, forward};
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cam.R[3 * r + c] = cols[c][r];
        cam.t[0] = eye.x, cam.t[1] = eye.y, cam.t[2] = eye.z;
        return cam;
    }
};

extern "C" {

const char* svr_fixture_last_error(void) { return svr_internal::g_fixture_err.c_str(); }

void svr_scene_spec_default(svr_scene_spec* s) {  // synthetic.hpp:13-30
    s->room_w = 2.4;
    s->room_d = 2.2;
    s->room_h = 2.0;
    s->n_objects = 2;
    s->n_frames = 24;
    s->width = 320;
    s->height = 240;
    s->fov_deg = 70.0;
    s->label_channels = 4;
    s->texture_amplitude = 0.25;
    s->texture_frequency = 4.0;
    s->seed = 1;
}

// SyntheticScene ctor (synthetic.cpp:42-69)
int svr_scene_create(const svr_scene_spec* spec, svr_scene** out) {
    const svr_scene_spec& s = *spec;
    if (s.label_channels < 4) {
        svr_internal::set_error("synthetic: label_channels must be >= 4");
        return SVR_ERR_CONFIG;
    }
    if (s.n_frames < 2 || s.width < 16 || s.height < 16 || s.room_w < 0.5 || s.room_d < 0.5 ||
        s.room_h < 0.5 || s.n_objects < 0 || s.n_objects > 4) {
        svr_internal::set_error("synthetic: invalid scene spec");
        return SVR_ERR_CONFIG;
    }
    auto* sc = new svr_scene();
    sc->spec = s;
    sc->room_half = {s.room_w / 2, s.room_d / 2, s.room_h / 2};
    std::mt19937_64 rng(s.seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < s.n_objects; ++i) {
        Object obj;
        obj.is_sphere = (i % 2 == 0);
        obj.label = obj.is_sphere ? kLabelSphere : kLabelBox;
        const double size = 0.16 + 0.10 * u(rng);
        const double ang = 2 * M_PI * u(rng);
        const double rad = 0.22 * std::min(sc->room_half.x, sc->room_half.y) * u(rng);
        obj.center = {rad * std::cos(ang), rad * std::sin(ang), -sc->room_half.z + size + 0.05};
        obj.half = obj.is_sphere ? V3{size, size, size} : V3{size, 0.8 * size, 1.2 * size};
        sc->objects.push_back(obj);
    }
    *out = sc;
    return SVR_OK;
}

void svr_scene_destroy(svr_scene* s) { delete s; }

int svr_scene_camera(const svr_scene* s, int32_t frame, svr_camera* out) {
    *out = s->camera(frame);
    return SVR_OK;
}

int svr_scene_depth(const svr_scene* s, const svr_camera* cams, uint32_t n, float* depth_out,
                    int32_t threads) {
    if (n == 0) return SVR_OK;
    const int W = cams[0].width, H = cams[0].height;
    const uint64_t rows = static_cast<uint64_t>(n) * H;
    bool escaped = false;
    parallel_range(rows, n_threads(threads), [&](uint64_t b, uint64_t e) {
        for (uint64_t r = b; r < e; ++r) {
            const uint32_t f = static_cast<uint32_t>(r / H);
            const int y = static_cast<int>(r % H);
            for (int x = 0; x < W; ++x) {
                double dep = 0.0;
                if (!s->raycast(cams[f], x, y, dep)) escaped = true;
                depth_out[r * W + x] = static_cast<float>(dep);
            }
        }
    });
    if (escaped) {
        svr_internal::set_error("synthetic: ray escaped the room");
        return SVR_ERR_DATA;
    }
    return SVR_OK;
}

int svr_scene_frames(const svr_scene* s, const svr_camera* cams, uint32_t n, float* depth_out,
                     float* rgb_out, float* semantic_out, int32_t C, float* normal_out, int32_t threads) {
    if (n == 0) return SVR_OK;
    if (semantic_out && C < 4) {
        svr_internal::set_error("synthetic: semantic images need label_channels >= 4");
        return SVR_ERR_CONFIG;
    }
    const int W = cams[0].width, H = cams[0].height;
    const uint64_t rows = static_cast<uint64_t>(n) * H;
    bool escaped = false;
    parallel_range(rows, n_threads(threads), [&](uint64_t b, uint64_t e) {
        for (uint64_t r = b; r < e; ++r) {
            const uint32_t f = static_cast<uint32_t>(r / H);
            const int y = static_cast<int>(r % H);
            for (int x = 0; x < W; ++x) {
                double dep = 0.0;
                int lab = 0;
                V3 p{0, 0, 0}, nw{0, 0, 1};
                if (!s->raycast(cams[f], x, y, dep, &lab, &p, &nw) || lab < 0) {
                    escaped = true;
                    lab = 0;
                }
                const uint64_t px = r * W + x;
                if (depth_out) depth_out[px] = static_cast<float>(dep);
                if (rgb_out) {  // synthetic.cpp:337-339
                    double c[3];
                    s->color(p, lab, c);
                    for (int k = 0; k < 3; ++k) rgb_out[3 * px + k] = static_cast<float>(c[k]);
                }
                if (normal_out) {  // synthetic.cpp:333-335: camera-frame normal R^T n
                    const svr_camera& c = cams[f];
                    for (int k = 0; k < 3; ++k)
                        normal_out[3 * px + k] =
                            static_cast<float>((c.R[k] * nw.x + c.R[3 + k] * nw.y) + c.R[6 + k] * nw.z);
                }
                if (semantic_out)  // synthetic.cpp:336: one-hot
                    for (int k = 0; k < C; ++k) semantic_out[C * px + k] = (k == lab) ? 1.0f : 0.0f;
            }
        }
    });
    if (escaped) {
        svr_internal::set_error("synthetic: ray escaped the room");
        return SVR_ERR_DATA;
    }
    return SVR_OK;
}

int svr_scene_sdf(const svr_scene* s, const double* x, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = s->sdf({x[3 * i], x[3 * i + 1], x[3 * i + 2]});
    return SVR_OK;
}

int svr_scene_fill_payload(const svr_scene* s, double h, int32_t B, int32_t C, double trunc,
                           const int32_t* coords, uint64_t nblocks, float* sdf, float* weight,
                           float* rgb, float* logits, int32_t threads) {
    const uint64_t V = static_cast<uint64_t>(B) * B * B;
    parallel_range(nblocks, n_threads(threads), [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) {
            for (uint64_t v = 0; v < V; ++v) {
                const int lx = static_cast<int>(v % B), ly = static_cast<int>((v / B) % B),
                          lz = static_cast<int>(v / (B * B));
                // voxel_to_world (grid.hpp:124-126): v * h
                const V3 x{static_cast<double>(coords[3 * i] * B + lx) * h,
                           static_cast<double>(coords[3 * i + 1] * B + ly) * h,
                           static_cast<double>(coords[3 * i + 2] * B + lz) * h};
                const uint64_t o = i * V + v;
                if (sdf) sdf[o] = static_cast<float>(std::min(std::max(s->sdf(x), -trunc), trunc));
                if (weight) weight[o] = 1.0f;
                if (rgb || logits) {
                    const int lab = s->label(x);
                    if (rgb) {
                        double c[3];
                        s->color(x, lab, c);
                        for (int k = 0; k < 3; ++k) rgb[3 * o + k] = static_cast<float>(c[k]);
                    }
                    if (logits)
                        for (int k = 0; k < C; ++k) logits[C * o + k] = (k == lab) ? 1.0f : 0.0f;
                }
            }
        }
    });
    return SVR_OK;
}

// Camera::ray_direction (camera.cpp:27-30)
static void ray_dir(const svr_camera& cam, double px, double py, double* d) {
    const double dc[3] = {(px - cam.cx) / cam.fx, (py - cam.cy) / cam.fy, 1.0};
    V3 r;
    double rr[3];
    for (int i = 0; i < 3; ++i)
        rr[i] = (cam.R[3 * i] * dc[0] + cam.R[3 * i + 1] * dc[1]) + cam.R[3 * i + 2] * dc[2];
    r = normalized(V3{rr[0], rr[1], rr[2]});
    d[0] = r.x, d[1] = r.y, d[2] = r.z;
}

int svr_scene_rays(const svr_scene* s, uint32_t n_poses, uint32_t rays_per_pose, uint64_t seed,
                   double* o, double* d) {
    std::mt19937_64 rng(seed);
    const uint64_t npix = static_cast<uint64_t>(s->spec.width) * s->spec.height;
    std::uniform_int_distribution<uint64_t> pick(0, npix - 1);
    uint64_t i = 0;
    for (uint32_t p = 0; p < n_poses; ++p) {
        const svr_camera cam = s->camera(static_cast<int>(p));
        for (uint32_t r = 0; r < rays_per_pose; ++r, ++i) {
            const uint64_t px = pick(rng);
            const double x = static_cast<double>(px % s->spec.width);
            const double y = static_cast<double>(px / s->spec.width);
            for (int a = 0; a < 3; ++a) o[3 * i + a] = cam.t[a];
            ray_dir(cam, x, y, d + 3 * i);
        }
    }
    return SVR_OK;
}

int svr_scene_image_rays(const svr_scene* s, int32_t frame, double* o, double* d) {
    const svr_camera cam = s->camera(frame);
    uint64_t i = 0;
    for (int y = 0; y < s->spec.height; ++y)
        for (int x = 0; x < s->spec.width; ++x, ++i) {
            for (int a = 0; a < 3; ++a) o[3 * i + a] = cam.t[a];
            ray_dir(cam, x, y, d + 3 * i);
        }
    return SVR_OK;
}

int svr_uniform_floats(uint64_t n, uint64_t seed, float lo, float hi, float* out) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> u(lo, hi);
    for (uint64_t i = 0; i < n; ++i) out[i] = u(rng);
    return SVR_OK;
}

}  // extern "C"
