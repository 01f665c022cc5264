// The reference's grid test scenarios (proj/tests/test_grid.cpp) re-run against the B200
// library through the C++ host mirror include/svr.hpp -- same call shapes, same expected
// answers.  Built and executed by tests/test_gpu_cpp.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "svr.hpp"

using namespace svr::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                \
    do {                                                                           \
        ++g_checks;                                                                \
        if (!(cond)) {                                                             \
            ++g_fail;                                                              \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                          \
    } while (0)

static void fill_all(SparseDenseGrid& g, float (*f)(double, double, double)) {
    const auto coords = g.coords();
    const std::size_t n = coords.size();
    std::vector<float> sdf(n * 512), w(n * 512, 1.0f), rgb(n * 512 * 3, 0.5f),
        lg(n * 512 * g.label_channels(), 0.0f);
    const double h = g.voxel_size();
    for (std::size_t i = 0; i < n; ++i)
        for (int v = 0; v < 512; ++v) {
            const int lx = v % 8, ly = (v / 8) % 8, lz = v / 64;
            sdf[i * 512 + v] = f((coords[i].x * 8 + lx) * h, (coords[i].y * 8 + ly) * h,
                                 (coords[i].z * 8 + lz) * h);
        }
    g.set_payload(0, static_cast<std::uint32_t>(n), sdf.data(), w.data(), rgb.data(), lg.data());
}

int main() {
    {  // test_grid.cpp:55  single point, no dilation
        SparseDenseGrid g(0.015, 8, 2);
        const double p[3] = {0.05, 0.05, 0.05};
        const auto r = allocate_for_points(g, p, 1, 0);
        CHECK(r.blocks_added == 1);
        CHECK(g.block_count() == 1);
    }
    {  // test_grid.cpp:63  R = 2 -> 5^3 ball
        SparseDenseGrid g(0.015, 8, 2);
        const double p[3] = {0.06, 0.06, 0.06};
        allocate_for_points(g, p, 1, 2);
        CHECK(g.block_count() == 125);
        for (int dz = -2; dz <= 2; ++dz)
            for (int dy = -2; dy <= 2; ++dy)
                for (int dx = -2; dx <= 2; ++dx)
                    CHECK(g.find_block(BlockCoord{dx, dy, dz}) != SparseDenseGrid::kInvalidBlock);
    }
    {  // test_grid.cpp:76  idempotent
        SparseDenseGrid g(0.015, 8, 2);
        std::mt19937_64 rng(1);
        std::uniform_real_distribution<double> u(-0.5, 0.5);
        std::vector<double> pts;
        for (int i = 0; i < 600; ++i) pts.push_back(u(rng));
        allocate_for_points(g, pts.data(), 200, 1);
        const std::size_t n = g.block_count();
        const auto again = allocate_for_points(g, pts.data(), 200, 1);
        CHECK(again.blocks_added == 0);
        CHECK(g.block_count() == n);
    }
    {  // test_grid.cpp:89  capacity exceeded reports the unallocated count
        SparseDenseGrid g(0.015, 8, 2, 10);
        std::vector<double> pts;
        for (int i = 0; i < 20; ++i) pts.insert(pts.end(), {0.13 * i, 0.0, 0.0});
        bool thrown = false;
        try {
            allocate_for_points(g, pts.data(), 20, 0);
        } catch (const CapacityError& e) {
            thrown = true;
            CHECK(e.unallocated_blocks == 10);
        }
        CHECK(thrown);
        CHECK(g.block_count() == 10);
    }
    {  // test_grid.cpp:177  zero weights -> invalid, value 0
        SparseDenseGrid g(0.015, 8, 2);
        const double p[3] = {0.05, 0.05, 0.05};
        allocate_for_points(g, p, 1, 0);
        double sdf = 1.0;
        CHECK(!g.query_sdf(p, sdf));
        CHECK(sdf == 0.0);
    }
    {  // test_grid.cpp:207  linear fields are reproduced, including the gradient
        SparseDenseGrid g(1.0 / 64.0, 8, 2);
        const double pts[6] = {0.05, 0.05, 0.05, -0.05, 0.02, 0.08};
        allocate_for_points(g, pts, 2, 1);
        fill_all(g, [](double x, double y, double z) { return float(0.5 * x + 0.25 * y - 0.75 * z + 0.125); });
        std::mt19937_64 rng(123);
        std::uniform_real_distribution<double> u(-0.05, 0.1);
        int checked = 0;
        for (int i = 0; i < 300; ++i) {
            const double x[3] = {u(rng), u(rng), u(rng)};
            double s, gr[3];
            if (!g.query_sdf_with_gradient(x, s, gr)) continue;
            ++checked;
            CHECK(std::abs(s - (0.5 * x[0] + 0.25 * x[1] - 0.75 * x[2] + 0.125)) < 1e-6);  // f32 payload
            CHECK(std::abs(gr[0] - 0.5) < 1e-4 && std::abs(gr[1] - 0.25) < 1e-4 && std::abs(gr[2] + 0.75) < 1e-4);
        }
        CHECK(checked > 100);
    }
    {  // test_grid.cpp:274  miss -> empty sample list
        SparseDenseGrid g(0.015, 8, 2);
        const double p[3] = {0.05, 0.05, 0.05};
        allocate_for_points(g, p, 1, 0);
        const double o[3] = {5.0, 5.0, 5.0}, d[3] = {1.0, 0.0, 0.0};
        std::uint32_t count = 7;
        std::vector<double> t(1000);
        g.march(o, d, 1, 0.01, 1000, &count, t.data(), nullptr);
        CHECK(count == 0);
    }
    {  // test_grid.cpp:283  axis-aligned ray through one block: 11..13 samples
        SparseDenseGrid g(0.015, 8, 2);
        const double p[3] = {0.06, 0.06, 0.06};
        allocate_for_points(g, p, 1, 0);
        const double o[3] = {-1.0, 0.06, 0.06}, d[3] = {1.0, 0.0, 0.0};
        std::uint32_t count = 0;
        std::vector<double> t(1000);
        g.march(o, d, 1, 0.01, 1000, &count, t.data(), nullptr);
        CHECK(count >= 11 && count <= 13);
        for (std::uint32_t k = 1; k < count; ++k) CHECK(t[k] > t[k - 1]);
    }
    {  // renderer: opaque wall -> depth at the first sample, weights sum to one
        SparseDenseGrid g(0.02, 8, 1);
        const double p[3] = {0.08, 0.08, 0.08};
        allocate_for_points(g, p, 1, 0);
        fill_all(g, [](double, double, double) { return -1.0f; });
        const double o[3] = {-1.0, 0.08, 0.08}, d[3] = {1.0, 0.0, 0.0};
        float rgb[3], depth, normal[3], wsum;
        std::uint32_t ns = 0;
        g.render_forward(o, d, 1, 0.01, 64, 1e-4, RenderOutputs{rgb, &depth, normal, &wsum, &ns});
        CHECK(ns > 10);
        CHECK(std::abs(wsum - 1.0f) < 1e-6f);
        CHECK(std::abs(rgb[0] - 0.5f) < 1e-6f);
        const float dC[3] = {1, 0, 0}, dD = 0, dN[3] = {0, 0, 0};
        g.zero_grad();
        g.render_backward(dC, &dD, dN);
        CHECK(g.active_blocks().size() == 1);
        // two replicas, each rendering the same ray: reduce_grads sums them into both
        SparseDenseGrid g2(0.02, 8, 1);
        allocate_for_points(g2, p, 1, 0);
        fill_all(g2, [](double, double, double) { return -1.0f; });
        g2.render_forward(o, d, 1, 0.01, 64, 1e-4, RenderOutputs{rgb, &depth, normal, &wsum, &ns});
        g2.zero_grad();
        g2.render_backward(dC, &dD, dN);
        std::vector<float> s1(512), r1(1536), s2(512), r2(1536);
        g.grads(s1.data(), r1.data());
        reduce_grads({&g, &g2}, SVR_REDUCE_PEER);
        g.grads(s2.data(), r2.data());
        bool doubled = true, nonzero = false;
        for (int i = 0; i < 1536; ++i) doubled &= r2[i] == 2.0f * r1[i], nonzero |= r1[i] != 0.0f;
        CHECK(doubled && nonzero);
        g2.grads(s1.data(), r1.data());
        CHECK(s1 == s2 && r1 == r2);
        CHECK(g2.active_blocks().size() == 1);
    }
    {  // SDGV round trip (test_grid.cpp:373)
        SparseDenseGrid g(0.0175, 8, 3);
        const double p[6] = {0.1, 0.2, -0.3, -0.2, 0.1, 0.3};
        allocate_for_points(g, p, 2, 0);
        fill_all(g, [](double x, double y, double z) { return float(x - 2 * y + z); });
        save_grid(g, "/tmp/svr_hpp_test.sdgv");
        SparseDenseGrid l = load_grid("/tmp/svr_hpp_test.sdgv");
        CHECK(l.block_count() == g.block_count());
        CHECK(l.voxel_size() == g.voxel_size());
        CHECK(l.label_channels() == 3);
    }
    {  // marching cubes on an analytic sphere (test_meshing.cpp:44-55) + export_ply
        SparseDenseGrid g(0.015, 8, 2);
        std::vector<double> shell;
        const int n = 6000;
        for (int i = 0; i < n; ++i) {  // fibonacci_sphere (test_meshing.cpp:18-30), r = 0.5
            const double z = 1.0 - 2.0 * (i + 0.5) / n, rad = std::sqrt(1.0 - z * z);
            const double th = M_PI * (3.0 - std::sqrt(5.0)) * i;
            shell.insert(shell.end(), {0.5 * rad * std::cos(th), 0.5 * rad * std::sin(th), 0.5 * z});
        }
        allocate_for_points(g, shell.data(), n, 1);
        fill_all(g, [](double x, double y, double z) { return float(std::sqrt(x * x + y * y + z * z) - 0.5); });
        const Mesh m = marching_cubes(g, 0.0);
        CHECK(m.vertex_count() > 1000 && m.triangle_count() > 2000);
        bool near = true;
        for (std::size_t i = 0; i < m.vertex_count(); ++i) {
            const double* v = &m.vertices[3 * i];
            near &= std::abs(std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) - 0.5) < 0.0075;
        }
        CHECK(near);
        export_ply(g, "/tmp/svr_hpp_test.ply");
        std::FILE* f = std::fopen("/tmp/svr_hpp_test.ply", "rb");
        CHECK(f != nullptr);
        if (f) std::fclose(f);
    }
    {  // ConfigError mirrors grid.cpp:83-85
        bool thrown = false;
        try {
            SparseDenseGrid bad(0.0, 8, 1);
        } catch (const ConfigError&) {
            thrown = true;
        }
        CHECK(thrown);
    }
    std::printf("svr.hpp mirror: %d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
