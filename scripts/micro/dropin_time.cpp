// Where the C++ drop-in's end-to-end time goes at C2 (B=32, L=1024, D=128).
#include <softdtw/softdtw.hpp>
#include <chrono>
#include <cstdio>
#include <cstring>
#include "softdtw_b200/dropin.hpp"
using namespace softdtw;
using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }
int main() {
    const size_t B = 32, L = 1024, D = 128, n = B * L * D;
    std::vector<float> xs(n), ys(n);
    for (size_t i = 0; i < n; ++i) { xs[i] = float((i * 2654435761u) % 1000) / 500.f - 1.f; ys[i] = float((i * 40503u) % 1000) / 500.f - 1.f; }
    SeriesBatch<float> x(xs, B, L, D), y(ys, B, L, D);
    SdtwConfig cfg; cfg.gamma = 0.1;
    for (int it = 0; it < 3; ++it) b200::sdtw_with_gradients(x, y, cfg);
    auto t0 = clk::now();
    for (int it = 0; it < 5; ++it) b200::sdtw_with_gradients(x, y, cfg);
    auto t1 = clk::now();
    std::printf("drop-in sdtw_with_gradients: %.2f ms\n", ms(t0, t1) / 5);
    auto &ctx = b200::context();
    softdtw_b200::Config c; c.gamma = 0.1;
    t0 = clk::now();
    for (int it = 0; it < 5; ++it) ctx.sdtw_with_gradients(x.raw(), y.raw(), B, L, L, D, c);
    t1 = clk::now();
    std::printf("Context::sdtw_with_gradients (vectors): %.2f ms\n", ms(t0, t1) / 5);
    std::vector<float> l(B), gx(n), gy(n);
    sdtw_config cc = c.c();
    t0 = clk::now();
    for (int it = 0; it < 5; ++it) sdtw_fwd_bwd_f32(ctx.get(), x.raw().data(), y.raw().data(), B, L, L, D, &cc, SDTW_PTR_HOST, l.data(), gx.data(), gy.data());
    t1 = clk::now();
    std::printf("C-ABI, pageable, preallocated outputs: %.2f ms\n", ms(t0, t1) / 5);
    t0 = clk::now();
    for (int it = 0; it < 5; ++it) { std::vector<float> a(n), b2(n); std::memset(a.data(), 1, 4); }
    t1 = clk::now();
    std::printf("two 16.8 MB vector allocations (zero fill + first touch): %.2f ms\n", ms(t0, t1) / 5);
    t0 = clk::now();
    for (int it = 0; it < 5; ++it) std::memcpy(gx.data(), xs.data(), n * 4);
    t1 = clk::now();
    std::printf("host memcpy 16.8 MB: %.2f ms\n", ms(t0, t1) / 5);
    return 0;
}
