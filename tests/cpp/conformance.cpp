// C++ drop-in conformance: the reference's API (namespace softdtw) served by
// the B200 engine (softdtw::b200, include/softdtw_b200/dropin.hpp) against
// the unmodified reference (T = double) on the same inputs.  Built by
// tests/cpp/Makefile against /root/reference/proj/include (never copied);
// run on a GPU by tests/test_cpp_dropin.py.
#include <softdtw/softdtw.hpp>

#include <cmath>
#include <cstdio>
#include <random>

#include "softdtw_b200/dropin.hpp"

using namespace softdtw;

static int fails = 0, checks = 0;
#define CHECK(cond, ...)                          \
    do {                                          \
        ++checks;                                 \
        if (!(cond)) {                            \
            ++fails;                              \
            std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);             \
            std::printf("\n");                    \
        }                                         \
    } while (0)

template <class T>
static SeriesBatch<T> randn(std::size_t B, std::size_t L, std::size_t D, unsigned seed)
{
    std::mt19937_64 g(seed);
    std::normal_distribution<double> n(0.0, 1.0);
    std::vector<T> v(B * L * D);
    for (auto &e : v) e = static_cast<T>(static_cast<float>(n(g)));
    return SeriesBatch<T>(std::move(v), B, L, D);
}

template <class A, class B>
static SeriesBatch<A> cast(const SeriesBatch<B> &s)
{
    std::vector<A> v(s.raw().begin(), s.raw().end());
    return SeriesBatch<A>(std::move(v), s.batch_size(), s.length(), s.feature_dim());
}

static double max_err(const std::vector<float> &a, const std::vector<double> &r)
{
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i)
        m = std::max(m, std::fabs((double)a[i] - r[i]) / std::max(1.0, std::fabs(r[i])));
    return m;
}

int main()
{
    // 1. sdtw_with_gradients: fp32 engine vs fp64 reference (both cost modes)
    for (double gamma : {1.0, 0.1, 0.01}) {
        for (bool fused : {false, true}) {
            auto xf = randn<float>(3, 90, 12, 7), yf = randn<float>(3, 110, 12, 8);
            SdtwConfig cfg;
            cfg.gamma = gamma;
            cfg.cost_mode = fused ? CostMode::fused : CostMode::unfused;
            auto ref = sdtw_with_gradients(cast<double>(xf), cast<double>(yf), cfg);
            AllocationLedger ledger;
            auto got = b200::sdtw_with_gradients(xf, yf, cfg, 0, &ledger);
            double le = 0;
            for (int b = 0; b < 3; ++b)
                le = std::max(le, std::fabs(got.loss[b] - ref.loss[b]) / std::max(1.0, std::fabs(ref.loss[b])));
            CHECK(le <= 1e-5, "loss rel err %.3g (gamma %g fused %d)", le, gamma, fused);
            const double gx = max_err(got.grads.grad_x, ref.grads.grad_x);
            const double gy = max_err(got.grads.grad_y, ref.grads.grad_y);
            CHECK(gx <= 1e-3 && gy <= 1e-3, "grad err %.3g %.3g (gamma %g fused %d)", gx, gy, gamma, fused);
            CHECK(ledger.peak_bytes > 0 && ledger.live_bytes == 0, "ledger peak %zu live %zu", ledger.peak_bytes,
                  ledger.live_bytes);
        }
    }
    // 2. the reference's exception taxonomy survives the drop-in
    {
        auto x = randn<float>(2, 20, 3, 1), y = randn<float>(2, 20, 4, 2);
        bool caught = false;
        try {
            b200::sdtw_with_gradients(x, y, SdtwConfig{});
        } catch (const ValidationError &) {
            caught = true;
        }
        CHECK(caught, "feature-dim mismatch -> ValidationError");
    }
    {
        auto x = randn<float>(1, 10, 3, 3), y = randn<float>(1, 40, 3, 4);
        SdtwConfig cfg;
        cfg.bandwidth = 2;
        bool caught = false;
        try {
            b200::sdtw_with_gradients(x, y, cfg);
        } catch (const ValidationError &) {
            caught = true;
        }
        CHECK(caught, "band narrower than |N - M| -> ValidationError (validate_config, types.hpp:230-243)");
    }
    {
        auto x = randn<float>(4, 200, 16, 5), y = randn<float>(4, 200, 16, 6);
        AllocationLedger ledger;
        ledger.limit_bytes = 4096;
        bool caught = false;
        try {
            b200::sdtw_with_gradients(x, y, SdtwConfig{}, 0, &ledger);
        } catch (const OutOfMemoryError &e) {
            caught = e.requested_bytes() > 0;
        }
        CHECK(caught, "ledger limit -> OutOfMemoryError");
    }
    // 3. barycenter_objective (unfused, log space, weights)
    {
        BarycenterProblem<float> pf;
        BarycenterProblem<double> pd;
        for (unsigned k = 0; k < 5; ++k) {
            auto m = randn<float>(1, 40, 4, 100 + k);
            pd.members.push_back(cast<double>(m));
            pf.members.push_back(std::move(m));
        }
        pf.weights = pd.weights = {0.5, 1.0, 0.25, 2.0, 1.0};
        pf.gamma = pd.gamma = 0.5;
        pf.target_length = pd.target_length = 30;
        auto z = randn<float>(1, 30, 4, 99);
        auto [vr, gr] = barycenter_objective(cast<double>(z), pd);
        auto [vg, gg] = b200::barycenter_objective(z, pf);
        CHECK(std::fabs(vg - vr) <= 1e-5 * std::max(1.0, std::fabs(vr)), "barycenter value %.9g vs %.9g", vg, vr);
        CHECK(max_err(gg, gr) <= 1e-3, "barycenter grad err %.3g", max_err(gg, gr));
    }
    std::printf("%s %d/%d checks\n", fails ? "FAIL" : "PASS", checks - fails, checks);
    return fails ? 1 : 0;
}
