// C++ drop-in conformance: the reference's API (namespace softdtw) served by
// the B200 engine (softdtw::b200, include/softdtw_b200/dropin.hpp) against
// the unmodified reference (T = double) on the same inputs.  Built by
// tests/cpp/Makefile against /root/reference/proj/include (never copied);
// run on a GPU by tests/test_cpp_dropin.py.
#include <softdtw/softdtw.hpp>

#include <cmath>
#include <cstdio>
#include <limits>
#include <random>

#include "softdtw_b200/dropin.hpp"
#include "softdtw_b200/bench.hpp"

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
    // 4. forward: loss, padded R table, cost tensor, norm cache (forward.hpp:43-81)
    for (bool fused : {false, true}) {
        auto xd = randn<double>(2, 37, 5, 11), yd = randn<double>(2, 53, 5, 12);
        SdtwConfig cfg;
        cfg.gamma = 0.3;
        cfg.cost_mode = fused ? CostMode::fused : CostMode::unfused;
        auto ref = forward(xd, yd, cfg);
        AllocationLedger ledger;
        auto got = b200::forward(xd, yd, cfg, 0, &ledger);
        double le = 0, te = 0, ce = 0, ne = 0;
        int inf_mismatch = 0;
        for (int b = 0; b < 2; ++b) {
            le = std::max(le, std::fabs(got.loss[b] - ref.loss[b]) / std::max(1.0, std::fabs(ref.loss[b])));
            for (std::size_t i = 0; i <= 38; ++i)
                for (std::size_t j = 0; j <= 54; ++j) {
                    const double r = ref.table.at(b, i, j), g = got.table.at(b, i, j);
                    if (std::isinf(r) || std::isinf(g)) inf_mismatch += !(r == g);
                    else te = std::max(te, std::fabs(g - r) / std::max(1.0, std::fabs(r)));
                }
            for (std::size_t i = 0; i < 37; ++i) ne = std::max(ne, std::fabs(got.cache.x_sq(b, i) - ref.cache.x_sq(b, i)));
            for (std::size_t j = 0; j < 53; ++j) ne = std::max(ne, std::fabs(got.cache.y_sq(b, j) - ref.cache.y_sq(b, j)));
        }
        CHECK(le <= 1e-11 && te <= 1e-11 && inf_mismatch == 0, "forward f64 fused %d: loss %.3g table %.3g inf %d", fused,
              le, te, inf_mismatch);
        CHECK(ne <= 1e-12, "norm cache err %.3g", ne);
        CHECK(got.costs.has_value() == ref.costs.has_value(), "cost tensor presence (fused %d)", fused);
        if (got.costs && ref.costs) {
            for (int b = 0; b < 2; ++b)
                for (std::size_t i = 1; i <= 37; ++i)
                    for (std::size_t j = 1; j <= 53; ++j)
                        ce = std::max(ce, std::fabs(got.costs->at(b, i, j) - ref.costs->at(b, i, j)));
            CHECK(ce <= 1e-11, "cost tensor err %.3g", ce);
        }
        CHECK(ledger.live_bytes > 0, "forward result tracked by the ledger (%zu live)", ledger.live_bytes);
        // fp32 engine against the fp64 reference on the same values
        auto gf = b200::forward(cast<float>(xd), cast<float>(yd), cfg);
        double lf = 0;
        for (int b = 0; b < 2; ++b)
            lf = std::max(lf, std::fabs(gf.loss[b] - ref.loss[b]) / std::max(1.0, std::fabs(ref.loss[b])));
        CHECK(lf <= 1e-5, "forward f32 loss err %.3g (fused %d)", lf, fused);
    }
    // 5. standalone backward_log / backward_linear from a forward table, both
    //    cost accessors, and input_gradients (backward.hpp:183-266)
    for (bool linear : {false, true}) {
        for (bool fused : {false, true}) {
            auto xd = randn<double>(2, 41, 4, 21), yd = randn<double>(2, 29, 4, 22);
            SdtwConfig cfg;
            cfg.gamma = 0.7;
            cfg.cost_mode = fused ? CostMode::fused : CostMode::unfused;
            cfg.backward_space = linear ? BackwardSpace::linear : BackwardSpace::log_space;
            auto rf = forward(xd, yd, cfg);
            auto gf = b200::forward(xd, yd, cfg);
            GradTableBatch<double> re, ge;
            if (fused) {
                FusedCosts<double> rc{&xd, &yd, &rf.cache}, gc{&xd, &yd, &gf.cache};
                re = linear ? backward_linear(std::move(rf.table), rc, cfg) : backward_log(std::move(rf.table), rc, cfg);
                ge = linear ? b200::backward_linear(std::move(gf.table), gc, cfg)
                            : b200::backward_log(std::move(gf.table), gc, cfg);
            } else {
                MaterializedCosts<double> rc{&*rf.costs}, gc{&*gf.costs};
                re = linear ? backward_linear(std::move(rf.table), rc, cfg) : backward_log(std::move(rf.table), rc, cfg);
                ge = linear ? b200::backward_linear(std::move(gf.table), gc, cfg)
                            : b200::backward_log(std::move(gf.table), gc, cfg);
            }
            double ee = 0;
            for (int b = 0; b < 2; ++b)
                for (std::size_t i = 0; i <= 42; ++i)
                    for (std::size_t j = 0; j <= 30; ++j) ee = std::max(ee, std::fabs(ge.at(b, i, j) - re.at(b, i, j)));
            CHECK(ee <= 1e-9 && ge.space() == GradSpace::linear, "backward (linear %d fused %d) E err %.3g", linear,
                  fused, ee);
            auto rg = input_gradients(re, xd, yd);
            auto gg = b200::input_gradients(re, xd, yd);  // the reference's own E table as input
            double ge2 = 0;
            for (std::size_t i = 0; i < rg.grad_x.size(); ++i) ge2 = std::max(ge2, std::fabs(gg.grad_x[i] - rg.grad_x[i]));
            for (std::size_t i = 0; i < rg.grad_y.size(); ++i) ge2 = std::max(ge2, std::fabs(gg.grad_y[i] - rg.grad_y[i]));
            CHECK(ge2 <= 1e-10, "input_gradients err %.3g", ge2);
        }
    }
    // 6. sdtw_with_gradients in linear space (the reference composes
    //    forward -> backward_linear -> input_gradients), fp64
    {
        auto xd = randn<double>(2, 33, 6, 31), yd = randn<double>(2, 47, 6, 32);
        SdtwConfig cfg;
        cfg.backward_space = BackwardSpace::linear;
        auto ref = sdtw_with_gradients(xd, yd, cfg);
        auto got = b200::sdtw_with_gradients(xd, yd, cfg);
        double e = 0;
        for (std::size_t i = 0; i < ref.grads.grad_x.size(); ++i)
            e = std::max(e, std::fabs(got.grads.grad_x[i] - ref.grads.grad_x[i]));
        for (std::size_t i = 0; i < ref.grads.grad_y.size(); ++i)
            e = std::max(e, std::fabs(got.grads.grad_y[i] - ref.grads.grad_y[i]));
        CHECK(e <= 1e-9 && std::fabs(got.loss[0] - ref.loss[0]) <= 1e-9, "linear sdtw_with_gradients err %.3g", e);
    }
    // 7. forward_normalized (forward.hpp:85-102), and its N != M check
    {
        auto xd = randn<double>(3, 40, 5, 41), yd = randn<double>(3, 40, 5, 42);
        SdtwConfig cfg;
        cfg.gamma = 0.2;
        auto ref = forward_normalized(xd, yd, cfg);
        auto got = b200::forward_normalized(xd, yd, cfg);
        double e = 0;
        for (int b = 0; b < 3; ++b) e = std::max(e, std::fabs(got[b] - ref[b]));
        CHECK(e <= 1e-9, "forward_normalized err %.3g", e);
        auto self = b200::forward_normalized(xd, xd, cfg);
        CHECK(std::fabs(self[0]) <= 1e-9, "normalized sdtw(x, x) = %.3g (exactly 0 in the reference)", self[0]);
        bool caught = false;
        try {
            b200::forward_normalized(xd, randn<double>(3, 41, 5, 43), cfg);
        } catch (const ValidationError &) {
            caught = true;
        }
        CHECK(caught, "normalized with N != M -> ValidationError");
    }
    // 8. IncompleteTableError: +inf at a reachable in-band cell of the table
    {
        auto xd = randn<double>(1, 12, 3, 51), yd = randn<double>(1, 12, 3, 52);
        SdtwConfig cfg;
        auto gf = b200::forward(xd, yd, cfg);
        gf.table.at(0, 5, 5) = std::numeric_limits<double>::infinity();
        bool caught = false;
        try {
            b200::backward_log(std::move(gf.table), MaterializedCosts<double>{&*gf.costs}, cfg);
        } catch (const IncompleteTableError &) {
            caught = true;
        }
        CHECK(caught, "backward on a table with +inf at a reachable cell -> IncompleteTableError");
    }
    // 9. barycenter objective: fp64, members of two lengths (the reference
    //    allows ragged members), weights
    {
        BarycenterProblem<double> p;
        for (unsigned k = 0; k < 6; ++k) p.members.push_back(randn<double>(1, k % 2 ? 35 : 28, 3, 200 + k));
        p.weights = {1.0, 0.5, 2.0, 0.0, 1.0, 0.25};
        p.gamma = 0.8;
        p.target_length = 30;
        auto z = randn<double>(1, 30, 3, 299);
        auto [vr, gr] = barycenter_objective(z, p);
        auto [vg, gg] = b200::barycenter_objective(z, p);
        double e = 0;
        for (std::size_t i = 0; i < gr.size(); ++i) e = std::max(e, std::fabs(gg[i] - gr[i]));
        CHECK(std::fabs(vg - vr) <= 1e-9 * std::max(1.0, std::fabs(vr)) && e <= 1e-9,
              "ragged barycenter f64 value %.12g vs %.12g, grad err %.3g", vg, vr, e);
    }
    // 10. solve_barycenter: the Adam loop, trace and best-so-far z (fp64)
    {
        BarycenterProblem<double> p;
        for (unsigned k = 0; k < 4; ++k) p.members.push_back(randn<double>(1, 24, 2, 300 + k));
        p.gamma = 1.0;
        p.target_length = 24;
        AdamOptions o;
        o.max_iters = 6;
        o.tol = 0;
        auto ref = solve_barycenter(p, BarycenterInit::euclidean_mean, o);
        auto got = b200::solve_barycenter(p, BarycenterInit::euclidean_mean, o);
        double te = 0, ze = 0;
        CHECK(ref.objective_per_iteration.size() == got.objective_per_iteration.size() &&
                  ref.iterations_run == got.iterations_run && ref.converged == got.converged,
              "solve_barycenter trace shape");
        for (std::size_t i = 0; i < std::min(ref.objective_per_iteration.size(), got.objective_per_iteration.size()); ++i)
            te = std::max(te, std::fabs(got.objective_per_iteration[i] - ref.objective_per_iteration[i]) /
                                  std::max(1.0, std::fabs(ref.objective_per_iteration[i])));
        for (std::size_t i = 0; i < ref.final_z.raw().size(); ++i)
            ze = std::max(ze, std::fabs(got.final_z.raw()[i] - ref.final_z.raw()[i]));
        CHECK(te <= 1e-9 && ze <= 1e-9, "solve_barycenter objective err %.3g, final z err %.3g", te, ze);
    }
    // 11. run_bench_row (bench.hpp:52-107): same generator and row semantics
    {
        BenchConfigRow row;
        row.batch = 2;
        row.length = 64;
        row.feature_dim = 8;
        row.repeats = 2;
        for (CostMode mode : {CostMode::unfused, CostMode::fused}) {
            row.cost_mode = mode;
            const auto ref = run_bench_row(row, 1);
            const auto got = b200::run_bench_row(row);
            CHECK(got.ok && ref.ok && got.peak_ledger_bytes > 0 && got.mean_runtime_ms > 0,
                  "run_bench_row ok (%s)", got.error.c_str());
            CHECK(std::fabs(got.loss0 - ref.loss0) <= 1e-5f * std::max(1.0f, std::fabs(ref.loss0)),
                  "run_bench_row loss0 %.7g vs reference %.7g", got.loss0, ref.loss0);
            CHECK(bench_csv_row(got).find(",ok") != std::string::npos, "bench CSV row status");
        }
        BenchConfigRow bad = row;
        bad.length = 300;
        const auto oom = b200::run_bench_row(bad, 0, 42, 4096);
        CHECK(!oom.ok && !oom.error.empty(), "ledger limit recorded in the row, not thrown");
    }
    // 12. series files (io.hpp: SDTW v1 binary and CSV) feed the drop-in
    //     unchanged: the reference's own readers produce the SeriesBatch the
    //     engine consumes
    {
        auto x = randn<double>(1, 45, 3, 61), y = randn<double>(1, 52, 3, 62);
        const std::string bx = "/tmp/sdtw_b200_conf_x.bin", cy = "/tmp/sdtw_b200_conf_y.csv";
        write_series_binary(bx, x);
        write_series_csv(cy, y);
        auto xr = read_series<double>(bx), yr = read_series<double>(cy);
        SdtwConfig cfg;
        cfg.gamma = 0.5;
        auto ref = sdtw_with_gradients(xr, yr, cfg);
        auto got = b200::sdtw_with_gradients(xr, yr, cfg);
        double e = std::fabs(got.loss[0] - ref.loss[0]);
        for (std::size_t i = 0; i < ref.grads.grad_x.size(); ++i)
            e = std::max(e, std::fabs(got.grads.grad_x[i] - ref.grads.grad_x[i]));
        CHECK(xr.raw() == x.raw() && e <= 1e-9, "series files through the drop-in: err %.3g", e);
        std::remove(bx.c_str());
        std::remove(cy.c_str());
    }
    std::printf("%s %d/%d checks\n", fails ? "FAIL" : "PASS", checks - fails, checks);
    return fails ? 1 : 0;
}
