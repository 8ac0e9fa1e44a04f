// ref_shim.cpp — extern "C" wrapper around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against the reference's
// own headers where they lie (/root/reference/proj/include, never copied) into
// oracle/_ref/libsdtw_ref.so.  Used (a) to pin the C restatement
// oracle/sdtw_oracle.c and to generate tests/golden/ fixtures, and (b) as the
// reference CPU implementation that bench.py times for its cpu_baseline leg
// and for `--impl reference`.  No product code links it.
//
// Every entry point calls the reference's own public API:
//   sdtw_with_gradients  backward.hpp:276-304
//   forward              forward.hpp:43-81
//   backward_log/linear  backward.hpp:183-203
//   barycenter_objective barycenter.hpp:60-86
//   solve_barycenter     barycenter.hpp:159-211
//   run_bench_row        bench.hpp:52-107
//   generate_dataset     datasets.hpp:21-80
#include <cstring>
#include <exception>
#include <random>
#include <vector>

#include "softdtw/softdtw.hpp"

using namespace softdtw;

namespace {

enum : int {
    REF_OK = 0,
    REF_EINVAL = 1,
    REF_ENOMEM = 2,
    REF_EUNREACHABLE = 3,
    REF_EINCOMPLETE = 4,
    REF_EOTHER = 5,
};

template <class Fn>
int guarded(Fn &&fn)
{
    try {
        fn();
        return REF_OK;
    } catch (const ValidationError &) {
        return REF_EINVAL;
    } catch (const OutOfMemoryError &) {
        return REF_ENOMEM;
    } catch (const UnreachableEndError &) {
        return REF_EUNREACHABLE;
    } catch (const IncompleteTableError &) {
        return REF_EINCOMPLETE;
    } catch (...) {
        return REF_EOTHER;
    }
}

SdtwConfig make_cfg(double gamma, size_t bw, int fused, int log_space)
{
    SdtwConfig cfg;
    cfg.gamma = gamma;
    cfg.bandwidth = bw;
    cfg.cost_mode = fused ? CostMode::fused : CostMode::unfused;
    cfg.backward_space =
        log_space ? BackwardSpace::log_space : BackwardSpace::linear;
    return cfg;
}

template <class T>
int with_gradients(const T *x, const T *y, size_t B, size_t N, size_t M,
                   size_t D, double gamma, size_t bw, int fused, int log_space,
                   unsigned threads, T *loss, T *gx, T *gy)
{
    return guarded([&] {
        SeriesBatch<T> xs(std::vector<T>(x, x + B * N * D), B, N, D);
        SeriesBatch<T> ys(std::vector<T>(y, y + B * M * D), B, M, D);
        auto out = sdtw_with_gradients(xs, ys, make_cfg(gamma, bw, fused,
                                                        log_space),
                                       threads);
        std::memcpy(loss, out.loss.data(), sizeof(T) * B);
        std::memcpy(gx, out.grads.grad_x.data(), sizeof(T) * B * N * D);
        std::memcpy(gy, out.grads.grad_y.data(), sizeof(T) * B * M * D);
    });
}

template <class T>
int forward_backward_tables(const T *x, const T *y, size_t B, size_t N,
                            size_t M, size_t D, double gamma, size_t bw,
                            int fused, int log_space, unsigned threads,
                            T *loss, T *R_out, T *costs_out, T *E_out)
{
    return guarded([&] {
        SeriesBatch<T> xs(std::vector<T>(x, x + B * N * D), B, N, D);
        SeriesBatch<T> ys(std::vector<T>(y, y + B * M * D), B, M, D);
        SdtwConfig cfg = make_cfg(gamma, bw, fused, log_space);
        auto fwd = forward(xs, ys, cfg, threads);
        std::memcpy(loss, fwd.loss.data(), sizeof(T) * B);
        const size_t cells = B * (N + 2) * (M + 2);
        if (R_out) std::memcpy(R_out, fwd.table.buffer().data(), sizeof(T) * cells);
        if (costs_out && fwd.costs)
            std::memcpy(costs_out, fwd.costs->buffer().data(),
                        sizeof(T) * B * N * M);
        if (!E_out) return;
        GradTableBatch<T> e;
        if (fwd.costs) {
            MaterializedCosts<T> cost{&*fwd.costs};
            e = log_space ? backward_log(std::move(fwd.table), cost, cfg, threads)
                          : backward_linear(std::move(fwd.table), cost, cfg,
                                            threads);
        } else {
            FusedCosts<T> cost{&xs, &ys, &fwd.cache};
            e = log_space ? backward_log(std::move(fwd.table), cost, cfg, threads)
                          : backward_linear(std::move(fwd.table), cost, cfg,
                                            threads);
        }
        for (size_t b = 0; b < B; ++b)
            for (size_t i = 0; i < N + 2; ++i)
                for (size_t j = 0; j < M + 2; ++j)
                    E_out[(b * (N + 2) + i) * (M + 2) + j] = e.at(b, i, j);
    });
}

template <class T>
int bary_objective(const T *z, size_t Lz, const T *members, size_t K,
                   size_t L, size_t D, double gamma, size_t bw,
                   const double *weights, unsigned threads, double *value,
                   T *grad)
{
    return guarded([&] {
        BarycenterProblem<T> prob;
        prob.members.reserve(K);
        for (size_t k = 0; k < K; ++k)
            prob.members.emplace_back(
                std::vector<T>(members + k * L * D, members + (k + 1) * L * D),
                1, L, D);
        prob.target_length = Lz;
        prob.gamma = gamma;
        prob.bandwidth = bw;
        if (weights) prob.weights.assign(weights, weights + K);
        prob.threads = threads;
        SeriesBatch<T> zs(std::vector<T>(z, z + Lz * D), 1, Lz, D);
        auto [v, g] = barycenter_objective(zs, prob);
        *value = v;
        std::memcpy(grad, g.data(), sizeof(T) * Lz * D);
    });
}

}  // namespace

extern "C" {

int ref_sdtw_with_gradients_f64(const double *x, const double *y, size_t B,
                                size_t N, size_t M, size_t D, double gamma,
                                size_t bw, int fused, int log_space,
                                unsigned threads, double *loss, double *gx,
                                double *gy)
{
    return with_gradients(x, y, B, N, M, D, gamma, bw, fused, log_space,
                          threads, loss, gx, gy);
}

int ref_sdtw_with_gradients_f32(const float *x, const float *y, size_t B,
                                size_t N, size_t M, size_t D, double gamma,
                                size_t bw, int fused, int log_space,
                                unsigned threads, float *loss, float *gx,
                                float *gy)
{
    return with_gradients(x, y, B, N, M, D, gamma, bw, fused, log_space,
                          threads, loss, gx, gy);
}

int ref_tables_f64(const double *x, const double *y, size_t B, size_t N,
                   size_t M, size_t D, double gamma, size_t bw, int fused,
                   int log_space, unsigned threads, double *loss,
                   double *R_out, double *costs_out, double *E_out)
{
    return forward_backward_tables(x, y, B, N, M, D, gamma, bw, fused,
                                   log_space, threads, loss, R_out, costs_out,
                                   E_out);
}

int ref_tables_f32(const float *x, const float *y, size_t B, size_t N,
                   size_t M, size_t D, double gamma, size_t bw, int fused,
                   int log_space, unsigned threads, float *loss, float *R_out,
                   float *costs_out, float *E_out)
{
    return forward_backward_tables(x, y, B, N, M, D, gamma, bw, fused,
                                   log_space, threads, loss, R_out, costs_out,
                                   E_out);
}

int ref_barycenter_objective_f64(const double *z, size_t Lz,
                                 const double *members, size_t K, size_t L,
                                 size_t D, double gamma, size_t bw,
                                 const double *weights, unsigned threads,
                                 double *value, double *grad)
{
    return bary_objective(z, Lz, members, K, L, D, gamma, bw, weights, threads,
                          value, grad);
}

int ref_barycenter_objective_f32(const float *z, size_t Lz,
                                 const float *members, size_t K, size_t L,
                                 size_t D, double gamma, size_t bw,
                                 const double *weights, unsigned threads,
                                 double *value, float *grad)
{
    return bary_objective(z, Lz, members, K, L, D, gamma, bw, weights, threads,
                          value, grad);
}

// solve_barycenter (barycenter.hpp:159-211), euclidean_mean init.
// objective_out holds max_iters+1 doubles; returns iterations run in *iters.
int ref_solve_barycenter_f64(const double *members, size_t K, size_t L,
                             size_t D, size_t Lz, double gamma, size_t bw,
                             double lr, size_t max_iters, double tol,
                             unsigned threads, double *objective_out,
                             size_t *iters, int *converged, double *final_z)
{
    return guarded([&] {
        BarycenterProblem<double> prob;
        for (size_t k = 0; k < K; ++k)
            prob.members.emplace_back(
                std::vector<double>(members + k * L * D,
                                    members + (k + 1) * L * D),
                1, L, D);
        prob.target_length = Lz;
        prob.gamma = gamma;
        prob.bandwidth = bw;
        prob.threads = threads;
        AdamOptions opts;
        opts.lr = lr;
        opts.max_iters = max_iters;
        opts.tol = tol;
        auto trace = solve_barycenter(prob, BarycenterInit::euclidean_mean,
                                      opts);
        std::memcpy(objective_out, trace.objective_per_iteration.data(),
                    sizeof(double) * trace.objective_per_iteration.size());
        *iters = trace.iterations_run;
        *converged = trace.converged ? 1 : 0;
        std::memcpy(final_z, trace.final_z.raw().data(),
                    sizeof(double) * Lz * D);
    });
}

// run_bench_row (bench.hpp:52-107): the reference's own timer.
int ref_run_bench_row(size_t B, size_t L, size_t D, double gamma, int fused,
                      int log_space, size_t repeats, size_t warmup,
                      unsigned threads, unsigned long long seed,
                      double *mean_ms, double *std_ms, size_t *peak_bytes,
                      float *loss0)
{
    BenchConfigRow row;
    row.batch = B;
    row.length = L;
    row.feature_dim = D;
    row.gamma = gamma;
    row.cost_mode = fused ? CostMode::fused : CostMode::unfused;
    row.backward_space =
        log_space ? BackwardSpace::log_space : BackwardSpace::linear;
    row.repeats = repeats;
    row.warmup = warmup;
    BenchResultRow r;
    int rc = guarded([&] { r = run_bench_row(row, threads, seed); });
    if (rc != REF_OK) return rc;
    if (!r.ok) return REF_EOTHER;
    *mean_ms = r.mean_runtime_ms;
    *std_ms = r.std_runtime_ms;
    *peak_bytes = r.peak_ledger_bytes;
    *loss0 = r.loss0;
    return REF_OK;
}

// The bench generator spec (bench.hpp:61-66): N(0,1) fp32 from
// mt19937_64(seed), all of x then all of y.
void ref_bench_inputs(size_t B, size_t L, size_t D, unsigned long long seed,
                      float *x, float *y)
{
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, 1.0f);
    const size_t count = B * L * D;
    for (size_t i = 0; i < count; ++i) x[i] = dist(rng);
    for (size_t i = 0; i < count; ++i) y[i] = dist(rng);
}

// generate_dataset (datasets.hpp:21-80); out holds count*length*dim doubles.
int ref_generate_dataset(int kind, size_t count, size_t length, size_t dim,
                         double noise, unsigned long long seed, double *out)
{
    return guarded([&] {
        auto ds = generate_dataset(static_cast<DatasetKind>(kind), count,
                                   length, dim, noise, seed);
        for (size_t k = 0; k < count; ++k)
            std::memcpy(out + k * length * dim, ds[k].raw().data(),
                        sizeof(double) * length * dim);
    });
}

unsigned ref_hardware_threads() { return resolve_threads(0); }

}  // extern "C"
