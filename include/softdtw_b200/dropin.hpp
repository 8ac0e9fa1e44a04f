// softdtw_b200/dropin.hpp — the reference's own API on the B200 engine.
//
// Include after the reference's <softdtw/softdtw.hpp>.  Provides, in
// namespace softdtw::b200, the reference's signatures on the reference's
// containers, each a drop-in for the function it names:
//   forward<T>(x, y, cfg, threads, ledger)               forward.hpp:43-81
//   forward_normalized<T>(x, y, cfg, threads, ledger)    forward.hpp:85-102
//   backward_log<T, Cost>(table&&, cost, cfg, ...)       backward.hpp:183-190
//   backward_linear<T, Cost>(table&&, cost, cfg, ...)    backward.hpp:196-203
//   input_gradients<T>(e, x, y, threads)                 backward.hpp:208-266
//   sdtw_with_gradients<T>(x, y, cfg, threads, ledger)   backward.hpp:276-304
//   barycenter_objective<T>(z, prob)                     barycenter.hpp:60-86
//   solve_barycenter<T>(prob, init, opts, index, user_z) barycenter.hpp:159-211
// (run_bench_row, bench.hpp:52-107, is in softdtw_b200/bench.hpp)
// Standalone tables (DpTableBatch / GradTableBatch / CostMatrixBatch /
// NormCache) are the reference's own host containers, filled from the
// engine's device results, so callers read them with .at() as before; the
// backward consumes the forward table and reuses its slab (backward.hpp:39).
// Engine errors are rethrown as the reference's exception types
// (types.hpp:17-54), so callers' catch clauses keep working.  `threads` is
// accepted and ignored (the GPU schedule replaces WorkerTeam,
// parallel.hpp:13-71); the ledger, if given, is charged with the engine's
// device peak (AllocationLedger semantics, types.hpp:60-88).
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <memory>
#include <random>
#include <cmath>
#include <tuple>
#include <type_traits>

#include "engine.hpp"

namespace softdtw {
namespace b200 {

inline softdtw_b200::Context &context()
{
    thread_local softdtw_b200::Context ctx(0);
    return ctx;
}

// Every visible device (one context each) for the pair-sharded hot path;
// nullptr when only one device is visible.
inline softdtw_b200::MultiContext *multi_context()
{
    thread_local std::unique_ptr<softdtw_b200::MultiContext> mc = [] {
        int n = 0;
        sdtw_device_count(&n);
        return n > 1 ? std::make_unique<softdtw_b200::MultiContext>(n) : nullptr;
    }();
    return mc.get();
}

template <class F>
auto translate(F &&f) -> decltype(f())
{
    try {
        return f();
    } catch (const softdtw_b200::ValidationError &e) {
        throw ValidationError(e.what());
    } catch (const softdtw_b200::OutOfMemoryError &e) {
        throw OutOfMemoryError(e.requested_bytes());
    } catch (const softdtw_b200::UnreachableEndError &e) {
        throw UnreachableEndError(e.what());
    } catch (const softdtw_b200::IncompleteTableError &e) {
        throw IncompleteTableError(e.what());
    } catch (const softdtw_b200::Error &e) {
        throw Error(e.what());
    }
}

inline softdtw_b200::Config engine_config(const SdtwConfig &cfg)
{
    softdtw_b200::Config c;
    c.gamma = cfg.gamma;
    c.bandwidth = cfg.bandwidth;
    c.fused = cfg.cost_mode == CostMode::fused;
    c.linear_backward = cfg.backward_space == BackwardSpace::linear;
    c.normalized = cfg.normalized;
    return c;
}

// The engine's device peak of the call, charged to the ledger transiently
// (AllocationLedger semantics, types.hpp:60-88); a limited ledger bounds the
// engine's device allocations.
inline void ledger_begin(AllocationLedger *ledger)
{
    auto &ctx = context();
    ctx.set_mem_limit(ledger && ledger->limit_bytes ? ledger->limit_bytes - ledger->live_bytes : 0);
    ctx.reset_peak();
}
inline void ledger_end(AllocationLedger *ledger)
{
    if (!ledger) return;
    const std::size_t peak = context().mem_stats().second;
    ledger->track(peak);
    ledger->release(peak);
}

template <class T>
ForwardResult<T> forward(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                         unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    (void)threads;
    if (x.batch_size() != y.batch_size()) throw ValidationError("forward: batch size mismatch");
    if (x.feature_dim() != y.feature_dim()) throw ValidationError("forward: feature dim mismatch");
    const std::size_t B = x.batch_size(), N = x.length(), M = y.length(), D = x.feature_dim();
    validate_config(cfg, N, M);
    const bool unfused = cfg.cost_mode == CostMode::unfused;
    ForwardResult<T> out;
    // host containers first, so a ledger limit refuses them like the reference's
    out.cache.x_sqnorms = TrackedBuffer<T>(B * N, T(0), ledger);
    out.cache.y_sqnorms = TrackedBuffer<T>(B * M, T(0), ledger);
    out.cache.batch = B;
    out.cache.n = N;
    out.cache.m = M;
    if (unfused) out.costs.emplace(B, N, M, ledger);
    out.table = DpTableBatch<T>(B, N, M, ledger);
    translate([&] {
        softdtw_b200::Config c = engine_config(cfg);
        c.normalized = false;
        ledger_begin(ledger);
        auto o = context().forward<T>(x.raw(), y.raw(), B, N, M, D, c, true, unfused, true);
        ledger_end(ledger);
        std::copy(o.R.begin(), o.R.end(), out.table.buffer().data());
        std::copy(o.norms.begin(), o.norms.begin() + B * N, out.cache.x_sqnorms.data());
        std::copy(o.norms.begin() + B * N, o.norms.end(), out.cache.y_sqnorms.data());
        if (unfused) std::copy(o.costs.begin(), o.costs.end(), const_cast<T *>(out.costs->buffer().data()));
        out.loss = std::move(o.loss);
        return 0;
    });
    return out;
}

template <class T>
std::vector<T> forward_normalized(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    (void)threads;
    if (x.length() != y.length()) throw ValidationError("normalized sdtw requires N == M");
    if (x.batch_size() != y.batch_size()) throw ValidationError("forward: batch size mismatch");
    if (x.feature_dim() != y.feature_dim()) throw ValidationError("forward: feature dim mismatch");
    SdtwConfig plain = cfg;
    plain.normalized = false;
    validate_config(plain, x.length(), y.length());
    return translate([&] {
        softdtw_b200::Config c = engine_config(cfg);
        c.normalized = true;
        ledger_begin(ledger);
        auto o = context().forward<T>(x.raw(), y.raw(), x.batch_size(), x.length(), y.length(), x.feature_dim(),
                                      c, false, false, false);
        ledger_end(ledger);
        return std::move(o.loss);
    });
}

namespace detail {

template <class T, class Cost>
GradTableBatch<T> backward(DpTableBatch<T> &&r, const Cost &cost, const SdtwConfig &cfg, AllocationLedger *ledger,
                           bool linear)
{
    const std::size_t B = r.batch_size(), N = r.n(), M = r.m();
    validate_config(cfg, N, M);
    std::vector<T> E(B * (N + 2) * (M + 2));
    translate([&] {
        softdtw_b200::Config c = engine_config(cfg);
        c.linear_backward = linear;
        ledger_begin(ledger);
        const T *R = r.buffer().data();
        if constexpr (std::is_same_v<Cost, MaterializedCosts<T>>) {
            const auto &d = *cost.d;
            if (d.batch_size() != B || d.n() != N || d.m() != M)
                throw softdtw_b200::ValidationError("backward: cost tensor shape mismatch");
            context().backward_table<T>(R, d.buffer().data(), nullptr, nullptr, B, N, M, 0, c, E.data());
        } else {
            static_assert(std::is_same_v<Cost, FusedCosts<T>>, "cost accessor: MaterializedCosts or FusedCosts");
            const auto &x = *cost.x, &y = *cost.y;
            if (x.batch_size() != B || x.length() != N || y.length() != M)
                throw softdtw_b200::ValidationError("backward: series shape mismatch");
            context().backward_table<T>(R, nullptr, x.raw().data(), y.raw().data(), B, N, M, x.feature_dim(), c,
                                        E.data());
        }
        ledger_end(ledger);
        return 0;
    });
    // the backward consumes the forward table and reuses its slab (backward.hpp:39, 176)
    TrackedBuffer<T> slab = std::move(r).take_buffer();
    std::copy(E.begin(), E.end(), slab.data());
    return GradTableBatch<T>(std::move(slab), B, N, M, GradSpace::linear);
}

}  // namespace detail

template <class T, class Cost>
GradTableBatch<T> backward_log(DpTableBatch<T> &&r, const Cost &cost, const SdtwConfig &cfg, unsigned threads = 0,
                               AllocationLedger *ledger = nullptr)
{
    (void)threads;
    return detail::backward<T, Cost>(std::move(r), cost, cfg, ledger, false);
}

template <class T, class Cost>
GradTableBatch<T> backward_linear(DpTableBatch<T> &&r, const Cost &cost, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    (void)threads;
    return detail::backward<T, Cost>(std::move(r), cost, cfg, ledger, true);
}

template <class T>
InputGradients<T> input_gradients(const GradTableBatch<T> &e, const SeriesBatch<T> &x, const SeriesBatch<T> &y,
                                  unsigned threads = 0)
{
    (void)threads;
    if (e.space() != GradSpace::linear)
        throw ValidationError("input_gradients: gradient table must be in linear space");
    if (e.batch_size() != x.batch_size() || e.n() != x.length() || e.m() != y.length() ||
        x.feature_dim() != y.feature_dim())
        throw ValidationError("input_gradients: shape mismatch");
    const std::size_t B = e.batch_size(), N = e.n(), M = e.m(), D = x.feature_dim();
    InputGradients<T> out;
    out.grad_x.assign(B * N * D, T(0));
    out.grad_y.assign(B * M * D, T(0));
    // the padded slab is contiguous; GradTableBatch exposes it through at()
    const T *E = &const_cast<GradTableBatch<T> &>(e).at(0, 0, 0);
    translate([&] {
        context().input_grads<T>(E, x.raw().data(), y.raw().data(), B, N, M, D, out.grad_x.data(),
                                 out.grad_y.data());
        return 0;
    });
    return out;
}

// sdtw_with_gradients (backward.hpp:276-304).  Log space (the hot path): one
// fused device pipeline.  Linear space (the reference's fragile recurrence,
// backward.hpp:192-203): forward table -> backward_linear -> input_gradients,
// as the reference composes it.
template <class T>
SdtwOutput<T> sdtw_with_gradients(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    if (x.batch_size() != y.batch_size()) throw ValidationError("forward: batch size mismatch");
    if (x.feature_dim() != y.feature_dim()) throw ValidationError("forward: feature dim mismatch");
    validate_config(cfg, x.length(), y.length());
    if (cfg.backward_space == BackwardSpace::linear) {
        ForwardResult<T> fwd = b200::forward(x, y, cfg, threads, ledger);
        GradTableBatch<T> e;
        if (fwd.costs) {
            e = b200::backward_linear(std::move(fwd.table), MaterializedCosts<T>{&*fwd.costs}, cfg, threads, ledger);
            fwd.costs.reset();
        } else {
            e = b200::backward_linear(std::move(fwd.table), FusedCosts<T>{&x, &y, &fwd.cache}, cfg, threads, ledger);
        }
        SdtwOutput<T> out;
        out.loss = std::move(fwd.loss);
        out.grads = b200::input_gradients(e, x, y, threads);
        return out;
    }
    return translate([&] {
        softdtw_b200::Config c = engine_config(cfg);
        c.normalized = false;  // the reference's forward computes the plain loss here
        // several GPUs: contiguous pair shards, one per device (a ledger
        // accounts one device's allocations, so a ledger keeps one device)
        auto *mc = ledger ? nullptr : multi_context();
        softdtw_b200::Output<T> o;
        if (mc && x.batch_size() > 1) {
            o = mc->sdtw_with_gradients<T>(x.raw(), y.raw(), x.batch_size(), x.length(), y.length(),
                                           x.feature_dim(), c);
        } else {
            ledger_begin(ledger);
            o = context().sdtw_with_gradients(x.raw(), y.raw(), x.batch_size(), x.length(), y.length(),
                                              x.feature_dim(), c);
            ledger_end(ledger);
        }
        for (const T v : o.loss)
            if (!std::isfinite(v))
                throw softdtw_b200::UnreachableEndError("forward: R[N,M] is not finite (end cell unreachable)");
        SdtwOutput<T> out;
        out.loss = std::move(o.loss);
        out.grads.grad_x = std::move(o.grad_x);
        out.grads.grad_y = std::move(o.grad_y);
        return out;
    });
}

// barycenter_objective (barycenter.hpp:60-86): unfused, log space (:69-73).
// Members of equal length run as one device batch (z broadcast); members of
// different lengths run as one batch per length, summed in member-group order.
template <class T>
std::pair<double, std::vector<T>> barycenter_objective(const SeriesBatch<T> &z, const BarycenterProblem<T> &prob)
{
    validate_problem(prob);
    if (z.batch_size() != 1 || z.feature_dim() != prob.members.front().feature_dim())
        throw ValidationError("barycenter: z shape mismatch");
    const std::size_t D = z.feature_dim(), Lz = z.length();
    std::vector<std::size_t> lengths;
    for (const auto &m : prob.members)
        if (std::find(lengths.begin(), lengths.end(), m.length()) == lengths.end()) lengths.push_back(m.length());
    return translate([&] {
        auto &ctx = context();
        ctx.set_mem_limit(0);
        double value = 0;
        std::vector<T> grad(Lz * D, T(0)), g(Lz * D);
        for (std::size_t L : lengths) {
            std::vector<T> flat;
            std::vector<double> w;
            std::size_t K = 0;
            for (std::size_t k = 0; k < prob.members.size(); ++k) {
                if (prob.members[k].length() != L) continue;
                flat.insert(flat.end(), prob.members[k].raw().begin(), prob.members[k].raw().end());
                w.push_back(prob.weights.empty() ? 1.0 : prob.weights[k]);
                ++K;
            }
            // several GPUs (fp32): member shards + one NCCL allreduce of grad_z
            auto *mc = multi_context();
            if constexpr (std::is_same<T, float>::value) {
                if (mc && K > 1) {
                    value += mc->barycenter_objective_into(z.raw().data(), Lz, flat.data(), K, L, D, prob.gamma,
                                                           prob.bandwidth, w.data(), g.data());
                    if (lengths.size() == 1) return std::make_pair(value, std::move(g));
                    for (std::size_t i = 0; i < grad.size(); ++i) grad[i] += g[i];
                    continue;
                }
            }
            value += ctx.barycenter_objective_into<T>(z.raw().data(), Lz, flat.data(), K, L, D, prob.gamma,
                                                      prob.bandwidth, w.data(), g.data());
            if (lengths.size() == 1) return std::make_pair(value, std::move(g));
            for (std::size_t i = 0; i < grad.size(); ++i) grad[i] += g[i];
        }
        return std::make_pair(value, std::move(grad));
    });
}

// solve_barycenter (barycenter.hpp:159-211): the reference's Adam loop with
// the objective and the Adam update (fp64 moments, :181-191) on the device.
template <class T>
BarycenterTrace<T> solve_barycenter(const BarycenterProblem<T> &prob,
                                    BarycenterInit init = BarycenterInit::euclidean_mean,
                                    const AdamOptions &opts = {}, std::size_t member_index = 0,
                                    const SeriesBatch<T> *user_z = nullptr)
{
    validate_problem(prob);
    SeriesBatch<T> z = softdtw::detail::initial_z(prob, init, member_index, user_z);
    BarycenterTrace<T> trace;
    auto [value, grad] = b200::barycenter_objective(z, prob);
    trace.objective_per_iteration.push_back(value);
    trace.final_z = z;
    double best = value, prev = value;
    std::vector<double> m1(grad.size(), 0.0), m2(grad.size(), 0.0);
    std::size_t calm = 0;
    for (std::size_t t = 1; t <= opts.max_iters; ++t) {
        translate([&] {
            context().adam_step<T>(z.raw().data(), grad.data(), m1.data(), m2.data(), grad.size(), t, opts.lr,
                                   opts.beta1, opts.beta2, opts.eps);
            return 0;
        });
        std::tie(value, grad) = b200::barycenter_objective(z, prob);
        trace.objective_per_iteration.push_back(value);
        trace.iterations_run = t;
        if (value < best) {
            best = value;
            trace.final_z = z;
        }
        const double delta = std::abs(value - prev) / std::max(1.0, std::abs(value));
        calm = delta < opts.tol ? calm + 1 : 0;
        prev = value;
        if (calm >= 5) {
            trace.converged = true;
            break;
        }
    }
    return trace;
}

}  // namespace b200
}  // namespace softdtw
