// softdtw_b200/dropin.hpp — the reference's own API on the B200 engine.
//
// Include after the reference's <softdtw/softdtw.hpp>.  Provides, in
// namespace softdtw::b200, the reference's signatures on the reference's
// containers, each a drop-in for the function it names:
//   sdtw_with_gradients<T>(x, y, cfg, threads, ledger)   backward.hpp:276-304
//   barycenter_objective<T>(z, prob)                     barycenter.hpp:60-86
// Engine errors are rethrown as the reference's exception types
// (types.hpp:17-54), so callers' catch clauses keep working.  `threads` is
// accepted and ignored (the GPU schedule replaces WorkerTeam,
// parallel.hpp:13-71); the ledger, if given, is charged with the engine's
// device peak (AllocationLedger semantics, types.hpp:60-88).
#pragma once
#include "engine.hpp"

namespace softdtw {
namespace b200 {

inline softdtw_b200::Context &context()
{
    thread_local softdtw_b200::Context ctx(0);
    return ctx;
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

template <class T>
SdtwOutput<T> sdtw_with_gradients(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    (void)threads;
    if (x.batch_size() != y.batch_size()) throw ValidationError("batch size mismatch");
    if (x.feature_dim() != y.feature_dim()) throw ValidationError("feature dim mismatch");
    return translate([&] {
        softdtw_b200::Config c;
        c.gamma = cfg.gamma;
        c.bandwidth = cfg.bandwidth;
        c.fused = cfg.cost_mode == CostMode::fused;
        c.linear_backward = cfg.backward_space == BackwardSpace::linear;
        c.normalized = cfg.normalized;
        auto &ctx = context();
        // a limited ledger bounds the engine's device allocations too
        ctx.set_mem_limit(ledger && ledger->limit_bytes ? ledger->limit_bytes - ledger->live_bytes : 0);
        ctx.reset_peak();
        auto o = ctx.sdtw_with_gradients(x.raw(), y.raw(), x.batch_size(), x.length(), y.length(),
                                         x.feature_dim(), c);
        if (ledger) {
            const std::size_t peak = ctx.mem_stats().second;
            ledger->track(peak);
            ledger->release(peak);
        }
        SdtwOutput<T> out;
        out.loss = std::move(o.loss);
        out.grads.grad_x = std::move(o.grad_x);
        out.grads.grad_y = std::move(o.grad_y);
        return out;
    });
}

template <class T>
std::pair<double, std::vector<T>> barycenter_objective(const SeriesBatch<T> &z, const BarycenterProblem<T> &prob)
{
    static_assert(sizeof(T) == 4, "the drop-in barycenter objective is the fp32 path");
    if (z.batch_size() != 1) throw ValidationError("barycenter: z shape mismatch");
    if (prob.members.empty()) throw ValidationError("barycenter: need at least one member series");
    const std::size_t K = prob.members.size(), L = prob.members.front().length(),
                      D = prob.members.front().feature_dim();
    std::vector<T> flat;
    flat.reserve(K * L * D);
    for (const auto &m : prob.members) {
        if (m.batch_size() != 1 || m.length() != L || m.feature_dim() != D)
            throw ValidationError("barycenter: members must share length and dim");
        flat.insert(flat.end(), m.raw().begin(), m.raw().end());
    }
    return translate([&] {
        auto &ctx = context();
        ctx.set_mem_limit(0);
        return ctx.barycenter_objective(z.raw(), z.length(), flat, K, L, D, prob.gamma, prob.bandwidth,
                                        prob.weights);
    });
}

}  // namespace b200
}  // namespace softdtw
