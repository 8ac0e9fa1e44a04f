// b200_redirect.hpp — the reference's own headers with its hot-path
// functions served by the B200 engine: the same-name drop-in.  Code written
// against the reference (its unit suite, its CLI tools/sdtw.cpp, a user's
// program) compiles unchanged and runs on the GPU when include/softdtw_redirect
// comes first on the include path and it links libsdtw_b200.so.
//
// This directory is put FIRST on the include path; its softdtw/forward.hpp,
// backward.hpp and barycenter.hpp all land here.  The reference's real
// headers are then included (#include_next) with their function names
// renamed to sdtw_ref_cpu_* by macros, and the names softdtw::forward,
// forward_normalized, backward_log, backward_linear, input_gradients,
// sdtw_with_gradients, barycenter_objective and solve_barycenter are defined
// to call softdtw::b200:: (include/softdtw_b200/dropin.hpp) with the same
// signatures and defaults (forward.hpp:43-102, backward.hpp:183-304,
// barycenter.hpp:60-211).  Types, errors, the oracle, datasets and the
// ledger are the reference's own.
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <tuple>
#include <type_traits>
#include <utility>
#include <vector>

#include "softdtw/cost.hpp"
#include "softdtw/parallel.hpp"
#include "softdtw/softmin.hpp"
#include "softdtw/types.hpp"
#include "softdtw/wavefront.hpp"

#define forward sdtw_ref_cpu_forward
#define forward_normalized sdtw_ref_cpu_forward_normalized
#define backward_log sdtw_ref_cpu_backward_log
#define backward_linear sdtw_ref_cpu_backward_linear
#define input_gradients sdtw_ref_cpu_input_gradients
#define sdtw_with_gradients sdtw_ref_cpu_sdtw_with_gradients
#define barycenter_objective sdtw_ref_cpu_barycenter_objective
#define solve_barycenter sdtw_ref_cpu_solve_barycenter
#include_next "softdtw/forward.hpp"
#include_next "softdtw/backward.hpp"
#include_next "softdtw/barycenter.hpp"
#undef forward
#undef forward_normalized
#undef backward_log
#undef backward_linear
#undef input_gradients
#undef sdtw_with_gradients
#undef barycenter_objective
#undef solve_barycenter

#include "softdtw_b200/dropin.hpp"

namespace softdtw {

template <class T>
ForwardResult<T> forward(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                         unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    return b200::forward(x, y, cfg, threads, ledger);
}

template <class T>
std::vector<T> forward_normalized(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    return b200::forward_normalized(x, y, cfg, threads, ledger);
}

template <class T, class Cost>
GradTableBatch<T> backward_log(DpTableBatch<T> &&r, const Cost &cost, const SdtwConfig &cfg, unsigned threads = 0,
                               AllocationLedger *ledger = nullptr)
{
    return b200::backward_log(std::move(r), cost, cfg, threads, ledger);
}

template <class T, class Cost>
GradTableBatch<T> backward_linear(DpTableBatch<T> &&r, const Cost &cost, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    return b200::backward_linear(std::move(r), cost, cfg, threads, ledger);
}

template <class T>
InputGradients<T> input_gradients(const GradTableBatch<T> &e, const SeriesBatch<T> &x, const SeriesBatch<T> &y,
                                  unsigned threads = 0)
{
    return b200::input_gradients(e, x, y, threads);
}

template <class T>
SdtwOutput<T> sdtw_with_gradients(const SeriesBatch<T> &x, const SeriesBatch<T> &y, const SdtwConfig &cfg,
                                  unsigned threads = 0, AllocationLedger *ledger = nullptr)
{
    return b200::sdtw_with_gradients(x, y, cfg, threads, ledger);
}

template <class T>
std::pair<double, std::vector<T>> barycenter_objective(const SeriesBatch<T> &z, const BarycenterProblem<T> &prob)
{
    return b200::barycenter_objective(z, prob);
}

template <class T>
BarycenterTrace<T> solve_barycenter(const BarycenterProblem<T> &prob,
                                    BarycenterInit init = BarycenterInit::euclidean_mean, const AdamOptions &opts = {},
                                    std::size_t member_index = 0, const SeriesBatch<T> *user_z = nullptr)
{
    return b200::solve_barycenter(prob, init, opts, member_index, user_z);
}

}  // namespace softdtw
