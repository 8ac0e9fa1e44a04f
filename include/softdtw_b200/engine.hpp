// softdtw_b200/engine.hpp — C++ host layer over the C-ABI (sdtw_capi.h).
//
// RAII context, typed errors and std::vector entry points that mirror the
// reference's functions (proj/include/softdtw/*.hpp) without depending on its
// headers: plain row-major buffers, the reference's argument meaning and its
// exception taxonomy (types.hpp:17-54).  dropin.hpp adapts these to the
// reference's own containers.
#pragma once
#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../sdtw_capi.h"

namespace softdtw_b200 {

// Error taxonomy of the reference (types.hpp:17-54), one class per status.
class Error : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
class ValidationError : public Error {
  public:
    using Error::Error;
};
class OutOfMemoryError : public Error {
  public:
    explicit OutOfMemoryError(std::size_t requested)
        : Error("allocation of " + std::to_string(requested) + " bytes refused"), requested_(requested)
    {
    }
    std::size_t requested_bytes() const { return requested_; }

  private:
    std::size_t requested_;
};
class UnreachableEndError : public Error {
  public:
    using Error::Error;
};
class IncompleteTableError : public Error {
  public:
    using Error::Error;
};

inline void check(int rc)
{
    switch (rc) {
        case SDTW_OK: return;
        case SDTW_EINVAL: throw ValidationError(sdtw_last_error());
        case SDTW_ENOMEM: throw OutOfMemoryError(sdtw_last_oom_bytes());
        case SDTW_EUNREACHABLE: throw UnreachableEndError(sdtw_last_error());
        case SDTW_EINCOMPLETE: throw IncompleteTableError(sdtw_last_error());
        default: throw Error(sdtw_last_error());
    }
}

// SdtwConfig (types.hpp:222-228) in C-ABI form.
struct Config {
    double gamma = 1.0;
    std::size_t bandwidth = 0;
    bool fused = false;
    bool linear_backward = false;
    bool normalized = false;
    sdtw_config c() const
    {
        return sdtw_config{gamma, bandwidth, fused ? SDTW_COST_FUSED : SDTW_COST_UNFUSED,
                           linear_backward ? SDTW_BWD_LINEAR : SDTW_BWD_LOG, normalized ? 1 : 0};
    }
};

template <class T>
struct Output {
    std::vector<T> loss;     // B
    std::vector<T> grad_x;   // B x N x D
    std::vector<T> grad_y;   // B x M x D
};

// One engine context per (thread, device); move-only.
class Context {
  public:
    explicit Context(int device = 0) { check(sdtw_ctx_create(device, &ctx_)); }
    ~Context()
    {
        if (ctx_) sdtw_ctx_destroy(ctx_);
    }
    Context(const Context &) = delete;
    Context &operator=(const Context &) = delete;
    Context(Context &&o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
    sdtw_ctx *get() const { return ctx_; }

    // AllocationLedger (types.hpp:60-88): live / peak device bytes, limit
    std::pair<std::size_t, std::size_t> mem_stats() const
    {
        std::size_t live = 0, peak = 0;
        check(sdtw_mem_stats(ctx_, &live, &peak));
        return {live, peak};
    }
    void reset_peak() { check(sdtw_mem_reset_peak(ctx_)); }
    void set_mem_limit(std::size_t bytes) { check(sdtw_set_mem_limit(ctx_, bytes)); }

    // sdtw_with_gradients (backward.hpp:276-304): host buffers in, host out.
    Output<float> sdtw_with_gradients(const std::vector<float> &x, const std::vector<float> &y, std::size_t B,
                                      std::size_t N, std::size_t M, std::size_t D, const Config &cfg)
    {
        return run<float>(x, y, B, N, M, D, cfg);
    }
    Output<double> sdtw_with_gradients(const std::vector<double> &x, const std::vector<double> &y,
                                       std::size_t B, std::size_t N, std::size_t M, std::size_t D,
                                       const Config &cfg)
    {
        return run<double>(x, y, B, N, M, D, cfg);
    }

    // barycenter_objective (barycenter.hpp:60-86): value and grad_z.
    std::pair<double, std::vector<float>> barycenter_objective(const std::vector<float> &z, std::size_t Lz,
                                                               const std::vector<float> &members,
                                                               std::size_t K, std::size_t L, std::size_t D,
                                                               double gamma, std::size_t bandwidth = 0,
                                                               const std::vector<double> &weights = {})
    {
        std::vector<float> grad(Lz * D);
        double value = 0;
        check(sdtw_barycenter_objective_f32(ctx_, z.data(), Lz, members.data(), K, L, D, gamma, bandwidth,
                                            weights.empty() ? nullptr : weights.data(), SDTW_PTR_HOST, &value,
                                            grad.data()));
        return {value, std::move(grad)};
    }

  private:
    template <class T>
    Output<T> run(const std::vector<T> &x, const std::vector<T> &y, std::size_t B, std::size_t N, std::size_t M,
                  std::size_t D, const Config &cfg)
    {
        if (x.size() != B * N * D || y.size() != B * M * D) throw ValidationError("buffer size mismatch");
        Output<T> out;
        out.loss.resize(B);
        out.grad_x.resize(B * N * D);
        out.grad_y.resize(B * M * D);
        const sdtw_config c = cfg.c();
        if constexpr (sizeof(T) == 4)
            check(sdtw_fwd_bwd_f32(ctx_, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST, out.loss.data(),
                                   out.grad_x.data(), out.grad_y.data()));
        else
            check(sdtw_fwd_bwd_f64(ctx_, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST, out.loss.data(),
                                   out.grad_x.data(), out.grad_y.data()));
        return out;
    }
    sdtw_ctx *ctx_ = nullptr;
};

}  // namespace softdtw_b200
