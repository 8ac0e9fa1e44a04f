// softdtw_b200/engine.hpp — C++ host layer over the C-ABI (sdtw_capi.h).
//
// RAII context, typed errors and std::vector entry points that mirror the
// reference's functions (proj/include/softdtw/*.hpp) without depending on its
// headers: plain row-major buffers, the reference's argument meaning and its
// exception taxonomy (types.hpp:17-54).  dropin.hpp adapts these to the
// reference's own containers.
#pragma once
#include <algorithm>
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

    // forward (forward.hpp:43-81): loss and, on request, the padded R table
    // B x (N+2) x (M+2), the cost tensor B x N x M (unfused mode) and the
    // norm cache (B*N x-norms then B*M y-norms).  cfg.normalized selects
    // forward_normalized (forward.hpp:85-102).
    template <class T>
    struct ForwardOut {
        std::vector<T> loss, R, costs, norms;
    };
    template <class T>
    ForwardOut<T> forward(const std::vector<T> &x, const std::vector<T> &y, std::size_t B, std::size_t N,
                          std::size_t M, std::size_t D, const Config &cfg, bool table, bool costs, bool norms)
    {
        if (x.size() != B * N * D || y.size() != B * M * D) throw ValidationError("buffer size mismatch");
        ForwardOut<T> o;
        o.loss.resize(B);
        if (table) o.R.resize(B * (N + 2) * (M + 2));
        if (costs) o.costs.resize(B * N * M);
        if (norms) o.norms.resize(B * (N + M));
        const sdtw_config c = cfg.c();
        T *r = table ? o.R.data() : nullptr, *d = costs ? o.costs.data() : nullptr,
          *nm = norms ? o.norms.data() : nullptr;
        if constexpr (sizeof(T) == 4)
            check(sdtw_forward_f32(ctx_, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST, o.loss.data(), r, d, nm));
        else
            check(sdtw_forward_f64(ctx_, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST, o.loss.data(), r, d, nm));
        return o;
    }

    // backward_log / backward_linear over a padded R table (backward.hpp:183-203).
    // costs: B x N x M (MaterializedCosts) or null with x / y (FusedCosts).
    // Returns the linear-space E table, B x (N+2) x (M+2).
    template <class T>
    void backward_table(const T *R, const T *costs, const T *x, const T *y, std::size_t B, std::size_t N,
                        std::size_t M, std::size_t D, const Config &cfg, T *E_out)
    {
        const sdtw_config c = cfg.c();
        if constexpr (sizeof(T) == 4)
            check(sdtw_backward_table_f32(ctx_, R, costs, x, y, B, N, M, D, &c, SDTW_PTR_HOST, E_out));
        else
            check(sdtw_backward_table_f64(ctx_, R, costs, x, y, B, N, M, D, &c, SDTW_PTR_HOST, E_out));
    }

    // input_gradients (backward.hpp:208-266) from a padded linear E table.
    template <class T>
    void input_grads(const T *E, const T *x, const T *y, std::size_t B, std::size_t N, std::size_t M,
                     std::size_t D, T *gx, T *gy)
    {
        if constexpr (sizeof(T) == 4)
            check(sdtw_input_grads_f32(ctx_, E, x, y, B, N, M, D, SDTW_PTR_HOST, gx, gy));
        else
            check(sdtw_input_grads_f64(ctx_, E, x, y, B, N, M, D, SDTW_PTR_HOST, gx, gy));
    }

    // barycenter_objective for either precision (members K x L x D, equal L).
    template <class T>
    double barycenter_objective_into(const T *z, std::size_t Lz, const T *members, std::size_t K, std::size_t L,
                                     std::size_t D, double gamma, std::size_t bandwidth, const double *weights,
                                     T *grad)
    {
        double value = 0;
        if constexpr (sizeof(T) == 4)
            check(sdtw_barycenter_objective_f32(ctx_, z, Lz, members, K, L, D, gamma, bandwidth, weights,
                                                SDTW_PTR_HOST, &value, grad));
        else
            check(sdtw_barycenter_objective_f64(ctx_, z, Lz, members, K, L, D, gamma, bandwidth, weights,
                                                SDTW_PTR_HOST, &value, grad));
        return value;
    }

    // One Adam step (barycenter.hpp:181-191): fp64 moments, z updated in place.
    template <class T>
    void adam_step(T *z, const T *grad, double *m1, double *m2, std::size_t n, std::size_t t, double lr,
                   double beta1, double beta2, double eps)
    {
        if constexpr (sizeof(T) == 4)
            check(sdtw_adam_step_f32(ctx_, z, grad, m1, m2, n, t, lr, beta1, beta2, eps, SDTW_PTR_HOST));
        else
            check(sdtw_adam_step_f64(ctx_, z, grad, m1, m2, n, t, lr, beta1, beta2, eps, SDTW_PTR_HOST));
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

// One context per visible device: sdtw_with_gradients over
// contiguous pair shards, all devices concurrently (no collective; bit for
// bit the single-device result), and the barycenter objective over member
// shards with one NCCL allreduce of grad_z (ncclCommInitAll, one process).
class MultiContext {
  public:
    // devices 0 .. ndev-1 (ndev < 0: every visible device)
    explicit MultiContext(int ndev = -1)
    {
        if (ndev < 0) check(sdtw_device_count(&ndev));
        if (ndev < 1) throw Error("no CUDA device available (the engine has no CPU fallback)");
        for (int d = 0; d < ndev; ++d) ctx_.emplace_back(d);
        for (auto &c : ctx_) raw_.push_back(c.get());
    }
    int devices() const { return (int)ctx_.size(); }
    Context &operator[](int g) { return ctx_[g]; }

    template <class T>
    Output<T> sdtw_with_gradients(const std::vector<T> &x, const std::vector<T> &y, std::size_t B, std::size_t N,
                                  std::size_t M, std::size_t D, const Config &cfg)
    {
        if (x.size() != B * N * D || y.size() != B * M * D) throw ValidationError("buffer size mismatch");
        Output<T> out;
        out.loss.resize(B);
        out.grad_x.resize(B * N * D);
        out.grad_y.resize(B * M * D);
        const sdtw_config c = cfg.c();
        const int G = (int)std::min<std::size_t>(raw_.size(), B);
        if constexpr (sizeof(T) == 4)
            check(sdtw_fwd_bwd_multi_f32(raw_.data(), G, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST,
                                         out.loss.data(), out.grad_x.data(), out.grad_y.data()));
        else
            check(sdtw_fwd_bwd_multi_f64(raw_.data(), G, x.data(), y.data(), B, N, M, D, &c, SDTW_PTR_HOST,
                                         out.loss.data(), out.grad_x.data(), out.grad_y.data()));
        return out;
    }

    // fp32 barycenter objective over all devices (one NCCL communicator,
    // created on first use); a single device takes the one-context path.
    double barycenter_objective_into(const float *z, std::size_t Lz, const float *members, std::size_t K,
                                     std::size_t L, std::size_t D, double gamma, std::size_t bandwidth,
                                     const double *weights, float *grad)
    {
        if (raw_.size() == 1)
            return ctx_[0].barycenter_objective_into<float>(z, Lz, members, K, L, D, gamma, bandwidth, weights, grad);
        if (!nccl_) {
            check(sdtw_nccl_init_all(raw_.data(), (int)raw_.size()));
            nccl_ = true;
        }
        double value = 0;
        check(sdtw_barycenter_objective_multi_f32(raw_.data(), (int)raw_.size(), z, Lz, members, K, L, D, gamma,
                                                  bandwidth, weights, SDTW_PTR_HOST, &value, grad));
        return value;
    }

  private:
    std::vector<Context> ctx_;
    std::vector<sdtw_ctx *> raw_;
    bool nccl_ = false;
};

}  // namespace softdtw_b200
