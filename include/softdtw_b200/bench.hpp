// softdtw_b200/bench.hpp — the benchmark row of the reference's `sdtw bench`
// (bench.hpp:52-138, tools/sdtw.cpp:166-211) measured on the engine.
//
// Include after <softdtw/softdtw.hpp> and softdtw_b200/dropin.hpp.
// measure_row() times one row two ways: end to end through the drop-in on
// the reference's host containers (what the reference's row reports), and
// on the device (the engine's phase events: the fwd+bwd kernels alone), and
// adds the derived figures the reference's CSV lacks: DP cells/s and the
// fraction of the SFU roofline (7 MUFU per cell).
// run_bench_row() is the reference's entry point on top of it.
#pragma once
#include <chrono>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "dropin.hpp"

namespace softdtw {
namespace b200 {

struct EngineBenchRow {
    BenchResultRow row;         // the reference's row (end-to-end times, ledger peak, loss0)
    double device_ms = 0;       // fwd + bwd + gradient kernels, mean over repeats
    double cells_per_s = 0;     // B L^2 / end-to-end mean
    double device_cells_per_s = 0;
    double sfu_fraction = 0;    // device rate / (SMs x 16 MUFU/clk x clock / 7)
};

// The reference's generator (bench.hpp:61-66): N(0,1) floats from
// mt19937_64(seed), every x value first, then every y value.
inline std::pair<std::vector<float>, std::vector<float>> bench_inputs(const BenchConfigRow &row, std::uint64_t seed)
{
    std::mt19937_64 gen(seed);
    std::normal_distribution<float> n01(0.0f, 1.0f);
    std::vector<float> x(row.batch * row.length * row.feature_dim), y(x.size());
    for (float &v : x) v = n01(gen);
    for (float &v : y) v = n01(gen);
    return {std::move(x), std::move(y)};
}

// sm_count, clock_mhz: the device's (148, 1965 on a B200 at max clock)
inline EngineBenchRow measure_row(const BenchConfigRow &row, std::uint64_t seed = 42, std::size_t mem_limit_bytes = 0,
                                  int sm_count = 148, double clock_mhz = 1965.0)
{
    validate_bench_row(row);
    EngineBenchRow res;
    res.row.config = row;
    try {
        auto [xs, ys] = bench_inputs(row, seed);
        const std::size_t B = row.batch, L = row.length, D = row.feature_dim;
        SeriesBatch<float> x(std::move(xs), B, L, D), y(std::move(ys), B, L, D);
        SdtwConfig cfg;
        cfg.gamma = row.gamma;
        cfg.cost_mode = row.cost_mode;
        cfg.backward_space = row.backward_space;
        AllocationLedger ledger;
        ledger.limit_bytes = mem_limit_bytes;
        double sum = 0, sum2 = 0, dev = 0;
        std::size_t timed = 0;
        auto &ctx = context();
        sdtw_ctx_enable_timing(ctx.get(), 1);
        for (std::size_t it = 0; it < row.warmup + row.repeats; ++it) {
            ledger.reset();
            const auto t0 = std::chrono::steady_clock::now();
            const SdtwOutput<float> out = b200::sdtw_with_gradients(x, y, cfg, 0, &ledger);
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            res.row.loss0 = out.loss.front();
            res.row.peak_ledger_bytes = ledger.peak_bytes;
            if (it < row.warmup) continue;
            float ph[SDTW_NUM_PHASES];
            sdtw_phase_times(ctx.get(), ph, SDTW_NUM_PHASES);
            for (float p : ph) dev += p > 0 ? p : 0;
            sum += ms;
            sum2 += ms * ms;
            ++timed;
        }
        sdtw_ctx_enable_timing(ctx.get(), 0);
        const double mean = sum / double(timed);
        res.row.mean_runtime_ms = mean;
        res.row.std_runtime_ms = std::sqrt(std::max(0.0, sum2 / double(timed) - mean * mean));
        res.device_ms = dev / double(timed);
        const double cells = double(B) * double(L) * double(L);
        res.cells_per_s = cells / (mean * 1e-3);
        res.device_cells_per_s = res.device_ms > 0 ? cells / (res.device_ms * 1e-3) : 0;
        res.sfu_fraction = res.device_cells_per_s / (double(sm_count) * 16.0 * clock_mhz * 1e6 / 7.0);
        res.row.ok = true;
    } catch (const std::exception &ex) {
        res.row.ok = false;
        res.row.error = ex.what();
    }
    return res;
}

// run_bench_row (bench.hpp:52-107): the reference's row semantics (same
// generator, end-to-end mean / std over `repeats` after `warmup`, ledger
// peak, loss of pair 0, failures recorded in the row); `threads` is ignored.
inline BenchResultRow run_bench_row(const BenchConfigRow &row, unsigned threads = 0, std::uint64_t seed = 42,
                                    std::size_t mem_limit_bytes = 0)
{
    (void)threads;
    return measure_row(row, seed, mem_limit_bytes).row;
}

}  // namespace b200
}  // namespace softdtw
