// bench_sweep — the reference's `sdtw bench` CSV (bench.hpp:109-138,
// tools/sdtw.cpp:166-211) on the B200 engine through the C++ drop-in
// (softdtw::b200::run_bench_row), over the paper's Fig. 1 axes at B = 32
// (SURVEY.md §8(d)): L in {128 .. 4096} at D = 128 and D in {16 .. 1024} at
// L = 256, both cost modes, log space.  Columns: the reference's own, then
// DP cells/s (B L^2 / mean time, end to end with host buffers), DP cells/s on
// the device (the fwd+bwd kernels alone) and that rate as a fraction of the
// SFU roofline (7 MUFU per cell), the GPU count, the host core count and the
// device peak in MB (softdtw::b200::measure_row, softdtw_b200/bench.hpp).
//
//   tools/_bin/bench_sweep [--quick] [--repeats R] [--gamma G] > sweep.csv
#include <softdtw/softdtw.hpp>

#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "softdtw_b200/dropin.hpp"
#include "softdtw_b200/bench.hpp"

using namespace softdtw;

int main(int argc, char **argv)
{
    bool quick = false;
    std::size_t repeats = 5;
    double gamma = 0.1;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--quick")) quick = true;
        else if (!std::strcmp(argv[i], "--repeats") && i + 1 < argc) repeats = std::stoul(argv[++i]);
        else if (!std::strcmp(argv[i], "--gamma") && i + 1 < argc) gamma = std::stod(argv[++i]);
    }
    std::vector<std::pair<std::size_t, std::size_t>> shapes;  // (L, D)
    const std::vector<std::size_t> Ls = quick ? std::vector<std::size_t>{128, 256}
                                              : std::vector<std::size_t>{128, 256, 512, 1024, 2048, 4096};
    const std::vector<std::size_t> Ds = quick ? std::vector<std::size_t>{16, 128}
                                              : std::vector<std::size_t>{16, 32, 64, 128, 256, 512, 1024};
    for (auto L : Ls) shapes.emplace_back(L, 128);
    for (auto D : Ds)
        if (D != 128) shapes.emplace_back(256, D);
    std::printf("%s,cells_per_s,device_cells_per_s,sfu_roofline_fraction,gpus,host_cores,device_peak_mb\n",
                bench_csv_header().c_str());
    for (auto [L, D] : shapes) {
        for (CostMode mode : {CostMode::unfused, CostMode::fused}) {
            BenchConfigRow row;
            row.batch = 32;
            row.length = L;
            row.feature_dim = D;
            row.gamma = gamma;
            row.cost_mode = mode;
            row.repeats = repeats;
            row.warmup = 1;
            const b200::EngineBenchRow e = b200::measure_row(row);
            const BenchResultRow &r = e.row;
            std::printf("%s,%.6g,%.6g,%.4f,1,%u,%.1f\n", bench_csv_row(r).c_str(), r.ok ? e.cells_per_s : 0.0,
                        r.ok ? e.device_cells_per_s : 0.0, r.ok ? e.sfu_fraction : 0.0,
                        std::thread::hardware_concurrency(), double(r.peak_ledger_bytes) / (1 << 20));
            std::fflush(stdout);
        }
    }
    return 0;
}
