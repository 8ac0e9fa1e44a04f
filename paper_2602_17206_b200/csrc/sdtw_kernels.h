// sdtw_kernels.h — host-side handles of the DP kernels, which are compiled in
// their own translation units (k_*.cu) so the library builds in parallel.
// Each handle returns the typed __global__ function pointer; the host
// launches it with cudaLaunchKernel (launch_ptr in sdtw_capi.cu), so the
// arguments are converted to the kernel's declared parameter types.
#pragma once
#include <cstdint>
#include "sdtw_dp3.cuh"
#include "sdtw_fused.cuh"

namespace sdtw {

template <class... P>
using KFn = void (*)(P...);

// k_fwd_f32.cu / k_fwd_f64.cu
template <class T, int K, bool kFused>
KFn<Dp3Args<T>> k_forward3();
KFn<Dp3Args<float>, FusedTcArgs> k_forward_tc(bool trace);  // trace: the %globaltimer / clock64 build
// k_bwd4.cu
template <class T, bool kFused, bool kTc, int kWin>
KFn<Dp3Args<T>, unsigned long long *, FusedTcArgs> k_backward4();
// k_gemm.cu
KFn<const uint8_t *, const uint8_t *, const float *, const float *, const unsigned *, int, int, int, int, int, int,
    int, int, float *>
k_cost_gemm();
KFn<const float *, const int4 *, const int *, int, const int *, const int *, int, int, int, int, int, int, int,
    const float *, const float *, const unsigned *, float *>
k_contract_tc();
constexpr int kContractTcThreads = 512;  // kCtThreads (sdtw_grad_tc.cuh)
constexpr size_t kContractTcSmem = 4 * 2 * (2 * 128 * 32 * 2 + 2 * 32 * 32 * 2);  // kCtGroups x kCtGroupSmem

// dependency waits that gave up, per translation unit (read and cleared)
int take_timeouts_fwd_f32();
int take_timeouts_fwd_f64();
int take_timeouts_bwd4();

}  // namespace sdtw

// defines take_timeouts_<name>() in a kernel translation unit
#define SDTW_TU_TIMEOUTS(name)                                                         \
    int take_timeouts_##name()                                                         \
    {                                                                                  \
        int n = 0;                                                                     \
        if (cudaMemcpyFromSymbol(&n, g_sdtw_wait_timeouts, sizeof(int)) != cudaSuccess) \
            return 0;                                                                  \
        if (n) {                                                                       \
            const int zero = 0;                                                        \
            cudaMemcpyToSymbol(g_sdtw_wait_timeouts, &zero, sizeof(int));              \
        }                                                                              \
        return n;                                                                      \
    }
