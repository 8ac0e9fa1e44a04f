// k_gemm.cu — the unfused cost tensor (sdtw_tc.cuh) and the input-gradient
// contraction (sdtw_grad_tc.cuh) on tcgen05.
#include "sdtw_kernels.h"
#include "sdtw_grad_tc.cuh"

namespace sdtw {

KFn<const uint8_t *, const uint8_t *, const float *, const float *, const unsigned *, int, int, int, int, int, int,
    int, int, float *>
k_cost_gemm()
{
    return cost_gemm_tc_kernel<0>;
}

KFn<const float *, const int4 *, const int *, int, const int *, const int *, int, int, int, int, int, int, int,
    const float *, const float *, const unsigned *, float *>
k_contract_tc()
{
    return contract_tc_kernel<0>;
}

}  // namespace sdtw
