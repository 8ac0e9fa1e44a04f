// k_gemm.cu — the unfused cost tensor on tcgen05 (sdtw_tc.cuh).
#include "sdtw_kernels.h"

namespace sdtw {

KFn<const uint8_t *, const uint8_t *, const float *, const float *, const unsigned *, int, int, int, int, int, int,
    int, int, float *>
k_cost_gemm()
{
    return cost_gemm_tc_kernel<0>;
}

}  // namespace sdtw
