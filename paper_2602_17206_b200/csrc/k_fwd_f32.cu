// k_fwd_f32.cu — fp32 forward kernels: the wavefront forward (sdtw_dp3.cuh,
// unfused and SIMT-fused) and the tensor-core fused forward (sdtw_fused.cuh).
#include "sdtw_kernels.h"

namespace sdtw {

template <class T, int K, bool kFused>
KFn<Dp3Args<T>> k_forward3()
{
    return sdtw_forward3_kernel<T, K, kFused>;
}
template KFn<Dp3Args<float>> k_forward3<float, 1, false>();
template KFn<Dp3Args<float>> k_forward3<float, 1, true>();

KFn<Dp3Args<float>, FusedTcArgs> k_forward_tc(bool trace)
{
    return trace ? sdtw_forward_tc_kernel<0, true> : sdtw_forward_tc_kernel<0, false>;
}

SDTW_TU_TIMEOUTS(fwd_f32)

}  // namespace sdtw
