// k_fwd_f64.cu — fp64 wavefront forward kernels (sdtw_dp3.cuh).
#include "sdtw_kernels.h"

namespace sdtw {

template <class T, int K, bool kFused>
KFn<Dp3Args<T>> k_forward3()
{
    return sdtw_forward3_kernel<T, K, kFused>;
}
template KFn<Dp3Args<double>> k_forward3<double, 1, false>();
template KFn<Dp3Args<double>> k_forward3<double, 1, true>();

SDTW_TU_TIMEOUTS(fwd_f64)

}  // namespace sdtw
