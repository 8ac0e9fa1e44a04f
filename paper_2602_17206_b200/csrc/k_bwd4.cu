// k_bwd4.cu — the tile-worker backward (sdtw_dp4.cuh); the fp32 fused mode
// runs its tensor-core variant.
#include "sdtw_kernels.h"
#include "sdtw_dp4.cuh"

namespace sdtw {

template <class T, bool kFused, bool kTc, int kWin>
KFn<Dp3Args<T>, unsigned long long *, FusedTcArgs> k_backward4()
{
    return sdtw_backward4_kernel<T, kFused, kTc, kWin>;
}
template KFn<Dp3Args<float>, unsigned long long *, FusedTcArgs> k_backward4<float, false, true, 3>();
template KFn<Dp3Args<float>, unsigned long long *, FusedTcArgs> k_backward4<float, false, false, 2>();
template KFn<Dp3Args<float>, unsigned long long *, FusedTcArgs> k_backward4<float, false, false, 3>();
template KFn<Dp3Args<float>, unsigned long long *, FusedTcArgs> k_backward4<float, true, false, 2>();
template KFn<Dp3Args<double>, unsigned long long *, FusedTcArgs> k_backward4<double, false, false, 2>();
template KFn<Dp3Args<double>, unsigned long long *, FusedTcArgs> k_backward4<double, false, false, 3>();
template KFn<Dp3Args<double>, unsigned long long *, FusedTcArgs> k_backward4<double, true, false, 2>();

SDTW_TU_TIMEOUTS(bwd4)

}  // namespace sdtw
