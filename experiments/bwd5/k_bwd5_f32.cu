// k_bwd5_f32.cu — the per-pair pipeline backward (sdtw_bwd5.cuh), float.
#include "sdtw_kernels.h"
#include "sdtw_bwd5.cuh"

namespace sdtw {

template <class T, int kCost, int NE, int NH>
KFn<Dp3Args<T>, T *, T *, int *> k_backward5()
{
    return sdtw_backward5_kernel<T, kCost, NE, NH>;
}
template KFn<Dp3Args<float>, float *, float *, int *> k_backward5<float, 0, 4, 12>();
template KFn<Dp3Args<float>, float *, float *, int *> k_backward5<float, 1, 4, 12>();

// diagnostics: the last timed-out waits of the backward (site, CTA, a, b)
int take_b5_dbg_f32(int *out, int n)
{
    int h[4 + 4 * 64];
    if (cudaMemcpyFromSymbol(h, g_b5_dbg, sizeof h) != cudaSuccess) return 0;
    for (int i = 0; i < n && i < 4 + 4 * 64; ++i) out[i] = h[i];
    static const int zero[4 + 4 * 64] = {};
    cudaMemcpyToSymbol(g_b5_dbg, zero, sizeof zero);
    return h[0];
}

void set_b5_spin_limit_f32(unsigned v) { cudaMemcpyToSymbol(g_b5_spin_limit, &v, sizeof v); }

SDTW_TU_TIMEOUTS(bwd5_f32)

}  // namespace sdtw
