// sdtw_common.cuh — numeric primitives shared by every Soft-DTW kernel.
//
// The engine never forms the accumulated cost R in a narrow type.  Every DP
// cell keeps the two edge differences of R that leave it,
//     v(i,j) = R(i,j) - R(i-1,j)        h(i,j) = R(i,j) - R(i,j-1),
// and evaluates the reference recurrence (forward.hpp:30-36,
// softmin.hpp:22-31) relative to the diagonal predecessor:
//     R(i,j) - R(i-1,j-1) = g = d(i,j) + softmin_gamma(0, u, l),
//     u = R(i-1,j) - R(i-1,j-1) = h(i-1,j),   l = R(i,j-1) - R(i-1,j-1) = v(i,j-1),
// so every quantity is O(cost) in magnitude and fp32 keeps ~1e-7 relative
// accuracy in it regardless of |R| (an fp32 R loses the
// backward weights at gamma <= 0.1).  The forward softmin's probabilities
//     P(pred) = exp(-(pred - min)/gamma) / sum
// are exactly the reference's backward transition weights
// exp((R_s - R_self - d_s)/gamma) (backward.hpp:105-121), so the backward is
// the linear recurrence E(i,j) = sum_s E(s) P_s(i,j) over weights in [0,1]:
// it cannot overflow and needs no exp/log at all.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

template <class T>
struct Num;

template <>
struct Num<float> {
    static __device__ __forceinline__ float ex2(float a)
    {
        float r;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
        return r;
    }
    static __device__ __forceinline__ float lg2(float a)
    {
        float r;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
        return r;
    }
    static __device__ __forceinline__ float rcp(float a)
    {
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
        return r;
    }
    static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
};

#ifndef SDTW_EXP_MODE
#define SDTW_EXP_MODE 0
#endif
// exp2 for the softmin probabilities.  Mode 0: MUFU ex2.approx.  Mode 1:
// double precision, rounded once (experiment).  Mode 2: degree-7 polynomial
// on the FMA pipe with round-to-nearest steps (unbiased to ~1 ulp).
__device__ __forceinline__ float exp2_prob(float a)
{
#if SDTW_EXP_MODE == 1
    return __double2float_rn(exp2((double)a));
#elif SDTW_EXP_MODE == 2
    if (!(a >= -126.0f)) return 0.0f;  // also maps -inf / NaN-free inputs to 0
    const float n = rintf(a);
    const float f = a - n;             // [-0.5, 0.5], exact
    float p = 1.5252733804059841e-05f;
    p = fmaf(p, f, 1.5403530393381606e-04f);
    p = fmaf(p, f, 1.3333558146428443e-03f);
    p = fmaf(p, f, 9.6181291076284772e-03f);
    p = fmaf(p, f, 5.5504108664821580e-02f);
    p = fmaf(p, f, 2.4022650695910071e-01f);
    p = fmaf(p, f, 6.9314718055994531e-01f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + ((int)n << 23));
#else
    return Num<float>::ex2(a);
#endif
}

template <>
struct Num<double> {
    static __device__ __forceinline__ double ex2(double a) { return exp2(a); }
    static __device__ __forceinline__ double lg2(double a) { return log2(a); }
    static __device__ __forceinline__ double rcp(double a) { return 1.0 / a; }
    static __device__ __forceinline__ double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
};

// Sakoe-Chiba band on 1-based DP coordinates (wavefront.hpp:31-36 uses
// 0-based ones; the difference is invariant).
__device__ __forceinline__ bool in_band(int i, int j, int bw)
{
    const int diff = i > j ? i - j : j - i;
    return bw == 0 || diff <= bw;
}

// Release/acquire progress flags between cooperating warps on different SMs.
__device__ __forceinline__ void flag_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Set when a dependency wait gave up (a scheduling bug, never expected); the
// host turns it into an error instead of letting a kernel spin forever.
// One copy per translation unit (the kernels live in several); the host
// reads and clears every copy after a call (check_wait_timeouts).
static __device__ int g_sdtw_wait_timeouts = 0;

// Every lane performs its own acquire so its later plain loads are ordered.
// Bounded: after ~2^24 polls (tens of seconds) the wait is abandoned and
// recorded, so a scheduling bug cannot hang the GPU.
__device__ __forceinline__ void wait_flag_geq(const int *p, int need)
{
    if (need <= 0) return;
    int v = flag_acquire(p);
    unsigned polls = 0;
    while (v < need) {
        __nanosleep(128);
        v = flag_acquire(p);
        if (++polls > (1u << 24)) {
            atomicAdd(&g_sdtw_wait_timeouts, 1);
            return;
        }
    }
}

// Outputs of one forward cell.
template <class T>
struct Cell {
    T v, h;           // edge differences leaving the cell
    T g;              // R(i,j) - R(i-1,j-1) (valid for interior non-special cells)
    T pd, pu, pl;     // softmin probabilities of the diag / up / left predecessor
};

// Cell kinds (boundary handling of the padded table, types.hpp:278-294):
//   (1,1): R = d; row 1: R = d + R(1,j-1); column 1: R = d + R(i-1,1);
//   out-of-band: R = +inf (never computed; edges leaving it are +inf).
template <class T, bool kProbs>
__device__ __forceinline__ Cell<T> dp_cell(int i, int j, int bw, T d, T u, T l,
                                           T k /*log2e/gamma*/, T gln2 /*gamma*ln2*/)
{
    Cell<T> c;
    const T inf = Num<T>::inf();
    c.pd = T(0);
    c.pu = T(0);
    c.pl = T(0);
    if (!in_band(i, j, bw)) {
        c.v = inf;
        c.h = inf;
        c.g = inf;
        return c;
    }
    if (i == 1 || j == 1) {
        c.g = d;
        if (i == 1 && j == 1) {
            c.v = -inf;
            c.h = -inf;
        } else if (i == 1) {
            c.h = d;
            c.v = -inf;
            c.pl = T(1);
        } else {
            c.v = d;
            c.h = -inf;
            c.pu = T(1);
        }
        return c;
    }
    // softmin_gamma(0, u, l), min-shifted (softmin.hpp:22-31), base-2 domain.
    T mn = u < l ? u : l;
    mn = mn < T(0) ? mn : T(0);
    const T nk = -k;
    T e0, eu, el;
    if (kProbs && sizeof(T) == 4) {
        e0 = (T)exp2_prob((float)(mn * k));
        eu = (T)exp2_prob((float)((u - mn) * nk));
        el = (T)exp2_prob((float)((l - mn) * nk));
    } else {
        e0 = Num<T>::ex2(mn * k);           // weight of the diagonal pred (value 0)
        eu = Num<T>::ex2((u - mn) * nk);     // +inf -> 0
        el = Num<T>::ex2((l - mn) * nk);
    }
    const T s = (e0 + eu) + el;
    const T sm = mn - gln2 * Num<T>::lg2(s);
    c.g = d + sm;
    // the same rounding as fwd_cell / prob_cell: a tile recomputed through
    // this general cell or through the branch-free one gives identical bits
    c.v = (d - u) + sm;
    c.h = (d - l) + sm;
    if (kProbs) {
        // One Newton step makes the three probabilities sum to 1 within an
        // ulp; an approximate reciprocal's bias would otherwise compound
        // along every alignment path (mass drift ~ L * bias).
        T r = Num<T>::rcp(s);
        r = r * (T(2) - s * r);
        c.pd = e0 * r;
        c.pu = eu * r;
        c.pl = el * r;
    }
    return c;
}

}  // namespace sdtw
