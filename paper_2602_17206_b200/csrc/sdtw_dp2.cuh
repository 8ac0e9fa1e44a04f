// sdtw_dp2.cuh — second-generation wavefront DP kernels.
//
// Same strip decomposition, checkpoints and ticket schedule as sdtw_dp.cuh
// (which documents them); what changes is how a warp is fed and how much
// independent work it carries:
//   * costs (unfused) arrive by cp.async into a per-warp shared-memory ring,
//     one 4 KB skewed row group (32 steps x 32 lanes) at a time, a group
//     ahead of use, so no step waits on HBM;
//   * forward: one warp owns K consecutive strips (a "virtual 32K-lane warp":
//     lane t runs rows t, t+32, ..., lagged 32 steps apart, the hand-off
//     between them is the same rotating shuffle as inside a strip), giving K
//     independent cells per step for latency hiding (ILP);
//   * forward softmin uses 2 ex2 + 1 lg2 (the minimum's term is exactly 1);
//   * halos between super-strips are published every 8 columns by lane 31
//     itself (its own release orders its stores), consumers prefetch them.
#pragma once
#include "sdtw_common.cuh"
#include "sdtw_dp.cuh"

namespace sdtw {

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Copies one skewed row group (32 rows x 32 lanes of T) to shared memory.
template <class T>
__device__ __forceinline__ void load_group(T *dst, const T *src, int lane)
{
    constexpr int kBytes = 32 * 32 * sizeof(T);
    const char *s = reinterpret_cast<const char *>(src);
    char *d = reinterpret_cast<char *>(dst);
#pragma unroll
    for (int o = lane * 16; o < kBytes; o += 32 * 16) cp_async16(d + o, s + o);
}

// Forward cell, interior case: softmin over (0, u, l) with 2 ex2 + 1 lg2.
// min/max via fmin/fmax (one FMNMX each; inputs are finite or +/-inf, never
// NaN), and v = (d - u) + sm, h = (d - l) + sm so the softmin is the last
// addition on the dependency chain into the next step's shuffle.
__device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double tmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }

// Three-input min / max (FMNMX3, sm_100): min3(u, l, 0), max3(u, l, 0) and
// the median min3(max(u, l), max(u, 0), max(l, 0)) are the exact values of
// the two-input sorting network below, two levels shallower on the chain.
__device__ __forceinline__ float min3f(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c)
{
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <class T>
__device__ __forceinline__ void fwd_cell(T d, T u, T l, T k, T gln2, T &g, T &v, T &h)
{
    if constexpr (sizeof(T) == 4) {
        const float mn = min3f(u, l, 0.f);
        const float mx = max3f(u, l, 0.f);
        const float md = min3f(fmaxf(u, l), fmaxf(u, 0.f), fmaxf(l, 0.f));
        const float e1 = Num<float>::ex2((mn - md) * k);
        const float e2 = Num<float>::ex2((mn - mx) * k);
        const float s = (e1 + e2) + 1.f;
        const float sm = mn - gln2 * Num<float>::lg2(s);
        g = d + sm;
        v = (d - u) + sm;
        h = (d - l) + sm;
        return;
    }
    const T lo = tmin(u, l);
    const T hi = tmax(u, l);
    const T mn = tmin(lo, T(0));
    const T mx = tmax(hi, T(0));
    const T md = tmax(lo, tmin(hi, T(0)));
    const T e1 = Num<T>::ex2((mn - md) * k);
    const T e2 = Num<T>::ex2((mn - mx) * k);
    const T s = (e1 + e2) + T(1);
    const T sm = mn - gln2 * Num<T>::lg2(s);
    g = d + sm;
    v = (d - u) + sm;
    h = (d - l) + sm;
}

template <class T, int K, bool kFused>
struct Fwd2Smem {
    static constexpr int kRing = kFused ? 0 : K * 2 * 32 * 32;  // T elements per warp
    static constexpr int kHalo = 32;
    static constexpr int kPerWarp = kRing + kHalo;
};

}  // namespace sdtw
