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
    // fused (SIMT costs): one feature block of the strip's 32 x rows and of
    // the 39 y rows a sub-group touches, staged per block (rows padded by 4)
    static constexpr int kKB = sizeof(T) == 4 ? 128 : 64;
    static constexpr int kStage = kFused ? (32 + 40) * (kKB + 1) : 0;
    static constexpr int kPerWarp = kRing + kHalo + kStage;
};

// The 8 costs a fused sub-group needs (lane t: row 32 s + t + 1, columns
// kb + kk - t, kk < 8), with the warp staging x / y feature blocks in shared
// memory (coalesced, each y row loaded once per sub-group instead of once per
// lane).  Same arithmetic, in the same order, as cost_cell: per lane, fp32
// with D % 4 == 0 and aligned rows four partial sums over k = 4 i + r, else
// one sequential sum, then (xn - 2 dot) + yn clamped at 0, so the results are
// bit-identical to the per-lane path (and to the unfused fp64 costs).
template <class T>
__device__ __forceinline__ void fused_costs_staged(const DpArgs<T> &a, int b, int s, int t, int kb, T *stg,
                                                   T (&dk)[8])
{
    constexpr int KB = Fwd2Smem<T, 1, true>::kKB, LD = KB + 1;  // odd stride: conflict-free rows
    T *xs = stg, *ys = stg + 32 * LD;
    const int D = a.D;
    const T *xb = a.x + (size_t)b * a.N * D;
    const T *yb = a.y + (size_t)b * a.M * D;
    const bool quad = sizeof(T) == 4 && (D & 3) == 0 &&
                      ((reinterpret_cast<uintptr_t>(a.x) | reinterpret_cast<uintptr_t>(a.y)) & 15) == 0;
    const int jlo = kb - 31;  // y row of ys[0]
    T acc[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[kk][r] = T(0);
    for (int k0 = 0; k0 < D; k0 += KB) {
        const int kn = min(KB, D - k0);
        __syncwarp();
        // stage: x rows 32 s .. 32 s + 31, y rows jlo .. jlo + 38 (zero
        // outside); 16-byte loads when rows allow, many in flight per lane
        if (quad) {
            const int kq = kn >> 2;
#pragma unroll 8
            for (int u = t; u < 32 * kq; u += 32) {
                const int r = u / kq, c = 4 * (u % kq), i = 32 * s + r;
                const float4 v = i < a.N ? __ldg(reinterpret_cast<const float4 *>(xb + (size_t)i * D + k0 + c))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                T *d = xs + r * LD + c;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
#pragma unroll 8
            for (int u = t; u < 39 * kq; u += 32) {
                const int r = u / kq, c = 4 * (u % kq), j = jlo + r;
                const float4 v = (j >= 0 && j < a.M)
                                     ? __ldg(reinterpret_cast<const float4 *>(yb + (size_t)j * D + k0 + c))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                T *d = ys + r * LD + c;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
        } else {
#pragma unroll 8
            for (int u = t; u < 32 * kn; u += 32) {
                const int r = u / kn, k = u % kn, i = 32 * s + r;
                xs[r * LD + k] = i < a.N ? xb[(size_t)i * D + k0 + k] : T(0);
            }
#pragma unroll 8
            for (int u = t; u < 39 * kn; u += 32) {
                const int r = u / kn, k = u % kn, j = jlo + r;
                ys[r * LD + k] = (j >= 0 && j < a.M) ? yb[(size_t)j * D + k0 + k] : T(0);
            }
        }
        __syncwarp();
        const T *xr = xs + t * LD;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const T *yr = ys + (kk - t + 31) * LD;  // column kb + kk - t
            if (quad) {
                for (int k = 0; k < kn; k += 4) {
                    acc[kk][0] = fma(xr[k], yr[k], acc[kk][0]);
                    acc[kk][1] = fma(xr[k + 1], yr[k + 1], acc[kk][1]);
                    acc[kk][2] = fma(xr[k + 2], yr[k + 2], acc[kk][2]);
                    acc[kk][3] = fma(xr[k + 3], yr[k + 3], acc[kk][3]);
                }
            } else {
                for (int k = 0; k < kn; ++k) acc[kk][0] = fma(xr[k], yr[k], acc[kk][0]);
            }
        }
    }
    const int i = 32 * s + t + 1;
    const T xn = i <= a.N ? a.xn[(size_t)b * a.N + (i - 1)] : T(0);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int col = kb + kk - t;
        const T dot = quad ? (acc[kk][0] + acc[kk][1]) + (acc[kk][2] + acc[kk][3]) : acc[kk][0];
        const T yn = (col >= 0 && col < a.M) ? a.yn[(size_t)b * a.M + col] : T(0);
        const T v = (xn - T(2) * dot) + yn;
        dk[kk] = v < T(0) ? T(0) : v;
    }
}

}  // namespace sdtw
