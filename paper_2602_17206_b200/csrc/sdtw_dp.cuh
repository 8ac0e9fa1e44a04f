// sdtw_dp.cuh — strip-pipelined wavefront DP kernels (forward and backward).
//
// Replaces the reference's per-anti-diagonal barrier sweep
// (wavefront.hpp:81-110, backward.hpp:29-177) with a persistent grid of warps.
//
// Work unit = one STRIP: 32 consecutive DP rows of one pair (lane t owns row
// 32*s + t + 1) swept over all M columns.  Inside a strip the 32 lanes run
// skewed by one column per lane, so at step k lane t handles column k - t + 1
// and every lane is on the same anti-diagonal: the up-neighbour's value
// arrives by one warp shuffle, the left-neighbour's stays in a register.
// Between strips the bottom row's edge differences go through global memory
// (L2) guarded by release/acquire progress flags.  Warps take strips from an
// atomic ticket counter in (strip-major, pair-minor) order and only ever wait
// on lower tickets, so the schedule cannot deadlock (SURVEY.md §7 hard part 2).
//
// Checkpoints written by the forward (and nothing else of the table):
//   hb[b][s][j]  h of the bottom row of strip s (the next strip's top halo),
//   vc[b][c][i]  v at column 32(c+1) (the left halo of 32-column chunk c+1).
// The backward recomputes each 32x32 tile's forward from them, turning the
// tile's softmin probabilities into E with the reverse recurrence.
#pragma once
#include "sdtw_common.cuh"

namespace sdtw {

template <class T>
struct DpArgs {
    int B, N, M, D;
    int S;       // strips  = ceil(N / 32)
    int C;       // chunks  = ceil(M / 32)
    int bw;      // Sakoe-Chiba radius, 0 = unconstrained
    int KK;      // skewed rows per strip in dsk (>= M + 31, multiple of 32)
    T k;         // log2(e) / gamma
    T gln2;      // gamma * ln(2)
    // cost sources (exactly one is used)
    const T *dsk;            // unfused: skewed costs [b][s][k][t], k in [0, KK)
    const T *x, *y;          // fused: raw series
    const T *xn, *yn;        // fused: squared norms (cost.hpp:22-56)
    // checkpoints / halos
    T *hb;                   // [B][S][M]
    T *vc;                   // [B][C][N]   (chunk c uses vc[c-1])
    T *sb;                   // [B][S][M]   backward: S of each strip's top row
    double *lpart;           // [B][S]      loss partials
    T *E;                    // [B][N][M]   alignment gradient (v1 output)
    int *flag_f;             // [B][S]      forward columns published
    int *flag_b;             // [B][S]      backward columns published (from the right)
    unsigned *tickets;       // [2]         forward / backward ticket counters
};

// Squared-Euclidean cost by the norm expansion, clamped at 0 (cost.hpp:63-78).
// One routine for the fused and unfused paths, so both are bit-identical.
template <class T>
__device__ __forceinline__ T cost_cell(const T *__restrict__ xr, const T *__restrict__ yr,
                                       T xn, T yn, int D)
{
    T dot = T(0);
    if constexpr (sizeof(T) == 4) {
        // fp32 (fused mode with D > 128): four independent partial sums
        // over 16-byte loads when rows are aligned, then (p0 + p1) + (p2 + p3)
        if ((D & 3) == 0 && ((reinterpret_cast<uintptr_t>(xr) | reinterpret_cast<uintptr_t>(yr)) & 15) == 0) {
            float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
            for (int kk = 0; kk < D; kk += 4) {
                const float4 a = __ldg(reinterpret_cast<const float4 *>(xr + kk));
                const float4 c = __ldg(reinterpret_cast<const float4 *>(yr + kk));
                p0 = fmaf(a.x, c.x, p0);
                p1 = fmaf(a.y, c.y, p1);
                p2 = fmaf(a.z, c.z, p2);
                p3 = fmaf(a.w, c.w, p3);
            }
            dot = (p0 + p1) + (p2 + p3);
        } else {
            for (int kk = 0; kk < D; ++kk) dot = fma(xr[kk], yr[kk], dot);
        }
    } else {
        for (int kk = 0; kk < D; ++kk) dot = fma(xr[kk], yr[kk], dot);
    }
    const T v = (xn - T(2) * dot) + yn;
    return v < T(0) ? T(0) : v;
}

template <class T, bool kFused>
__device__ __forceinline__ T load_cost(const DpArgs<T> &a, int b, int s, int t, int i, int j)
{
    if (kFused) {
        return cost_cell(a.x + ((size_t)b * a.N + (i - 1)) * a.D,
                         a.y + ((size_t)b * a.M + (j - 1)) * a.D,
                         a.xn[(size_t)b * a.N + (i - 1)], a.yn[(size_t)b * a.M + (j - 1)], a.D);
    } else {
        const int kk = j - 1 + t;
        return a.dsk[(((size_t)b * a.S + s) * a.KK + kk) * 32 + t];
    }
}

__device__ __forceinline__ unsigned warp_ticket(unsigned *counter)
{
    unsigned tk = 0;
    if ((threadIdx.x & 31) == 0) tk = atomicAdd(counter, 1u);
    return __shfl_sync(kFull, tk, 0);
}

// Sums strip partials in strip order (deterministic).
template <int kTU = 0>
__global__ void sdtw_loss_reduce_kernel(const double *lpart, int B, int S, float *lf,
                                        double *ld)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += lpart[(size_t)b * S + s];
    if (lf) lf[b] = (float)acc;
    if (ld) ld[b] = acc;
}

}  // namespace sdtw
