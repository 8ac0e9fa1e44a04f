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
    for (int kk = 0; kk < D; ++kk) dot = fma(xr[kk], yr[kk], dot);
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

// --------------------------------------------------------------------------
// Forward: fills nothing but the checkpoints and the loss partials.
// loss[b] = R(N,M) = R(1,1) + sum_{t=2..min} g(t,t) + straight tail
// (row N for M > N, column M for N > M), accumulated in double.
// --------------------------------------------------------------------------
template <class T, bool kFused>
__global__ void __launch_bounds__(32) sdtw_forward_kernel(DpArgs<T> a)
{
    __shared__ T halo_s[1][32];
    __shared__ T out_s[1][32];
    const int w = 0, t = threadIdx.x & 31;
    const int total = a.B * a.S;
    for (;;) {
        const unsigned tk = warp_ticket(&a.tickets[0]);
        if ((int)tk >= total) return;
        const int s = (int)tk / a.B, b = (int)tk % a.B;
        const int i = 32 * s + t + 1;
        const bool row_ok = i <= a.N;
        T h_prev = T(0), l_carry = T(0);
        double lacc = 0.0;
        T *hb_row = a.hb + ((size_t)b * a.S + s) * a.M;
        const T *hb_top = a.hb + ((size_t)b * a.S + (s - 1)) * a.M;
        const int steps = a.M + 31;
        for (int k = 0; k < steps; ++k) {
            if ((k & 31) == 0 && s > 0 && k < a.M) {
                const int need = min(k + 32, a.M);
                wait_flag_geq(&a.flag_f[b * a.S + s - 1], need);
                halo_s[w][t] = (k + t < a.M) ? hb_top[k + t] : T(0);
                __syncwarp();
            }
            const T src = (t == 31) ? halo_s[w][k & 31] : h_prev;
            const T u = __shfl_sync(kFull, src, (t + 31) & 31);
            const int j = k - t + 1;
            T h = h_prev;
            if (row_ok && j >= 1 && j <= a.M) {
                const T d = in_band(i, j, a.bw) ? load_cost<T, kFused>(a, b, s, t, i, j) : T(0);
                const Cell<T> c = dp_cell<T, false>(i, j, a.bw, d, u, l_carry, a.k, a.gln2);
                if (i == j) lacc += (double)c.g;
                if (i == a.N && j > a.N) lacc += (double)c.h;
                if (j == a.M && i > a.M) lacc += (double)c.v;
                if ((j & 31) == 0 && j < a.M)
                    a.vc[((size_t)b * a.C + (j / 32 - 1)) * a.N + (i - 1)] = c.v;
                l_carry = c.v;
                h = c.h;
                if (t == 31) out_s[w][(j - 1) & 31] = h;
            }
            h_prev = h;
            // lane 31 finished column j31 = k - 30: publish a full group
            const int j31 = k - 30;
            if (j31 >= 1 && ((j31 & 31) == 0 || j31 == a.M)) {
                __syncwarp();
                const int base = (j31 - 1) & ~31;
                if (base + t < j31) hb_row[base + t] = out_s[w][t];
                __syncwarp();
                if (t == 0) {
                    __threadfence();
                    flag_release(&a.flag_f[b * a.S + s], j31);
                }
            }
        }
        // fixed-order warp reduction: deterministic loss partial
        for (int off = 16; off > 0; off >>= 1) lacc += __shfl_xor_sync(kFull, lacc, off);
        if (t == 0) a.lpart[(size_t)b * a.S + s] = lacc;
        __syncwarp();
    }
}

// Sums strip partials in strip order (deterministic).
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

// --------------------------------------------------------------------------
// Backward: reverse strips, chunks right to left.  Per 32-column chunk:
//  phase R  recompute the tile's forward from (hb of strip s-1, vc of the
//           chunk) and keep its softmin probabilities in shared memory;
//  phase E  E(i,j) = E(i,j+1) P_l(i,j+1) + [E(i+1,j) P_u(i+1,j) +
//           E(i+1,j+1) P_d(i+1,j+1)], the bracket arriving from the lane
//           below (or from strip s+1 through sb for lane 31), capped at 1 as
//           the reference caps Ebar at 0 (backward.hpp:133-137).
// --------------------------------------------------------------------------
template <class T, bool kFused>
__global__ void __launch_bounds__(32) sdtw_backward_kernel(DpArgs<T> a)
{
    // [jj][lane] for the probabilities and [lane][jj] for E: both access
    // patterns (jj = q - t and jj = q' - t) are bank-conflict free at
    // stride 32, and E rows read out as one 128-byte line per store.
    __shared__ T pd_s[1][32][32];
    __shared__ T pu_s[1][32][32];
    __shared__ T pl_s[1][32][32];
    __shared__ T et_s[1][32][32];
    __shared__ T halo_s[1][32];
    __shared__ T sio_s[1][32];
    const int w = 0, t = threadIdx.x & 31;
    const int total = a.B * a.S;
    for (;;) {
        const unsigned tk = warp_ticket(&a.tickets[1]);
        if ((int)tk >= total) return;
        const int s = a.S - 1 - (int)tk / a.B, b = (int)tk % a.B;
        const int i = 32 * s + t + 1;
        const bool row_ok = i <= a.N;
        T e_right = T(0), pl_right = T(0), pd_right = T(0);
        for (int c = a.C - 1; c >= 0; --c) {
            const int j0 = 32 * c + 1;
            const int width = min(32, a.M - 32 * c);
            // ---- phase R: recompute the tile forward -------------------
            T l_carry = (c > 0 && row_ok) ? a.vc[((size_t)b * a.C + (c - 1)) * a.N + (i - 1)] : T(0);
            halo_s[w][t] = (s > 0 && t < width) ? a.hb[((size_t)b * a.S + (s - 1)) * a.M + (j0 - 1) + t] : T(0);
            __syncwarp();
            T h_prev = T(0);
            for (int q = 0; q < width + 31; ++q) {
                const T src = (t == 31) ? halo_s[w][q < width ? q : 0] : h_prev;
                const T u = __shfl_sync(kFull, src, (t + 31) & 31);
                const int jj = q - t;
                T h = h_prev;
                if (row_ok && jj >= 0 && jj < width) {
                    const int j = j0 + jj;
                    const T d = in_band(i, j, a.bw) ? load_cost<T, kFused>(a, b, s, t, i, j) : T(0);
                    const Cell<T> cc = dp_cell<T, true>(i, j, a.bw, d, u, l_carry, a.k, a.gln2);
                    pd_s[w][jj][t] = cc.pd;
                    pu_s[w][jj][t] = cc.pu;
                    pl_s[w][jj][t] = cc.pl;
                    l_carry = cc.v;
                    h = cc.h;
                }
                h_prev = h;
            }
            // ---- phase E: reverse sweep over the tile ------------------
            if (s < a.S - 1) {
                wait_flag_geq(&a.flag_b[b * a.S + s + 1], a.M - j0 + 1);
                sio_s[w][t] = (t < width) ? a.sb[((size_t)b * a.S + (s + 1)) * a.M + (j0 - 1) + t] : T(0);
            } else {
                sio_s[w][t] = T(0);
            }
            __syncwarp();
            T s_prev = T(0);
            for (int q = 0; q < width + 31; ++q) {
                // lane 31 handles jj = width-1-q; lane t lags by 31-t steps
                const int jj = width - 1 - q + (31 - t);
                const int jj31 = width - 1 - q;
                const T src = (t == 0) ? sio_s[w][jj31 >= 0 ? jj31 : 0] : s_prev;
                const T s_in = __shfl_sync(kFull, src, (t + 1) & 31);
                T s_out = s_prev;
                if (row_ok && jj >= 0 && jj < width) {
                    const int j = j0 + jj;
                    T e;
                    if (i == a.N && j == a.M) e = T(1);
                    else if (!in_band(i, j, a.bw)) e = T(0);
                    else {
                        e = fma(e_right, pl_right, s_in);
                        e = e < T(1) ? e : T(1);
                    }
                    const T pd = pd_s[w][jj][t], pu = pu_s[w][jj][t], pl = pl_s[w][jj][t];
                    s_out = fma(e, pu, e_right * pd_right);
                    e_right = e;
                    pl_right = pl;
                    pd_right = pd;
                    et_s[w][t][jj] = e;
                    if (t == 0) halo_s[w][jj] = s_out;
                }
                s_prev = s_out;
            }
            __syncwarp();
            // ---- outputs of the chunk ----------------------------------
            for (int r = 0; r < 32; ++r) {
                const int ir = 32 * s + r + 1;
                if (ir <= a.N && t < width)
                    a.E[((size_t)b * a.N + (ir - 1)) * a.M + (j0 - 1) + t] = et_s[w][r][t];
            }
            if (t < width) a.sb[((size_t)b * a.S + s) * a.M + (j0 - 1) + t] = halo_s[w][t];
            __syncwarp();
            if (t == 0) {
                __threadfence();
                flag_release(&a.flag_b[b * a.S + s], a.M - j0 + 1);
            }
            __syncwarp();
        }
    }
}

}  // namespace sdtw
