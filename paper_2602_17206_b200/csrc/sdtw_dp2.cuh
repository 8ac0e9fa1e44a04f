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

template <class T>
__device__ __forceinline__ void fwd_cell(T d, T u, T l, T k, T gln2, T &g, T &v, T &h)
{
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

template <class T, int K, bool kFused>
__global__ void __launch_bounds__(128) sdtw_forward2_kernel(DpArgs<T> a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using SM = Fwd2Smem<T, K, kFused>;
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
    T *ring = reinterpret_cast<T *>(smem_raw) + w * SM::kPerWarp;
    T *halo_s = ring + SM::kRing;
    const int SS = (a.S + K - 1) / K;
    const int total = a.B * SS;
    const T inf = Num<T>::inf();
    for (;;) {
        const unsigned tk = warp_ticket(&a.tickets[0]);
        if ((int)tk >= total) return;
        const int ss = (int)tk / a.B, b = (int)tk % a.B;
        const int s0 = ss * K;
        int row[K];
        bool row_ok[K];
        T h_prev[K], l_carry[K];
        const T *dsrc[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
            row[q] = 32 * (s0 + q) + t + 1;
            row_ok[q] = (s0 + q < a.S) && row[q] <= a.N;
            h_prev[q] = T(0);
            l_carry[q] = T(0);
            dsrc[q] = kFused ? nullptr : a.dsk + ((size_t)b * a.S + min(s0 + q, a.S - 1)) * (size_t)a.KK * 32;
        }
        const int qlast = min(K, a.S - s0) - 1;  // last real strip of this super-strip
        double lacc = 0.0;
        const T *hb_top = a.hb + ((size_t)b * a.S + (s0 - 1)) * a.M;
        const int *flag_top = a.flag_f + b * a.S + (s0 - 1);
        int *flag_out = a.flag_f + b * a.S + (s0 + qlast);
        const int ngroups_row = a.KK / 32;
        const int steps = a.M + 32 * qlast + 31;
        // prologue: strip 0, row group 0
        if (!kFused) {
            load_group(ring, dsrc[0], t);
            cp_async_commit();
        }
        for (int k0 = 0; k0 < steps; k0 += 32) {
            const int G = k0 >> 5;
            __syncwarp();  // every lane is done with the ring slots refilled below
            if (!kFused) {
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const int g = G + 1 - q;
                    if (q <= qlast && g >= 0 && g < ngroups_row)
                        load_group(ring + (q * 2 + (g & 1)) * 1024, dsrc[q] + (size_t)g * 1024, t);
                }
                cp_async_commit();
                cp_async_wait<1>();
            }
            // top halo of this group's columns [k0, k0 + 32)
            if (s0 > 0 && k0 < a.M) {
                wait_flag_geq(flag_top, min(k0 + 32, a.M));
                halo_s[t] = (k0 + t < a.M) ? hb_top[k0 + t] : T(0);
            }
            __syncwarp();
#pragma unroll 4
            for (int kk = 0; kk < 32; ++kk) {
                const int k = k0 + kk;
                T src[K], u[K];
#pragma unroll
                for (int q = 0; q < K; ++q)
                    src[q] = (t == 31) ? (q == 0 ? halo_s[kk] : h_prev[q - 1]) : h_prev[q];
#pragma unroll
                for (int q = 0; q < K; ++q) u[q] = __shfl_sync(kFull, src[q], (t + 31) & 31);
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const int kq = k - 32 * q;
                    const int col = kq - t;  // 0-based column
                    const int i = row[q], j = col + 1;
                    if (!(row_ok[q] && col >= 0 && col < a.M)) continue;
                    T d;
                    if (kFused) {
                        d = load_cost<T, true>(a, b, s0 + q, t, i, j);
                    } else {
                        d = ring[(q * 2 + ((kq >> 5) & 1)) * 1024 + (kq & 31) * 32 + t];
                    }
                    T g, v, h;
                    if (i > 1 && j > 1 && in_band(i, j, a.bw)) {
                        fwd_cell<T>(d, u[q], l_carry[q], a.k, a.gln2, g, v, h);
                    } else if (!in_band(i, j, a.bw)) {
                        g = inf; v = inf; h = inf;
                    } else if (i == 1 && j == 1) {
                        g = d; v = -inf; h = -inf;
                    } else if (i == 1) {
                        g = d; h = d; v = -inf;
                    } else {
                        g = d; v = d; h = -inf;
                    }
                    if (i == j) lacc += (double)g;
                    if (i == a.N && j > a.N) lacc += (double)h;
                    if (j == a.M && i > a.M) lacc += (double)v;
                    if ((j & 31) == 0 && j < a.M) a.vc[((size_t)b * a.C + (j / 32 - 1)) * a.N + (i - 1)] = v;
                    l_carry[q] = v;
                    h_prev[q] = h;
                    if (t == 31) {
                        // bottom row of every strip: the backward's top halo; the
                        // super-strip's last one is also the next warp's input
                        a.hb[((size_t)b * a.S + (s0 + q)) * a.M + col] = h;
                        if (q == qlast && (((j & 7) == 0) || j == a.M)) flag_release(flag_out, j);
                    }
                }
            }
        }
        if (!kFused) cp_async_wait<0>();
        for (int off = 16; off > 0; off >>= 1) lacc += __shfl_xor_sync(kFull, lacc, off);
        if (t == 0) {
            // partials are indexed per strip; the super-strip's sum goes to its first strip
            a.lpart[(size_t)b * a.S + s0] = lacc;
            for (int q = 1; q <= qlast; ++q) a.lpart[(size_t)b * a.S + s0 + q] = 0.0;
        }
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// Backward v2: per warp one strip, chunks right to left; per chunk phase R
// (recompute the 32x32 tile's forward, probabilities to shared memory) then
// phase E (reverse sweep).  Costs of the chunk's two skewed row groups come
// from a 3-slot cp.async ring (group c-1 prefetched while chunk c runs).
// --------------------------------------------------------------------------
template <class T, bool kFused>
struct Bwd2Smem {
    static constexpr int kP = 3 * 32 * 32;               // pd, pu, pl [jj][t]
    static constexpr int kE = 32 * 32;                   // E tile [t][jj]
    static constexpr int kRing = kFused ? 0 : 3 * 1024;  // skewed cost row groups
    static constexpr int kHalo = 2 * 32;                 // top halo, S from below
    static constexpr int kPerWarp = kP + kE + kRing + kHalo;
};

template <class T, bool kFused>
__global__ void __launch_bounds__(128) sdtw_backward2_kernel(DpArgs<T> a)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    using SM = Bwd2Smem<T, kFused>;
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
    T *base = reinterpret_cast<T *>(smem_raw) + w * SM::kPerWarp;
    T *pd_s = base, *pu_s = base + 1024, *pl_s = base + 2048;
    T *et_s = base + SM::kP;
    T *ring = et_s + SM::kE;
    T *halo_s = ring + SM::kRing;
    T *sio_s = halo_s + 32;
    const int total = a.B * a.S;
    for (;;) {
        const unsigned tk = warp_ticket(&a.tickets[1]);
        if ((int)tk >= total) return;
        const int s = a.S - 1 - (int)tk / a.B, b = (int)tk % a.B;
        const int i = 32 * s + t + 1;
        const bool row_ok = i <= a.N;
        const T *dsrc = kFused ? nullptr : a.dsk + ((size_t)b * a.S + s) * (size_t)a.KK * 32;
        const int ngroups_row = a.KK / 32;
        T e_right = T(0), pl_right = T(0), pd_right = T(0);
        // prologue: groups C-1 and C of the last chunk
        if (!kFused) {
            for (int g = a.C - 1; g <= a.C; ++g)
                if (g < ngroups_row) load_group(ring + (g % 3) * 1024, dsrc + (size_t)g * 1024, t);
            cp_async_commit();
        }
        for (int c = a.C - 1; c >= 0; --c) {
            const int j0 = 32 * c + 1;
            const int width = min(32, a.M - 32 * c);
            if (!kFused) {
                if (c > 0) load_group(ring + ((c - 1) % 3) * 1024, dsrc + (size_t)(c - 1) * 1024, t);
                cp_async_commit();
                cp_async_wait<1>();
            }
            T l_carry = (c > 0 && row_ok) ? a.vc[((size_t)b * a.C + (c - 1)) * a.N + (i - 1)] : T(0);
            halo_s[t] = (s > 0 && t < width) ? a.hb[((size_t)b * a.S + (s - 1)) * a.M + (j0 - 1) + t] : T(0);
            __syncwarp();
            // ---- phase R ----
            T h_prev = T(0);
            for (int q = 0; q < width + 31; ++q) {
                const T src = (t == 31) ? halo_s[q < width ? q : 0] : h_prev;
                const T u = __shfl_sync(kFull, src, (t + 31) & 31);
                const int jj = q - t;
                T h = h_prev;
                if (row_ok && jj >= 0 && jj < width) {
                    const int j = j0 + jj;
                    T d;
                    if (kFused) {
                        d = in_band(i, j, a.bw) ? load_cost<T, true>(a, b, s, t, i, j) : T(0);
                    } else {
                        const int kk = 32 * c + q;  // skewed row of (i, j)
                        d = ring[((kk >> 5) % 3) * 1024 + (kk & 31) * 32 + t];
                    }
                    const Cell<T> cc = dp_cell<T, true>(i, j, a.bw, d, u, l_carry, a.k, a.gln2);
                    pd_s[jj * 32 + t] = cc.pd;
                    pu_s[jj * 32 + t] = cc.pu;
                    pl_s[jj * 32 + t] = cc.pl;
                    l_carry = cc.v;
                    h = cc.h;
                }
                h_prev = h;
            }
            // ---- phase E ----
            if (s < a.S - 1) {
                wait_flag_geq(&a.flag_b[b * a.S + s + 1], a.M - j0 + 1);
                sio_s[t] = (t < width) ? a.sb[((size_t)b * a.S + (s + 1)) * a.M + (j0 - 1) + t] : T(0);
            } else {
                sio_s[t] = T(0);
            }
            __syncwarp();
            T s_prev = T(0);
            for (int q = 0; q < width + 31; ++q) {
                const int jj = width - 1 - q + (31 - t);
                const int jj31 = width - 1 - q;
                const T src = (t == 0) ? sio_s[jj31 >= 0 ? jj31 : 0] : s_prev;
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
                    const T pd = pd_s[jj * 32 + t], pu = pu_s[jj * 32 + t], pl = pl_s[jj * 32 + t];
                    s_out = fma(e, pu, e_right * pd_right);
                    e_right = e;
                    pl_right = pl;
                    pd_right = pd;
                    et_s[t * 32 + jj] = e;
                    if (t == 0) halo_s[jj] = s_out;
                }
                s_prev = s_out;
            }
            __syncwarp();
            for (int r = 0; r < 32; ++r) {
                const int ir = 32 * s + r + 1;
                if (ir <= a.N && t < width) a.E[((size_t)b * a.N + (ir - 1)) * a.M + (j0 - 1) + t] = et_s[r * 32 + t];
            }
            if (t < width) a.sb[((size_t)b * a.S + s) * a.M + (j0 - 1) + t] = halo_s[t];
            __syncwarp();
            if (t == 0) {
                __threadfence();
                flag_release(&a.flag_b[b * a.S + s], a.M - j0 + 1);
            }
            __syncwarp();
        }
        if (!kFused) cp_async_wait<0>();
    }
}

}  // namespace sdtw
