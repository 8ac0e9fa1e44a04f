// sdtw_dp3.cuh — third-generation wavefront DP kernels.
//
// Changes over sdtw_dp2.cuh (whose strip/super-strip scheme they keep):
//
//  * Fence-free halos.  A halo entry is the value and the call's epoch packed
//    in one 64-bit word (fp32) and written with one relaxed store; the
//    consumer polls the data itself until the epoch matches.  No release /
//    acquire pairs, no L1 invalidation on the critical path between strips
//    (the v2 profile showed ~25% of warp samples in ERRBAR / CCTL.IVALL).
//
//  * Exact zero-tile skipping in the backward.  E(i,j) = E(i,j+1) P_l +
//    E(i+1,j) P_u + E(i+1,j+1) P_d: when the E values entering a 32x32 tile
//    from the right and from below are all exactly 0 (and the tile does not
//    hold (N,M)), every E in the tile is exactly 0, so its recompute and its
//    gradient contribution are skipped with bit-identical results.  In fp32
//    the alignment gradient underflows to 0 outside a narrow band around the
//    soft path: measured 75% (gamma=1, L=256) to 98.4% (gamma=0.01, L=4096)
//    of tiles are exactly zero on N(0,1) data.
//
//  * Input gradients without the dense E: the backward queues each non-zero
//    E tile (4 KB) in a compact store, contracted in a fixed order by
//    sdtw_grad.cuh (backward.hpp:208-266).  If a capped store overflows, the
//    backward contracts the remaining tiles itself (tile_contract_fx) into
//    64-bit fixed-point accumulators (integer atomics are associative, so the
//    result is bit-identical for any schedule).  E reaches HBM only if the
//    caller asks for it.
#pragma once
#include "sdtw_common.cuh"
#include "sdtw_dp.cuh"
#include "sdtw_dp2.cuh"

namespace sdtw {

// ---- tagged halo entries ----------------------------------------------------
template <class T>
struct Tagged;

template <>
struct Tagged<float> {
    using Ent = unsigned long long;
    static __device__ __forceinline__ void store(Ent *p, float v, unsigned tag)
    {
        const Ent w = ((Ent)tag << 32) | (Ent)__float_as_uint(v);
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w));
    }
    static __device__ __forceinline__ bool load(const Ent *p, float &v, unsigned tag)
    {
        Ent w;
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p));
        v = __uint_as_float((unsigned)(w & 0xffffffffull));
        return (unsigned)(w >> 32) == tag;
    }
    static __device__ __forceinline__ float value(const Ent *p)
    {
        return __uint_as_float((unsigned)(*p & 0xffffffffull));
    }
    static __device__ __forceinline__ void store_if(Ent *p, float v, unsigned tag, bool pred)
    {
        const Ent w = ((Ent)tag << 32) | (Ent)__float_as_uint(v);
        asm volatile(
            "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.relaxed.gpu.global.b64 [%0], %1;\n\t}" ::"l"(p),
            "l"(w), "r"((int)pred)
           );
    }
    static __device__ __forceinline__ Ent load_raw(const Ent *p)
    {
        Ent w;
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p));
        return w;
    }
};

template <>
struct Tagged<double> {
    struct __align__(16) Ent {
        double v;
        unsigned long long tag;
    };
    static __device__ __forceinline__ void store(Ent *p, double v, unsigned tag)
    {
        asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(&p->v), "d"(v) : "memory");
        __threadfence();
        asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(&p->tag), "l"((unsigned long long)tag)
                     : "memory");
    }
    static __device__ __forceinline__ bool load(const Ent *p, double &v, unsigned tag)
    {
        unsigned long long t;
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(t) : "l"(&p->tag) : "memory");
        // the whole word: genuine fp64 tags have a zero high word, while fp32
        // entries and backward status words left by earlier calls carry an
        // epoch >= 1 there (the arena is shared across calls and dtypes)
        if (t != (unsigned long long)tag) return false;
        __threadfence();
        asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(&p->v) : "memory");
        return true;
    }
    static __device__ __forceinline__ double value(const Ent *p) { return p->v; }
    static __device__ __forceinline__ void store_if(Ent *p, double v, unsigned tag, bool pred)
    {
        if (pred) store(p, v, tag);
    }
};

template <class T>
struct Dp3Args {
    DpArgs<T> a;
    typename Tagged<T>::Ent *hbt;  // [B][S][M] bottom-row h of every strip (tagged)
    typename Tagged<T>::Ent *sbt;  // [B][S][M] top-row S of every strip (tagged)
    unsigned epoch;
    // Input-gradient accumulators in 64-bit fixed point: integer addition is
    // associative, so atomics from any number of tiles in any order give
    // bit-identical sums (the reference's determinism guarantee,
    // acceptance.cpp:348-377).  value = acc * 2^-fx_*.
    long long *gx_fx, *gy_fx;      // [B][N][D] sum_j E y_j,  [B][M][D] sum_i E x_i
    long long *rs_fx, *cs_fx;      // [B][N] row marginals, [B][M] column marginals
    const unsigned *absmax;        // [2 b] max|x|, [2 b + 1] max|y| of pair b (fp32 bit patterns)
    // compact store of non-zero E tiles for the contraction (sdtw_grad.cuh):
    // strip (b, s) owns slots [(b S + s) quota, +quota), filled in its
    // processing order (chunks right to left); tiles past the quota are
    // contracted by the backward itself into the fixed-point accumulators
    T *tiles;                      // [B S quota][32][32]
    int4 *tile_meta;               // [B S quota] (b, s, c, width)
    int *strip_tiles;              // [B S] tiles stored per strip
    int tile_quota;
    unsigned *stats;               // [0] live tiles, [1] tiles stored, [2] overflow (in-warp),
                                   // [3] band miss (fused band cache, below)
    unsigned long long *trace;     // optional [B*S][2] %globaltimer at strip start / end (forward)
    // Fused-mode band cache (fp32, tensor-core fused forward): the forward
    // keeps, per strip, the skewed cost row groups [band_lo, band_lo +
    // band_ng) around the strip's diagonal (the groups of tiles [-W, W + 2]
    // from the diagonal, band_ng = 2 W + 4: the backward's speculative
    // recompute reaches two tiles further right, sdtw_dp4.cuh COMMIT), so the
    // backward reads them like
    // the unfused cost tensor instead of recomputing them on the tensor
    // cores.  A backward tile outside the band sets stats[3]; the tensor-core
    // backward then reruns the call (band_gate launches exit unless it is
    // set), so results never depend on the band's width.
    int spec_right;                // sdtw_dp4.cuh: verdict-free sweeps up to this many chunks right of the diagonal
    T *band;                       // [B][S][band_ng][32][32] skewed groups, or null
    int band_ng;
    int band_gate;                 // 1: run only if stats[3] != 0
};

// First cached group of strip s (shared by the forward that fills the band
// cache and the backward that reads it): the diagonal's chunk at the strip's
// middle row, W = ng / 2 - 2 groups to the left, clamped into [0, G - ng].
// the diagonal's chunk at strip s's middle row
__host__ __device__ __forceinline__ int diag_chunk(int s, int N, int M)
{
    const long long mid = 32LL * s + 16;
    return (int)((mid * M / (N > 0 ? N : 1)) >> 5);
}
__host__ __device__ __forceinline__ int band_lo(int s, int N, int M, int G, int ng)
{
    const int cd = diag_chunk(s, N, M);
    const int lo = cd - (ng / 2 - 2);
    const int hi = G - ng > 0 ? G - ng : 0;
    return lo < 0 ? 0 : (lo > hi ? hi : lo);
}

__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Fixed-point exponents: |sum_j E_ij y_jk| <= M max|y| (E <= 1), etc.
struct FxScales {
    double gx, gy, rs, cs;  // multipliers (2^e)
};
__device__ __forceinline__ double fx_pow2_for(double bound)
{
    int e;
    frexp(bound > 1e-300 ? bound : 1e-300, &e);  // bound < 2^e
    return ldexp(1.0, 61 - e);
}
__device__ __forceinline__ FxScales fx_scales(const unsigned *absmax, int N, int M)
{
    const double mx = (double)__uint_as_float(absmax[0]), my = (double)__uint_as_float(absmax[1]);
    FxScales f;
    f.gx = fx_pow2_for(4.0 * M * my + 1e-30);
    f.gy = fx_pow2_for(4.0 * N * mx + 1e-30);
    f.rs = fx_pow2_for(4.0 * M);
    f.cs = fx_pow2_for(4.0 * N);
    return f;
}
__device__ __forceinline__ void fx_add(long long *p, double v, double scale)
{
    const long long q = __double2ll_rn(v * scale);
    if (q != 0) atomicAdd(reinterpret_cast<unsigned long long *>(p), (unsigned long long)q);
}

// Per-pair absolute maxima for the fixed-point scales (float and double):
// pair b = blockIdx.y, n elements per pair, into out[2 b + which].
template <class T>
__global__ void absmax_any_kernel(const T *__restrict__ v, size_t n, unsigned *out, int which)
{
    const T *p = v + (size_t)blockIdx.y * n;
    float m = 0.f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmaxf(m, (float)fabs((double)p[i]));
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out + 2 * blockIdx.y + which, __float_as_uint(m) + 1u);  // round up
}

// Spins until `n` consecutive tagged entries starting at p carry `tag`; lane t
// (< n) returns entry t's value.
#ifndef POLL_SLEEP_NS
#define POLL_SLEEP_NS 0  // measured: a tight spin shortens the strip hand-off (C2 fwd -10%)
#endif
template <class T>
__device__ __forceinline__ T poll_entries(const typename Tagged<T>::Ent *p, int n, unsigned tag, int lane)
{
    T v = T(0);
    bool ok = lane >= n || Tagged<T>::load(p + lane, v, tag);
    unsigned polls = 0;
    while (!__all_sync(kFull, ok)) {
        if (!ok) {
            if (POLL_SLEEP_NS > 0) __nanosleep(POLL_SLEEP_NS);
            ok = Tagged<T>::load(p + lane, v, tag);
        }
        if (++polls > (1u << 26)) {
            if (lane == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
            break;
        }
    }
    return v;
}

// --------------------------------------------------------------------------
// Forward v3
// --------------------------------------------------------------------------
template <class T, int K, bool kFused>
__global__ void __launch_bounds__(128) sdtw_forward3_kernel(Dp3Args<T> A)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const DpArgs<T> &a = A.a;
    using SM = Fwd2Smem<T, K, kFused>;
    using TG = Tagged<T>;
    const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
    T *ring = reinterpret_cast<T *>(smem_raw) + w * SM::kPerWarp;
    T *halo_s = ring + SM::kRing;
    const int SS = (a.S + K - 1) / K;
    const int total = a.B * SS;
    const T inf = Num<T>::inf();
    const unsigned epoch = A.epoch;
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
        const int qlast = min(K, a.S - s0) - 1;
        if (A.trace && t == 0) A.trace[2 * ((size_t)b * a.S + s0)] = global_ns();
        double lacc = 0.0;  // tail terms (slow path only)
        T gdiag[K];         // this lane's diagonal cell g (at most one per strip)
        int kdiag[K];       // step at which lane t of strip q meets i == j
#pragma unroll
        for (int q = 0; q < K; ++q) {
            gdiag[q] = T(0);
            kdiag[q] = 32 * s0 + 64 * q + 2 * t;
        }
        const typename TG::Ent *hb_top = A.hbt + ((size_t)b * a.S + (s0 - 1)) * a.M;
        const int ngroups_row = a.KK / 32;
        const int steps = a.M + 32 * qlast + 31;
        // A group is "plain" when every cell it touches is interior: no row 1,
        // no column 1, no tail cell (row N with M > N, column M with N > M),
        // and fully in band.  Plain and fill/drain groups share one
        // branch-free step body; only boundary / tail / band fix-ups differ.
        // lane 0 of a pair's first strip is row 1 (R(0, j) = inf): three
        // selects in every step instead of the fix-up path for the whole strip
        const bool r1 = s0 == 0 && t == 0;
        const bool has_rowN = 32 * (s0 + qlast + 1) >= a.N;
        const bool strip_full = 32 * (s0 + qlast + 1) <= a.N;  // every lane's row exists
        unsigned long long pf_w = 0;  // prefetched halo entry (lanes 0..7)
        int pf_kb = -1;
        if (!kFused) {
            load_group(ring, dsrc[0], t);
            cp_async_commit();
        }
        for (int k0 = 0; k0 < steps; k0 += 32) {
            const int G = k0 >> 5;
            __syncwarp();
            if (!kFused) {
#pragma unroll
                for (int q = 0; q < K; ++q) {
                    const int g = G + 1 - q;
                    if (q <= qlast && g >= 0 && g < ngroups_row)
                        load_group(ring + (q * 2 + (g & 1)) * 1024, dsrc[q] + (size_t)g * 1024, t);
                }
                cp_async_commit();
                cp_async_wait<1>();
                __syncwarp();
            }
            // columns touched by this group (0-based): [k0 - 32 qlast - 31, k0 + 31]
            const int cmin = k0 - 32 * qlast - 31, cmax = k0 + 31;
            const bool fixup = cmin <= 0 ||
                               (a.bw != 0 && (32 * s0 - k0 - 31 < -a.bw || 32 * s0 + 64 * qlast + 62 - k0 > a.bw));
            const bool tail = (has_rowN && a.M > a.N && cmax >= a.N) || (a.N > a.M && cmax >= a.M - 1);
            T vck[K];
#pragma unroll
            for (int q = 0; q < K; ++q) vck[q] = T(0);
#pragma unroll 1
            for (int k8 = 0; k8 < 32; k8 += 8) {
                const int kb = k0 + k8;
                // top halo for columns [kb, kb + 8): polled as data (no flags),
                // the next sub-group prefetched
                if (s0 > 0 && kb < a.M) {
                    const int n = min(8, a.M - kb);
                    T hv = T(0);
                    if constexpr (sizeof(T) == 4) {
                        bool ok = t >= n;
                        if (!ok) {
                            unsigned long long w8 = (pf_kb == kb) ? pf_w : TG::load_raw(hb_top + kb + t);
                            ok = (unsigned)(w8 >> 32) == epoch;
                            hv = __uint_as_float((unsigned)(w8 & 0xffffffffull));
                        }
                        if (!__all_sync(kFull, ok)) hv = poll_entries<T>(hb_top + kb, n, epoch, t);
                        const int kb2 = kb + 8;
                        if (kb2 < a.M && t < min(8, a.M - kb2)) {
                            pf_w = TG::load_raw(hb_top + kb2 + t);
                            pf_kb = kb2;
                        }
                    } else {
                        hv = poll_entries<T>(hb_top + kb, n, epoch, t);
                    }
                    if (t < n) halo_s[(kb + t) & 31] = hv;
                    __syncwarp();
                }
                // fused mode: the sub-group's costs up front, 8 independent
                // SIMT dot products per strip (they do not depend on the DP
                // state, so they leave the step chain; same values)
                T dk[K][8];
                if constexpr (kFused && K == 1) {
                    // staged feature blocks (fused_costs_staged, sdtw_dp2.cuh)
                    T d8[8];
                    fused_costs_staged<T>(a, b, s0, t, kb, halo_s + SM::kHalo, d8);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int col = kb + kk - t;
                        dk[0][kk] = (row_ok[0] && col >= 0 && col < a.M) ? d8[kk] : T(0);
                    }
                } else if (kFused) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                        for (int q = 0; q < K; ++q) {
                            const int col = kb + kk - 32 * q - t;
                            const bool active = row_ok[q] && col >= 0 && col < a.M;
                            dk[q][kk] = active ? load_cost<T, true>(a, b, s0 + q, t, row[q], col + 1) : T(0);
                        }
                }
                // Lean sub-group (one strip per warp, unfused): every lane's
                // cell is interior and active (col in [1, M), full strip),
                // not strip 0 (no row-1 selects) and no lane meets its
                // diagonal cell here (no loss capture), so the step is the
                // cell, the chunk-boundary capture and lane 31's store at an
                // immediate offset: ~12 fewer instructions per step than the
                // plain body below (same arithmetic, same results).
                const bool lean = K == 1 && !kFused && !fixup && !tail && s0 > 0 && strip_full &&
                                  kb >= 31 && kb + 7 < a.M && (kb + 7 < 32 * s0 || kb > 32 * s0 + 62);
                if (lean) {
                    const T *rgk = ring + (G & 1) * 1024 + k8 * 32 + t;
                    typename TG::Ent *hp = A.hbt + ((size_t)b * a.S + s0) * a.M + (kb - 31);
                    // lane 31's h leave after the sub-group (the strip below
                    // consumes 8 columns at a time: no added lag)
                    T hb[8];
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int kl = k8 + kk;
                        const T src = (t == 31) ? halo_s[kl] : h_prev[0];
                        const T u = __shfl_sync(kFull, src, (t + 31) & 31);
                        const T d = rgk[kk * 32];
                        T g, v, h;
                        fwd_cell<T>(d, u, l_carry[0], a.k, a.gln2, g, v, h);
                        vck[0] = (kl == ((t - 1) & 31)) ? v : vck[0];
                        l_carry[0] = v;
                        h_prev[0] = h;
                        hb[kk] = h;
                    }
                    if (t == 31) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) TG::store(hp + kk, hb[kk], epoch);
                    }
                    __syncwarp();
                } else if (fixup || tail) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int k = kb + kk;
                        const int kl = k8 + kk;  // step within the group
                        T src[K], u[K];
                        const T hs = halo_s[kl];
    #pragma unroll
                        for (int q = 0; q < K; ++q) src[q] = (t == 31) ? (q == 0 ? hs : h_prev[q - 1]) : h_prev[q];
    #pragma unroll
                        for (int q = 0; q < K; ++q) u[q] = __shfl_sync(kFull, src[q], (t + 31) & 31);
    #pragma unroll
                        for (int q = 0; q < K; ++q) {
                            const int col = k - 32 * q - t;  // 0-based column of this lane's cell
                            const bool active = row_ok[q] && col >= 0 && col < a.M;
                            T d;
                            if (kFused) {
                                d = dk[q][kk];
                            } else {
                                d = ring[(q * 2 + ((G - q) & 1)) * 1024 + kl * 32 + t];
                            }
                            T g, v, h;
                            fwd_cell<T>(d, u[q], l_carry[q], a.k, a.gln2, g, v, h);
                            if (q == 0) {
                                g = r1 ? d : g;
                                v = r1 ? -inf : v;
                                h = r1 ? d : h;
                            }
                            if (fixup) {  // warp-uniform: boundary row / column, band
                                const bool j1 = col == 0, r1 = row[q] == 1;
                                g = (j1 || r1) ? d : g;
                                v = r1 ? -inf : (j1 ? d : v);
                                h = j1 ? -inf : (r1 ? d : h);
                                if (a.bw != 0 && !in_band(row[q], col + 1, a.bw)) {
                                    g = inf; v = inf; h = inf;
                                }
                            }
                            if (tail && active) {  // warp-uniform branch, rare
                                const int i = row[q], j = col + 1;
                                if (i == a.N && j > a.N) lacc += (double)h;
                                if (j == a.M && i > a.M) lacc += (double)v;
                            }
                            gdiag[q] = (active && k == kdiag[q]) ? g : gdiag[q];
                            vck[q] = (kl == ((t - 1) & 31)) ? v : vck[q];
                            l_carry[q] = v;
                            h_prev[q] = h;
                            // lane 31: bottom row of the strip (predicated, no divergence)
                            TG::store_if(A.hbt + ((size_t)b * a.S + (s0 + q)) * a.M + col, h, epoch, t == 31 && active);
                        }
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int k = kb + kk;
                        const int kl = k8 + kk;  // step within the group
                        T src[K], u[K];
                        const T hs = halo_s[kl];
    #pragma unroll
                        for (int q = 0; q < K; ++q) src[q] = (t == 31) ? (q == 0 ? hs : h_prev[q - 1]) : h_prev[q];
    #pragma unroll
                        for (int q = 0; q < K; ++q) u[q] = __shfl_sync(kFull, src[q], (t + 31) & 31);
    #pragma unroll
                        for (int q = 0; q < K; ++q) {
                            const int col = k - 32 * q - t;  // 0-based column of this lane's cell
                            const bool active = row_ok[q] && col >= 0 && col < a.M;
                            T d;
                            if (kFused) {
                                d = dk[q][kk];
                            } else {
                                d = ring[(q * 2 + ((G - q) & 1)) * 1024 + kl * 32 + t];
                            }
                            T g, v, h;
                            fwd_cell<T>(d, u[q], l_carry[q], a.k, a.gln2, g, v, h);
                            if (q == 0) {
                                g = r1 ? d : g;
                                v = r1 ? -inf : v;
                                h = r1 ? d : h;
                            }
                            gdiag[q] = (active && k == kdiag[q]) ? g : gdiag[q];
                            vck[q] = (kl == ((t - 1) & 31)) ? v : vck[q];
                            l_carry[q] = v;
                            h_prev[q] = h;
                            // lane 31: bottom row of the strip (predicated, no divergence)
                            TG::store_if(A.hbt + ((size_t)b * a.S + (s0 + q)) * a.M + col, h, epoch, t == 31 && active);
                        }
                    }
                }
            }
            // chunk-boundary v captured in registers: lanes 1..31 hold column
            // 32 (G - q) (1-based), lane 0 the next boundary
#pragma unroll
            for (int q = 0; q < K; ++q) {
                const int bidx = (t == 0) ? (G - q) : (G - q - 1);
                const int jb = 32 * (bidx + 1);
                if (bidx >= 0 && jb < a.M && row_ok[q]) a.vc[((size_t)b * a.C + bidx) * a.N + (row[q] - 1)] = vck[q];
            }
        }
#pragma unroll
        for (int q = 0; q < K; ++q) lacc += (double)gdiag[q];
        if (A.trace && t == 0) A.trace[2 * ((size_t)b * a.S + s0) + 1] = global_ns();
        if (!kFused) cp_async_wait<0>();
        for (int off = 16; off > 0; off >>= 1) lacc += __shfl_xor_sync(kFull, lacc, off);
        if (t == 0) {
            a.lpart[(size_t)b * a.S + s0] = lacc;
            for (int q = 1; q <= qlast; ++q) a.lpart[(size_t)b * a.S + s0 + q] = 0.0;
        }
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// Gradient contraction of the backward's non-zero E tiles
// --------------------------------------------------------------------------
// Contraction of one non-zero E tile (32 x 32, [r][jj] in shared memory):
//   gx[i0+r][k] += sum_jj E[r][jj] y[j0+jj][k],  gy[j0+jj][k] += sum_r E[r][jj] x[i0+r][k]
// plus both marginals, into the fixed-point accumulators.  One warp; lane =
// row (X pass) or column (Y pass); the y / x rows come through `stage`
// (32 rows x 32 features per round, 4 KB of T).
template <class T>
__device__ __forceinline__ void tile_contract_fx(const Dp3Args<T> &A, const FxScales &fx, int b, int s, int c,
                                                 int width, const T *et_s, T *stage, int t, int es = 32)
{
    const DpArgs<T> &a = A.a;
    const int i0 = 32 * s, j0 = 32 * c;  // 0-based
    const int D = a.D;
    const int rows = min(32, a.N - i0);
    T rs = T(0), cs = T(0);
    for (int jj = 0; jj < width; ++jj) rs += et_s[t * es + jj];
    for (int r = 0; r < rows; ++r) cs += et_s[r * es + t];
    if (t < rows) fx_add(A.rs_fx + (size_t)b * a.N + i0 + t, (double)rs, fx.rs);
    if (t < width) fx_add(A.cs_fx + (size_t)b * a.M + j0 + t, (double)cs, fx.cs);
    for (int pass = 0; pass < 2; ++pass) {
        // pass 0: lane = row r, sum over columns jj of E[r][jj] * y[j0+jj]
        // pass 1: lane = column jj, sum over rows r of E[r][jj] * x[i0+r]
        const T *src = pass == 0 ? a.y + ((size_t)b * a.M + j0) * D : a.x + ((size_t)b * a.N + i0) * D;
        const int nsrc = pass == 0 ? width : rows;
        const int nown = pass == 0 ? rows : width;
        for (int k0 = 0; k0 < D; k0 += 32) {
            const int kn = min(32, D - k0);
            __syncwarp();
            for (int r = 0; r < 32; ++r)  // stage[r][kk] = src[r][k0 + kk]
                stage[r * 33 + t] = (r < nsrc && t < kn) ? src[(size_t)r * D + k0 + t] : T(0);
            __syncwarp();
            T acc[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) acc[q] = T(0);
            for (int m = 0; m < nsrc; ++m) {
                const T e = pass == 0 ? et_s[t * es + m] : et_s[m * es + t];
#pragma unroll
                for (int q = 0; q < 32; ++q) acc[q] = fma(e, stage[m * 33 + q], acc[q]);
            }
            if (t < nown) {
                long long *dst = pass == 0 ? A.gx_fx + ((size_t)b * a.N + i0 + t) * D + k0
                                           : A.gy_fx + ((size_t)b * a.M + j0 + t) * D + k0;
                const double sc = pass == 0 ? fx.gx : fx.gy;
#pragma unroll
                for (int q = 0; q < 32; ++q)
                    if (q < kn) fx_add(dst + q, (double)acc[q], sc);
            }
        }
    }
}

}  // namespace sdtw
