// sdtw_grad.cuh — input gradients from the backward's non-zero E tiles,
// deterministic and atomic-free.
//
// Reference: input_gradients (backward.hpp:208-266):
//   dX_i = 2 (x_i sum_j E_ij - sum_j E_ij y_j),  dY_j = 2 (y_j sum_i E_ij - sum_i E_ij x_i).
// The backward stores every non-zero 32 x 32 E tile of strip (b, s) in that
// strip's slots of the tile store, in its own processing order, so the dX
// bucket of a strip is simply its slot range; the dY buckets (per chunk)
// come from a counting sort, each bucket sorted by strip.  One CTA per bucket
// contracts its tiles in that fixed order (fp32 dot products, fp64
// marginals): the result is bit-identical run to run (the reference's
// determinism guarantee, acceptance.cpp:348-377) without atomics.  Tiles past
// a strip's quota (only when the store is capped) were contracted by the
// backward itself into 64-bit fixed-point accumulators (deterministic too)
// and are added by finalize_grads_fx_add_kernel.
#pragma once
#include "sdtw_common.cuh"
#include "sdtw_dp3.cuh"

namespace sdtw {

// Chunk buckets: count the stored tiles of each (b, c).
template <int kTU = 0>
__global__ void tile_hist_kernel(const int4 *__restrict__ meta, const int *__restrict__ strip_tiles, int quota,
                                 int nstrips, int C, int *cnt_c)
{
    const size_t n = (size_t)nstrips * quota;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if ((int)(i % quota) >= strip_tiles[i / quota]) continue;
        const int4 m = meta[i];
        atomicAdd(cnt_c + m.x * C + m.z, 1);
    }
}

// Exclusive scan of cnt[0..n) into off[0..n] (one block).
template <int kTU = 0>
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const int *__restrict__ cnt, int n, int *__restrict__ off)
{
    __shared__ int warp_sums[32];
    __shared__ int carry;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + tid;
        const int v = i < n ? cnt[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            int s = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const int excl = carry + (w > 0 ? warp_sums[w - 1] : 0) + x - v;
        if (i < n) off[i] = excl;
        __syncthreads();
        if (tid == 1023) carry = excl + v;
        __syncthreads();
    }
    if (tid == 0) off[n] = carry;
}

// Bucket fill: cnt is consumed (counted down), so positions are unique;
// the order inside a bucket is fixed afterwards by segment_sort_kernel.
template <int kTU = 0>
__global__ void tile_scatter_kernel(const int4 *__restrict__ meta, const int *__restrict__ strip_tiles, int quota,
                                    int nstrips, int C, const int *__restrict__ off_c, int *cnt_c, int *ord_c)
{
    const size_t n = (size_t)nstrips * quota;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        if ((int)(i % quota) >= strip_tiles[i / quota]) continue;
        const int4 m = meta[i];
        const int kc = m.x * C + m.z;
        ord_c[off_c[kc] + atomicSub(cnt_c + kc, 1) - 1] = (int)i;
    }
}

// Insertion sort of each chunk bucket by strip (meta.y).
template <int kTU = 0>
__global__ void segment_sort_kernel(const int *__restrict__ off, int *ord, const int4 *__restrict__ meta, int nseg)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nseg; k += gridDim.x * blockDim.x) {
        const int lo = off[k], hi = off[k + 1];
        for (int a = lo + 1; a < hi; ++a) {
            const int v = ord[a];
            const int kv = meta[v].y;
            int p = a - 1;
            while (p >= lo && meta[ord[p]].y > kv) {
                ord[p + 1] = ord[p];
                --p;
            }
            ord[p + 1] = v;
        }
    }
}

// One CTA per bucket (strip b,s for which = 0; chunk b,c for which = 1):
//   acc[o][k] = sum over the bucket's tiles (fixed order) of sum_m E_o,m p_m,k
//   marg[o]   = sum over tiles of sum_m E_o,m
//   grad[o][k] = 2 (v[o][k] marg[o] - acc[o][k])
// o = output row (strip row / chunk column), m = partner index (chunk column /
// strip row), p = partner rows (y chunk / x strip).  Buckets: which = 0: the
// strip's own slots [key quota, + strip_tiles[key]); which = 1: ord[off[key]
// .. off[key + 1]).  256 threads, each a 4 (o) x 4 (k) register block of a
// 32 x 128 feature block: per partner index one 16-byte shared load of E and
// one of p feed 16 FMAs.  Dot products accumulate in fp32 (fixed order), the
// marginals and the final 2 (v marg - acc) in fp64.
// strips per pair the in-kernel chunk bucketing handles (static shared memory)
template <class T>
constexpr int max_list_strips() { return sizeof(T) == 4 ? 2048 : 256; }

#ifndef CONTRACT_MIN_BLOCKS
#define CONTRACT_MIN_BLOCKS 3
#endif
// KW = feature-block width: 128, or 64 when D <= 64 (C5: D = 64), so that no
// thread multiplies zero padding; each thread holds a RA (o) x 4 (k) block,
// RA = KW / 32.  The per-element fp32 accumulation order (tiles in order,
// partners in order) is the same for both widths.
template <class T, int KW>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? CONTRACT_MIN_BLOCKS : 1)
    contract_ordered_kernel(const T *__restrict__ tiles, const int4 *__restrict__ meta,
                            const int *__restrict__ strip_tiles, int quota, const int *__restrict__ off,
                            const int *__restrict__ ord, int which, int B, int S, int C, int N, int M, int D,
                            const T *__restrict__ vout, const T *__restrict__ vpart, T *__restrict__ grad)
{
    constexpr int RA = KW / 32;          // output rows per thread
    constexpr int KG = KW / 4;           // feature groups of 4
    constexpr int NP = 32 * KW / 256;    // partner values staged per thread per tile
    __shared__ __align__(16) T Et[32][36];   // [m][o]
    __shared__ __align__(16) T P[32][132];   // [m][k]
    __shared__ double marg_s[32];
    // which = 1 without a global bucket sort (ord == nullptr, S <= list size):
    // the chunk's tiles in strip order, found by scanning the strips' own
    // tile lists (each strip holds at most one tile of a chunk)
    __shared__ int lst[max_list_strips<T>()];
    __shared__ int wcnt[8];
    const int tid = threadIdx.x;
    const int og = tid / KG, kg = tid % KG;  // rows RA og .. +RA-1, features 4 kg .. +3
    const int per_b = which == 0 ? S : C;
    const int Rout = which == 0 ? N : M, Rpart = which == 0 ? M : N;
    // work item = (bucket, KW-feature block): at D = 1024 a bucket's eight
    // feature blocks run on eight CTAs instead of one after the other
    const int nkb = (D + KW - 1) / KW;
    for (int item = blockIdx.x; item < B * per_b * nkb; item += gridDim.x) {
        const int key = item / nkb, kb = KW * (item % nkb);
        const int b = key / per_b, blk = key % per_b;
        const int o0 = 32 * blk;
        int lo, hi;
        const int *ordp = ord;
        if (which == 0) {
            lo = key * quota;
            hi = lo + strip_tiles[key];
        } else if (ord) {
            lo = off[key];
            hi = off[key + 1];
        } else {
            // ordered compaction, 256 strips at a time
            int n = 0;
            for (int sb = 0; sb < S; sb += 256) {
                const int s = sb + tid;
                int found = -1;
                if (s < S) {
                    const int ks = b * S + s, nt = strip_tiles[ks];
                    for (int q = 0; q < nt; ++q)
                        if (meta[ks * quota + q].z == blk) {
                            found = ks * quota + q;
                            break;
                        }
                }
                const unsigned bal = __ballot_sync(kFull, found >= 0);
                const int w = tid >> 5, ln = tid & 31;
                __syncthreads();  // lst / wcnt of the previous round consumed
                if (ln == 0) wcnt[w] = __popc(bal);
                __syncthreads();
                int pre = n;
                for (int q = 0; q < w; ++q) pre += wcnt[q];
                if (found >= 0) lst[pre + __popc(bal & ((1u << ln) - 1u))] = found;
                for (int q = 0; q < 8; ++q) n += wcnt[q];
            }
            __syncthreads();
            lo = 0;
            hi = n;
            ordp = lst;
        }
        const T *vo = vout + (size_t)b * Rout * D;
        const T *vp = vpart + (size_t)b * Rpart * D;
        T *g = grad + (size_t)b * Rout * D;
        if (lo == hi) {
            // no non-zero E tile touches this block: the gradient is exactly 0
#pragma unroll
            for (int a = 0; a < RA; ++a) {
                const int o = RA * og + a;
                if (o0 + o >= Rout) continue;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int k = kb + 4 * kg + q;
                    if (k < D) g[(size_t)(o0 + o) * D + k] = T(0);
                }
            }
            continue;
        }
        T acc[RA][4];
#pragma unroll
        for (int a = 0; a < RA; ++a)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[a][q] = T(0);
        double marg_acc = 0.0;  // warp 0: marginal of output row tid
        // tile operands go through registers one tile ahead: the loads of
        // tile e + 1 are in flight while tile e is contracted
        T re[4], rp[NP];
        int np_next = 0;
        auto load_tile = [&](int e) {
            const int idx = which == 0 ? e : ordp[e];
            const int4 m = meta[idx];
            const T *et = tiles + (size_t)idx * 1024;  // [r][jj]
            const int p0 = which == 0 ? 32 * m.z : 32 * m.y;
            const int np = which == 0 ? m.w : min(32, N - 32 * m.y);
            np_next = np;
#pragma unroll
            for (int q = 0; q < 4; ++q) re[q] = et[tid + 256 * q];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int u = tid + 256 * q;
                const int r = u / KW, k = u % KW;
                rp[q] = (r < np && kb + k < D) ? vp[(size_t)(p0 + r) * D + kb + k] : T(0);
            }
        };
        load_tile(lo);
        for (int e = lo; e < hi; ++e) {
            const int np = np_next;
            __syncthreads();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int u = tid + 256 * q;
                const int r = u >> 5, jj = u & 31;
                if (which == 0) Et[jj][r] = re[q];  // o = r, m = jj
                else Et[r][jj] = re[q];             // o = jj, m = r
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int u = tid + 256 * q;
                P[u / KW][u % KW] = rp[q];
            }
            __syncthreads();
            if (e + 1 < hi) load_tile(e + 1);
            // marginals in fp64 (tile order, then partner order): warp 0,
            // outside the FMA loop (no divergent fp64 adds in it)
            if (tid < 32) {
                double mgt = marg_acc;
                for (int mm = 0; mm < np; ++mm) mgt += (double)Et[mm][tid];
                marg_acc = mgt;
            }
            for (int mm = 0; mm < np; ++mm) {
                T ev[RA], pv[4];
                if constexpr (sizeof(T) == 4 && RA == 4) {
                    const float4 e4 = *reinterpret_cast<const float4 *>(&Et[mm][4 * og]);
                    ev[0] = e4.x; ev[1] = e4.y; ev[2] = e4.z; ev[3] = e4.w;
                } else if constexpr (sizeof(T) == 4 && RA == 2) {
                    const float2 e2 = *reinterpret_cast<const float2 *>(&Et[mm][2 * og]);
                    ev[0] = e2.x; ev[1] = e2.y;
                } else {
#pragma unroll
                    for (int a = 0; a < RA; ++a) ev[a] = Et[mm][RA * og + a];
                }
                if constexpr (sizeof(T) == 4) {
                    const float4 p4 = *reinterpret_cast<const float4 *>(&P[mm][4 * kg]);
                    pv[0] = p4.x; pv[1] = p4.y; pv[2] = p4.z; pv[3] = p4.w;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) pv[q] = P[mm][4 * kg + q];
                }
#pragma unroll
                for (int a = 0; a < RA; ++a)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[a][q] = fma(ev[a], pv[q], acc[a][q]);
            }
        }
        if (tid < 32) marg_s[tid] = marg_acc;
        __syncthreads();
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            const int o = RA * og + a;
            if (o0 + o >= Rout) continue;
            const double mg = marg_s[o];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = kb + 4 * kg + q;
                if (k < D) {
                    const size_t id = (size_t)(o0 + o) * D + k;
                    g[id] = (T)(2.0 * ((double)vo[id] * mg - (double)acc[a][q]));
                }
            }
        }
    }
}

// grad += 2 (v * marginal - acc) from the fixed-point accumulators (tiles the
// capped store could not hold).
template <class T>
__global__ void finalize_grads_fx_add_kernel(const T *__restrict__ v, const long long *__restrict__ marg_fx,
                                             const long long *__restrict__ acc_fx, const unsigned *absmax,
                                             const unsigned *stats, int N, int M, int rows, int D, int which,
                                             T *__restrict__ grad)
{
    if (stats[2] == 0) return;  // no tile overflowed the store: nothing to add
    const size_t total = (size_t)rows * D;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t r = idx / D;
        const int b = (int)(r / (which == 0 ? N : M));
        const FxScales fx = fx_scales(absmax + 2 * b, N, M);
        const double sm = 1.0 / (which == 0 ? fx.rs : fx.cs);
        const double sa = 1.0 / (which == 0 ? fx.gx : fx.gy);
        const double marg = (double)marg_fx[r] * sm;
        const double acc = (double)acc_fx[idx] * sa;
        if (marg != 0.0 || acc != 0.0) grad[idx] = (T)((double)grad[idx] + 2.0 * ((double)v[idx] * marg - acc));
    }
}

}  // namespace sdtw
