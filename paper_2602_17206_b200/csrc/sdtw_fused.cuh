// sdtw_fused.cuh — fused-distance mode on the tensor cores (fp32 path).
//
// Reference: cost_mode == CostMode::fused computes every cost on the fly from
// the series and the norm cache (cost.hpp:63-78, 112-121) instead of reading
// a materialised B x N x M tensor (cost.hpp:82-109).  Here the fused forward
// and the fused backward compute 128 x 32 (forward) or 32 x 32 (backward)
// cost blocks with tcgen05.mma from fp16 hi/lo operand blocks that producer
// warps stage in shared memory (fp32 rows loaded and split on the fly), with
// fp32 accumulators in TMEM, and feed them straight into the DP: no cost
// tensor reaches HBM.  The forward also keeps each strip's cost groups of a
// narrow band around the diagonal (the band cache, Dp3Args::band: O(B N W)
// bytes) for the backward, which falls back to recomputing on the tensor
// cores (sdtw_dp4.cuh, kTc) when an alignment leaves the band.
//
// Bit-compatibility.  Each cost is the same instruction sequence as the
// unfused tcgen05 GEMM (cost_gemm_tc_kernel): K steps of 16 in increasing
// order, per step the hi.hi, hi.lo, lo.hi passes, the same operand split and
// scale, the same epilogue fmaf(-2 inv, acc, xn + yn) clamped at 0.  A
// tensor-core output element depends only on its own A row and B column, so
// fused == unfused bit for bit (tested), and the backward's recompute sees
// exactly the costs the forward used.
//
// Forward CTA: 1 per SM, two independent "slots".  A slot owns a super-strip
// of 128 rows (4 DP strips, warp w of the slot = strip w = TMEM lane quarter
// w) of one pair; two producer warps per slot stage the super-strip's X rows
// once and stream 32-column Y chunks in, and the first of them issues the
// MMAs into an 8-deep ring of 128 x 32 TMEM tiles; each DP warp
// reads its quarter of chunk G with tcgen05.ld when it starts skewed group G,
// applies the epilogue and writes the two skewed groups the chunk feeds into
// its private shared-memory ring, from which the forward step body (the v3
// one) runs.  Strips of one slot hand the bottom-row h to the strip below
// through shared memory (32-column ring + progress counters) instead of L2;
// the slot's top strip polls the previous super-strip's tagged halo as v3.
#pragma once
#include <type_traits>
#include "sdtw_common.cuh"
#include "sdtw_dp2.cuh"
#include "sdtw_dp3.cuh"
#include "sdtw_tc.cuh"

namespace sdtw {

// Operand staging: rows [r0, r0 + rows) of a [R][D] fp32 series, split into
// fp16 hi / lo (scale sc) as the SWIZZLE_NONE K-major image of a rows-row
// operand tile (K-block stride rows * 16 bytes; features >= D and rows >= R
// zero), hi at `dst`, lo at dst + rows * dpad * 2.  One warp; lane = row
// within each 32-row group, so the 16-byte shared stores are conflict-free.
// The values are exactly those cost_gemm_tc_kernel stages (split_store8).
__device__ __forceinline__ void stage_split_rows(const float *__restrict__ src, int ld, int r0, int rows, int R,
                                                 int D, int dpad, float sc, uint8_t *dst, int lane, int nlanes = 32)
{
    uint8_t *hi = dst, *lo = dst + (size_t)rows * dpad * 2;
    const bool vec = (ld & 7) == 0;
    const int kbn = dpad / 8;
    for (int u = lane; u < rows * kbn; u += nlanes) {
        const int r = u % rows, kb = u / rows;
        const int row = r0 + r, k = kb * 8;
        const int nk = row < R ? max(0, min(8, D - k)) : 0;
        const float *p = src + (size_t)min(row, R - 1) * ld + min(k, D - 1);
        tc::split_store8(p, sc, hi, lo, tc::kmajor_off(r, kb, rows * 16), nk, vec && nk == 8);
    }
}

// 8 floats (scaled by sc) -> fp16 hi and lo halves, two per conversion
// instruction; the same round-to-nearest values as split_store8.
__device__ __forceinline__ void split8_packed(const float (&f)[8], float sc, uint4 &hq, uint4 &lq)
{
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 v = make_float2(f[2 * e] * sc, f[2 * e + 1] * sc);
        const __half2 h2 = __float22half2_rn(v);
        const float2 hb = __half22float2(h2);
        const __half2 l2 = __float22half2_rn(make_float2(v.x - hb.x, v.y - hb.y));
        hw[e] = *reinterpret_cast<const uint32_t *>(&h2);
        lw[e] = *reinterpret_cast<const uint32_t *>(&l2);
    }
    hq = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    lq = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

// Asynchronous variant for one warp: raw fp32 rows land in shared memory by
// cp.async (zero-filled past row R / feature D; needs D % 4 == 0), then are
// split shared -> shared.  raw: rows x (kc + 4) floats (padded stride: the
// per-row 32-byte reads of the split are bank-conflict free).
__device__ __forceinline__ void cp_async16_zfill(void *smem_dst, const void *gmem_src, int src_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src), "r"(src_bytes)
                 : "memory");
}
// issue: rows [r0, r0 + rows) x features [k0, k0 + kc) of src[R][ld] (valid D)
__device__ __forceinline__ void raw_rows_async(float *raw, const float *__restrict__ src, int ld, int r0, int rows, int R,
                                               int k0, int kc, int D, int lane)
{
    const int pieces = kc / 4;
    for (int u = lane; u < rows * pieces; u += 32) {
        const int r = u / pieces, pc = u % pieces;
        const int row = r0 + r, k = k0 + 4 * pc;
        const int nb = row < R ? max(0, min(16, (D - k) * 4)) : 0;
        const float *p = src + (size_t)min(row, R - 1) * ld + min(k, D - 4);
        cp_async16_zfill(raw + r * (kc + 4) + 4 * pc, p, nb);
    }
}
// split: raw rows [0, rows) -> operand tile rows [row0, row0 + rows), K blocks
// [0, kc / 8) (K-block stride kbs bytes), hi at `hi`, lo at `lo`
__device__ __forceinline__ void split_raw_rows(const float *raw, int rows, int kc, float sc, uint8_t *hi, uint8_t *lo,
                                               int row0, int kbs, int lane)
{
    const int kbn = kc / 8;
    for (int u = lane; u < rows * kbn; u += 32) {
        const int r = u % rows, kb = u / rows;
        const float4 a4 = *reinterpret_cast<const float4 *>(raw + r * (kc + 4) + 8 * kb);
        const float4 b4 = *reinterpret_cast<const float4 *>(raw + r * (kc + 4) + 8 * kb + 4);
        const float f[8] = {a4.x, a4.y, a4.z, a4.w, b4.x, b4.y, b4.z, b4.w};
        __align__(16) __half hh[8];
        __align__(16) __half ll[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float v = f[e] * sc;
            hh[e] = __float2half_rn(v);
            ll[e] = __float2half_rn(v - __half2float(hh[e]));
        }
        const uint32_t off = tc::kmajor_off(row0 + r, kb, kbs);
        *reinterpret_cast<uint4 *>(hi + off) = *reinterpret_cast<const uint4 *>(hh);
        *reinterpret_cast<uint4 *>(lo + off) = *reinterpret_cast<const uint4 *>(ll);
    }
}


struct FusedTcArgs {
    int dpad;  // D rounded up to 64 (<= kFtcMaxD): the unfused GEMM's K padding
};

constexpr int kFtcMaxD = 128;
constexpr int kFtcRing = 8;       // TMEM cost tiles per slot (128 lanes x 32 columns)
constexpr int kFtcHx = 32;        // intra-slot h hand-off ring (columns)
constexpr int kFtcThreads = 384;  // 8 DP warps + 4 producer warps

__host__ __device__ constexpr size_t ftc_slot_bytes(int dpad)
{
    return (size_t)128 * dpad * 4 + (size_t)32 * dpad * 4 + (size_t)4 * 2048 * 4;
}

struct FtcShared {
    uint64_t full[2][kFtcRing];   // MMA of a ring tile done (tcgen05.commit)
    uint64_t empty[2][kFtcRing];  // the 4 DP warps of the slot read the ring tile
    uint64_t tkfull[2][2], tkempty[2][2];
    int tkq[2][2];
    unsigned rd[2][4];                       // cumulative columns of top halo consumed by strip w
    unsigned long long hx[2][3][kFtcHx];     // (position << 32 | h) bottom-row h of strips 0..2
    float halo[8][32];                       // top halo stage of each DP warp
    uint32_t tmem_base;
};

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p)));
    return v;
}
__device__ __forceinline__ void st_volatile_u32(unsigned *p, unsigned v)
{
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(tc::smem_u32(p)), "r"(v));
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(tc::smem_u32(p)));
    return v;
}
__device__ __forceinline__ void st_shared_u64_if(unsigned long long *p, unsigned long long v, bool pred)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.volatile.shared.u64 [%0], %1;\n\t}" ::"r"(
                     tc::smem_u32(p)),
                 "l"(v), "r"((int)pred)
                );
}
__device__ __forceinline__ void named_bar(int id, int threads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Register-staged half of a 32-row operand chunk: rows [16 q, 16 q + 16) of
// the chunk, 16-byte K blocks; lane item i covers (row u & 15, K block u >> 4)
// with u = lane + 32 i.  Loads are issued one chunk ahead of the stores.
struct HalfChunk {
    float4 v[8][2];
};
__device__ __forceinline__ void half_chunk_load(HalfChunk &h, const float *__restrict__ src, int ld, int r0, int R,
                                                int D, int kbn, int lane)
{
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int u = lane + 32 * i;
        const int r = u & 15, kb = u >> 4;
        if (kb < kbn) {
            const int row = r0 + r, k = kb * 8;
            const float *p = src + (size_t)min(row, R - 1) * ld + min(k, D - 1);
            if (row < R && k + 8 <= D && (ld & 7) == 0) {
                h.v[i][0] = __ldg(reinterpret_cast<const float4 *>(p));
                h.v[i][1] = __ldg(reinterpret_cast<const float4 *>(p) + 1);
            } else {
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = (row < R && k + e < D) ? p[e] : 0.f;
                h.v[i][0] = make_float4(f[0], f[1], f[2], f[3]);
                h.v[i][1] = make_float4(f[4], f[5], f[6], f[7]);
            }
        }
    }
}
// Stores the 16 rows as tile rows [row0, row0 + 16) of an operand tile with
// K-block stride kbs bytes (hi at `hi`, lo at `lo`).
__device__ __forceinline__ void half_chunk_store(const HalfChunk &h, float sc, uint8_t *hi, uint8_t *lo, int row0,
                                                 int kbs, int kbn, int lane)
{
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int u = lane + 32 * i;
        const int r = u & 15, kb = u >> 4;
        if (kb < kbn) {
            const float f[8] = {h.v[i][0].x, h.v[i][0].y, h.v[i][0].z, h.v[i][0].w,
                                h.v[i][1].x, h.v[i][1].y, h.v[i][1].z, h.v[i][1].w};
            uint4 hq, lq;
            split8_packed(f, sc, hq, lq);
            const uint32_t off = tc::kmajor_off(row0 + r, kb, kbs);
            *reinterpret_cast<uint4 *>(hi + off) = hq;
            *reinterpret_cast<uint4 *>(lo + off) = lq;
        }
    }
}

// ---------------------------------------------------------------------------
// One strip of a slot (super-strip of 4 strips, warp w = strip w): the v3
// forward step body with the slot's shared-memory hand-off between its strips
// and the tagged L2 halo for strip 0.  `fill(G, lap)` makes the costs of
// skewed group G available in `ring` (two 1024-float groups, slot G & 1):
// the fused kernel's TMEM epilogue or the unfused kernel's cp.async of the
// cost tensor.
// ---------------------------------------------------------------------------
template <bool kTrace, class Fill>
__device__ __forceinline__ void slot_strip_forward(const Dp3Args<float> &A, int b, int s, int w, unsigned base,
                                                   float *ring, float *halo_s, unsigned *rd,
                                                   unsigned long long (*hx)[kFtcHx], Fill &&fill)
{
    using TG = Tagged<float>;
    const DpArgs<float> &a = A.a;
    const int t = threadIdx.x & 31;
    const unsigned epoch = A.epoch;
    const unsigned Mu = (unsigned)a.M;
    const float inf = Num<float>::inf();
            const int row = 32 * s + t + 1;
    const bool row_ok = row <= a.N;
    // trace: [16 B S + 4 (b S + s) + e]: e = 0 ticket, 1 first 32 columns
    // done, 2 half the columns done, 3 end
    // trace mode is a separate instantiation: the product kernel carries no
    // clock reads or trace tests on the step path
    unsigned long long *trc = (kTrace && A.trace) ? A.trace + 16 * (size_t)a.B * a.S + 4 * ((size_t)b * a.S + s) : nullptr;
    if (trc && t == 0) trc[0] = global_ns();
    // cycle accounting (trace mode): [24 B S + 8 (b S + s) + e]:
    // e = 0 cost-tile wait, 1 epilogue, 2 halo wait, 3 back-pressure, 4 steps
    long long cyc[5] = {0, 0, 0, 0, 0};
    long long c_mark = trc ? clock64() : 0;
    auto lap = [&](int e) {
if (trc) {
    const long long now = clock64();
    cyc[e] += now - c_mark;
    c_mark = now;
}
    };
    const bool top_global = w == 0;             // halo from the previous super-strip (L2)
    const bool pub_local = w < 3 && s + 1 < a.S;  // hand h to the strip below in smem
    float h_prev = 0.f, l_carry = 0.f;
    double lacc = 0.0;
    float gdiag = 0.f;
    const int kdiag = 32 * s + 2 * t;
    const typename TG::Ent *hb_top = A.hbt + ((size_t)b * a.S + (s - 1)) * a.M;
    typename TG::Ent *hb_me = A.hbt + ((size_t)b * a.S + s) * a.M;
    const unsigned long long *hx_up = w > 0 ? hx[w - 1] : nullptr;
    unsigned long long *hx_me = w < 3 ? hx[w] : hx[0];
    const int steps = a.M + 31;
    const bool r1 = row == 1;  // lane 0 of a pair's first strip: R(0, j) = inf
    const bool has_rowN = 32 * (s + 1) >= a.N;
    const bool strip_full = 32 * (s + 1) <= a.N;  // every lane's row exists
    unsigned long long pf_w = 0;
    int pf_kb = -1;
    for (int k0 = 0; k0 < steps; k0 += 32) {
const int G = k0 >> 5;
__syncwarp();
if (trc && t == 0 && (G == 1 || G == a.C / 2)) trc[G == 1 ? 1 : 2] = global_ns();
fill(G, lap);
const int cmin = k0 - 31, cmax = k0 + 31;
const bool fixup = cmin <= 0 ||
                   (a.bw != 0 && (32 * s - k0 - 31 < -a.bw || 32 * s + 62 - k0 > a.bw));
const bool tail = (has_rowN && a.M > a.N && cmax >= a.N) || (a.N > a.M && cmax >= a.M - 1);
float vck = 0.f;
const float *rg = ring + (G & 1) * 1024;
#pragma unroll 1
for (int k8 = 0; k8 < 32; k8 += 8) {
    const int kb = k0 + k8;
    // ---- top halo for columns [kb, kb + 8): tagged entries,
    // from L2 (strip 0 of the slot) or from the slot's ring
    lap(4);
    if (s > 0 && kb < a.M) {
        const int nn = min(8, a.M - kb);
        float hv = 0.f;
        if (top_global) {
            bool ok = t >= nn;
            if (!ok) {
                const unsigned long long w8 = (pf_kb == kb) ? pf_w : TG::load_raw(hb_top + kb + t);
                ok = (unsigned)(w8 >> 32) == epoch;
                hv = __uint_as_float((unsigned)(w8 & 0xffffffffull));
            }
            if (!__all_sync(kFull, ok)) hv = poll_entries<float>(hb_top + kb, nn, epoch, t);
            const int kb2 = kb + 8;
            if (kb2 < a.M && t < min(8, a.M - kb2)) {
                pf_w = TG::load_raw(hb_top + kb2 + t);
                pf_kb = kb2;
            }
        } else {
            const unsigned pos = base + (unsigned)(kb + t);
            bool ok = t >= nn;
            unsigned polls = 0;
            for (;;) {
                if (!ok) {
                    const unsigned long long e8 = ld_volatile_u64(hx_up + (pos & (kFtcHx - 1)));
                    ok = (unsigned)(e8 >> 32) == pos;
                    hv = __uint_as_float((unsigned)(e8 & 0xffffffffull));
                }
                if (__all_sync(kFull, ok)) break;
                if (++polls > (1u << 28)) {
                    if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                    break;
                }
            }
        }
        if (t < nn) halo_s[(kb + t) & 31] = hv;
        __syncwarp();
        if (!top_global && t == 0) st_volatile_u32(&rd[w], base + (unsigned)(kb + nn));
    }
    lap(2);
    // ---- back-pressure: the strip below must have consumed the
    // hand-off entries these 8 steps overwrite
    if (pub_local) {
        const int cw = kb + 8 - 31;  // columns [.., cw) final after this sub-group
        if (cw > 0) {
            const unsigned need = base + (unsigned)cw - (unsigned)kFtcHx;
            unsigned polls = 0;
            while ((int)(ld_volatile_u32(&rd[w + 1]) - need) < 0) {
                if (++polls > (1u << 28)) {
                    if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                    break;
                }
            }
        }
    }
    lap(3);
    // two copies of the 8 steps: with the boundary / band / tail
    // fix-ups, and the plain branch-free one (warp-uniform choice)
    auto steps8 = [&](auto fix_tag) {
        constexpr bool kFix = decltype(fix_tag)::value;
        // the 8 halo values and costs up front: no shared load
        // on the step's dependency chain
        float hsv[8], dvv[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            hsv[kk] = halo_s[k8 + kk];
            dvv[kk] = rg[(k8 + kk) * 32 + t];
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int k = kb + kk;
            const int kl = k8 + kk;
            const float src = (t == 31) ? hsv[kk] : h_prev;
            const float uu = __shfl_sync(kFull, src, (t + 31) & 31);
            const int col = k - t;
            const bool active = row_ok && col >= 0 && col < a.M;
            const float d = dvv[kk];
            float g, v, h;
            fwd_cell<float>(d, uu, l_carry, a.k, a.gln2, g, v, h);
            // row 1 in every group (three selects, no branch)
            g = r1 ? d : g;
            v = r1 ? -inf : v;
            h = r1 ? d : h;
            if constexpr (kFix) {
                if (fixup) {
                    const bool j1 = col == 0;
                    g = j1 ? d : g;
                    v = r1 ? -inf : (j1 ? d : v);
                    h = j1 ? -inf : h;
                    if (a.bw != 0 && !in_band(row, col + 1, a.bw)) {
                        g = inf; v = inf; h = inf;
                    }
                }
                if (tail && active) {
                    const int i = row, j = col + 1;
                    if (i == a.N && j > a.N) lacc += (double)h;
                    if (j == a.M && i > a.M) lacc += (double)v;
                }
            }
            gdiag = (active && k == kdiag) ? g : gdiag;
            vck = (kl == ((t - 1) & 31)) ? v : vck;
            l_carry = v;
            h_prev = h;
            TG::store_if(hb_me + col, h, epoch, t == 31 && active);
            const unsigned pos = base + (unsigned)col;
            st_shared_u64_if(hx_me + (pos & (kFtcHx - 1)), ((unsigned long long)pos << 32) | __float_as_uint(h),
                             pub_local && t == 31 && active);
        }
    };
    // lean sub-group: interior, every lane active (full strip, columns in
    // [1, M)), not strip 0, no lane at its diagonal cell: the cell, the
    // chunk-boundary capture and lane 31's two hand-off stores only (same
    // arithmetic as the plain body, ~10 fewer instructions per step)
    const bool lean = !fixup && !tail && s > 0 && strip_full && kb >= 31 && kb + 7 < a.M &&
                      (kb + 7 < 32 * s || kb > 32 * s + 62);
    if (lean) {
        float hsv[8], dvv[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            hsv[kk] = halo_s[k8 + kk];
            dvv[kk] = rg[(k8 + kk) * 32 + t];
        }
        typename TG::Ent *hp = hb_me + (kb - 31);
        const unsigned pos0 = base + (unsigned)(kb - 31);
        // lane 31's eight bottom-row h leave after the sub-group, not one
        // predicated store pair per step on the step's issue path: the strip
        // below consumes them 8 columns at a time anyway (no added lag)
        float hb[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int kl = k8 + kk;
            const float src = (t == 31) ? hsv[kk] : h_prev;
            const float uu = __shfl_sync(kFull, src, (t + 31) & 31);
            float g, v, h;
            fwd_cell<float>(dvv[kk], uu, l_carry, a.k, a.gln2, g, v, h);
            vck = (kl == ((t - 1) & 31)) ? v : vck;
            l_carry = v;
            h_prev = h;
            hb[kk] = h;
        }
        if (t == 31) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                TG::store(hp + kk, hb[kk], epoch);
                const unsigned pos = pos0 + (unsigned)kk;
                if (pub_local)
                    st_shared_u64_if(hx_me + (pos & (kFtcHx - 1)),
                                     ((unsigned long long)pos << 32) | __float_as_uint(hb[kk]), true);
            }
        }
        __syncwarp();
    } else if (fixup || tail) {
        steps8(std::true_type{});
    } else {
        steps8(std::false_type{});
    }
}
const int bidx = (t == 0) ? G : (G - 1);
const int jb = 32 * (bidx + 1);
if (bidx >= 0 && jb < a.M && row_ok) a.vc[((size_t)b * a.C + bidx) * a.N + (row - 1)] = vck;
    }
    if (t == 0) st_volatile_u32(&rd[w], base + Mu);
    if (trc && t == 0) trc[3] = global_ns();
    lap(4);
    if (trc && t == 0)
for (int e = 0; e < 5; ++e)
    A.trace[24 * (size_t)a.B * a.S + 8 * ((size_t)b * a.S + s) + e] = (unsigned long long)cyc[e];
    lacc += (double)gdiag;
    for (int off = 16; off > 0; off >>= 1) lacc += __shfl_xor_sync(kFull, lacc, off);
    if (t == 0) a.lpart[(size_t)b * a.S + s] = lacc;
}

// ---------------------------------------------------------------------------
// Fused forward (fp32).  384 threads: warps 0-3 slot 0 DP, 4-7 slot 1 DP,
// 8-9 / 10-11 the producer pair of slot 0 / 1 (the first of a pair takes the
// tickets and issues the MMAs).  Tickets over super-strips (strip-major,
// pair-minor) from a.tickets[0].
// ---------------------------------------------------------------------------
template <int kTU = 0, bool kTrace = false>
__global__ void __launch_bounds__(kFtcThreads, 1) sdtw_forward_tc_kernel(Dp3Args<float> A, FusedTcArgs F)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ FtcShared sh;
    using TG = Tagged<float>;
    const DpArgs<float> &a = A.a;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const int dpad = F.dpad;
    const int SSn = (a.S + 3) / 4;
    const int total = a.B * SSn;
    const unsigned Mu = (unsigned)a.M;

    if (threadIdx.x == 0) {
        for (int p = 0; p < 2; ++p) {
            for (int r = 0; r < kFtcRing; ++r) {
                tc::mbar_init(&sh.full[p][r], 1);
                tc::mbar_init(&sh.empty[p][r], 4);
            }
            for (int q = 0; q < 2; ++q) {
                tc::mbar_init(&sh.tkfull[p][q], 1);
                tc::mbar_init(&sh.tkempty[p][q], 4);
            }
            for (int w = 0; w < 4; ++w) sh.rd[p][w] = 0;
        }
        tc::fence_barrier_init();
    }
    for (int e = threadIdx.x; e < 2 * 3 * kFtcHx; e += blockDim.x)
        (&sh.hx[0][0][0])[e] = 0xffffffff00000000ull;  // no position matches
    if (warp == 0) tc::tmem_alloc<512>(&sh.tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = sh.tmem_base;

    if (warp >= 8) {
        // ------------------------------------------------------------ producers
        const int p = (warp - 8) >> 1, q = (warp - 8) & 1;
        const bool leader = q == 0;
        uint8_t *xs = smem_raw + (size_t)p * ftc_slot_bytes(dpad);
        uint8_t *ys = xs + (size_t)128 * dpad * 4;
        const uint32_t idesc = tc::idesc_f16_f32(128, 32);
        const int ksteps = dpad / 16, kbn = dpad / 8;
        unsigned u = 0;  // cumulative chunk count of this slot
        HalfChunk pre;
        for (unsigned n = 0;; ++n) {
            if (leader) {
                const unsigned tk = warp_ticket(&a.tickets[0]);
                tc::mbar_wait(&sh.tkempty[p][n & 1], ((n >> 1) & 1) ^ 1);
                if (t == 0) {
                    sh.tkq[p][n & 1] = (int)tk;
                    tc::mbar_arrive(&sh.tkfull[p][n & 1]);
                }
            } else {
                tc::mbar_wait(&sh.tkfull[p][n & 1], (n >> 1) & 1);
            }
            const int tk = sh.tkq[p][n & 1];
            named_bar(1 + p, 64);  // both have read the ticket
            if (tk >= total) break;
            const int ss = tk / a.B, b = tk % a.B;
            const float *xb = a.x + (size_t)b * a.N * a.D;
            const float *yb = a.y + (size_t)b * a.M * a.D;
            const SplitScale sc = split_scale(A.absmax + 2 * b);
            // X: rows [128 ss + 64 q, +64) of the super-strip (previous MMAs done)
            for (int m = 0; m < 4; ++m) {
                half_chunk_load(pre, xb, a.D, 128 * ss + 64 * q + 16 * m, a.N, a.D, kbn, t);
                half_chunk_store(pre, sc.sx, xs, xs + 128 * dpad * 2, 64 * q + 16 * m, 2048, kbn, t);
            }
            half_chunk_load(pre, yb, a.D, 16 * q, a.M, a.D, kbn, t);
            for (int c = 0; c < a.C; ++c, ++u) {
                const int sl = (int)(u % kFtcRing);
                half_chunk_store(pre, sc.sy, ys, ys + 32 * dpad * 2, 16 * q, 512, kbn, t);
                if (c + 1 < a.C) half_chunk_load(pre, yb, a.D, 32 * (c + 1) + 16 * q, a.M, a.D, kbn, t);
                tc::fence_async_smem();
                named_bar(1 + p, 64);  // X / Y chunk staged by both warps
                if (leader) {
                    tc::mbar_wait(&sh.empty[p][sl], ((u / kFtcRing) & 1) ^ 1);
                    tc::tc_fence_after();
                    if (t == 0) {
                        const uint32_t d = tmem + 256u * p + 32u * sl;
                        const uint32_t ah = tc::smem_u32(xs), al = ah + 128u * dpad * 2;
                        const uint32_t bh = tc::smem_u32(ys), bl = bh + 32u * dpad * 2;
                        for (int ks = 0; ks < ksteps; ++ks) {
                            const uint32_t oa = ks * 2 * 2048, ob = ks * 2 * 512;
                            const uint32_t acc0 = ks > 0 ? 1u : 0u;
                            tc::mma_f16(d, tc::smem_desc(ah + oa, 2048, 128), tc::smem_desc(bh + ob, 512, 128), idesc, acc0);
                            tc::mma_f16(d, tc::smem_desc(ah + oa, 2048, 128), tc::smem_desc(bl + ob, 512, 128), idesc, 1u);
                            tc::mma_f16(d, tc::smem_desc(al + oa, 2048, 128), tc::smem_desc(bh + ob, 512, 128), idesc, 1u);
                        }
                        tc::mma_commit(&sh.full[p][sl]);
                    }
                    __syncwarp();
                }
                // the Y buffer (and, after the last chunk, X) is free once the MMAs finished
                tc::mbar_wait(&sh.full[p][sl], (u / kFtcRing) & 1);
            }
        }
    } else {
        // ------------------------------------------------------------ DP warps
        const int p = warp >> 2, w = warp & 3;
        float *ring = reinterpret_cast<float *>(smem_raw + (size_t)p * ftc_slot_bytes(dpad) +
                                                (size_t)160 * dpad * 4) +
                      w * 2048;
        float *halo_s = sh.halo[warp];
        const float inf = Num<float>::inf();
        const uint32_t tq = tmem + 256u * p + ((uint32_t)(32 * w) << 16);
        unsigned u = 0;
        for (unsigned n = 0;; ++n) {
            tc::mbar_wait(&sh.tkfull[p][n & 1], (n >> 1) & 1);
            const int tk = sh.tkq[p][n & 1];
            __syncwarp();
            if (t == 0) tc::mbar_arrive(&sh.tkempty[p][n & 1]);
            if (tk >= total) break;
            const int ss = tk / a.B, b = tk % a.B;
            const int s = 4 * ss + w;
            const float m2 = -2.0f * split_scale(A.absmax + 2 * b).inv;
            const unsigned base = n * Mu;  // cumulative column base of this super-strip
            if (s >= a.S) {
                // no strip here: keep the ring protocol going
                for (int c = 0; c < a.C; ++c, ++u) {
                    const int sl = (int)(u % kFtcRing);
                    tc::mbar_wait(&sh.full[p][sl], (u / kFtcRing) & 1);
                    __syncwarp();
                    if (t == 0) tc::mbar_arrive(&sh.empty[p][sl]);
                }
                if (t == 0) st_volatile_u32(&sh.rd[p][w], base + Mu);
                continue;
            }
            const int row_f = 32 * s + t + 1;
            const float xi = row_f <= a.N ? a.xn[(size_t)b * a.N + row_f - 1] : 0.f;
            float yn_next = t < a.M ? a.yn[(size_t)b * a.M + t] : 0.f;
            const bool row_ok = row_f <= a.N;
            const int row = row_f;
            const int glo = A.band ? band_lo(s, a.N, a.M, a.KK / 32, A.band_ng) : 1 << 30;
            float *band_s = A.band ? A.band + ((size_t)b * a.S + s) * (size_t)A.band_ng * 1024 : nullptr;
            auto fill = [&](int G, auto &lap) {
                if (G < a.C) {
                    // cost chunk G: TMEM quarter -> epilogue -> skewed ring
                    const unsigned uu = u + G;
                    const int sl = (int)(uu % kFtcRing);
                    lap(4);
                    tc::mbar_wait(&sh.full[p][sl], (uu / kFtcRing) & 1);
                    lap(0);
                    tc::tc_fence_after();
                    float acc[32];
                    tc::tmem_ld32(tq + 32u * sl, acc);
                    tc::tc_fence_before();
                    __syncwarp();
                    if (t == 0) tc::mbar_arrive(&sh.empty[p][sl]);
                    const int j0 = 32 * G;
                    // column norms of this chunk (prefetched one group ahead)
                    const float yv = yn_next;
                    yn_next = (j0 + 32 + t < a.M) ? a.yn[(size_t)b * a.M + j0 + 32 + t] : 0.f;
                    // skewed rows (G & 1) * 32 + e + t of the two-group ring
                    const int rb = (G & 1) * 32 + t;
                    if (j0 + 32 <= a.M && a.bw == 0) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const float yj = __shfl_sync(kFull, yv, e);
                            ring[((rb + e) & 63) * 32 + t] = tc_cost(acc[e], xi, yj, m2, row_ok);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const float yj = __shfl_sync(kFull, yv, e);
                            const int j = j0 + e;
                            const bool ok = row_ok && j < a.M && in_band(row, j + 1, a.bw);
                            ring[((rb + e) & 63) * 32 + t] = tc_cost(acc[e], xi, yj, m2, ok);
                        }
                    }
                    __syncwarp();
                    lap(1);
                }
                // band cache: group G is complete once chunk G is in (its
                // other half came with chunk G - 1); entries off the matrix
                // are stored as zero, like the unfused cost tensor's
                const int gg = G - glo;
                if (gg >= 0 && gg < A.band_ng) {
                    const float *src = ring + (G & 1) * 1024;
                    float *dst = band_s + (size_t)gg * 1024;
#pragma unroll 8
                    for (int r = 0; r < 32; ++r) {
                        const int col = 32 * G + r - t;
                        const float v = src[r * 32 + t];
                        dst[r * 32 + t] = (row_ok && col >= 0 && col < a.M) ? v : 0.f;
                    }
                }
            };
            slot_strip_forward<kTrace>(A, b, s, w, base, ring, halo_s, sh.rd[p], sh.hx[p], fill);
            u += (unsigned)a.C;
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace sdtw
