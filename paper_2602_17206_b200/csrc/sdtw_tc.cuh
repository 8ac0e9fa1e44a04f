// sdtw_tc.cuh — Blackwell tensor-core plumbing (tcgen05 / TMEM / mbarrier)
// and the dense contractions of the Soft-DTW path:
//   * the pairwise cost tile  D = ||x||^2 + ||y||^2 - 2 X Y^T   (cost.hpp:63-99)
// computed with tcgen05.mma kind::f16, operands in shared memory, fp32
// accumulators in TMEM, read back with tcgen05.ld for the norm epilogue.
//
// Precision: fp32 operands are split x = s^-1 (x_hi + x_lo) with x_hi, x_lo
// fp16 (11 + 11 significant bits) under a power-of-two scale s that keeps
// |x s| <= 2^14; X Y^T = s^-2 (hi.hi + hi.lo + lo.hi) in three MMA passes with
// fp32 accumulation (the lo.lo term is below 2^-22 relative).  A single fp16
// (or TF32) pass perturbs costs by ~2^-11 relative and breaks gradient parity
// at gamma = 1.
#pragma once
#include <cuda_fp16.h>

#include "sdtw_common.cuh"

namespace sdtw {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// try_wait suspends the warp until the phase completes or the hint (ns)
// expires: waiting warps (producers ahead of their consumers, consumers
// ahead of the MMA) then take no issue slots from the warps they wait for
#ifndef SDTW_MBAR_SUSPEND_NS
#define SDTW_MBAR_SUSPEND_NS 0x989680
#endif
constexpr uint32_t kMbarSuspendNs = SDTW_MBAR_SUSPEND_NS;
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(kMbarSuspendNs)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Generic-proxy shared-memory writes -> visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMEM -----------------------------------------------------------------
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---- descriptors ------------------------------------------------------------
// Shared-memory matrix descriptor, SWIZZLE_NONE, K-major canonical layout:
// core matrices of 8 rows x 16 bytes (row r of a core at +16 r); LBO = byte
// distance between the two 16-byte K halves of one MMA-K step, SBO = byte
// distance between consecutive 8-row groups.  (PTX ISA "matrix descriptor";
// field layout as in CUTLASS's UMMA::SmemDescriptor.)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
    // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0: SWIZZLE_NONE
    return d;
}

// Instruction descriptor, kind::f16: A/B fp16, D fp32, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16_f32(int M, int N)
{
    return (1u << 4)                  // D format f32
           | (0u << 7) | (0u << 10)   // A, B format f16
           | (0u << 15) | (0u << 16)  // A, B K-major
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 1-D bulk copy shared -> global (TMA engine), tracked by the thread's bulk group.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the same with an L2 eviction-priority hint (createpolicy)
__device__ __forceinline__ void bulk_s2g_hint(void *dst, const void *src, uint32_t bytes, uint64_t policy)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(policy)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// the thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// the thread's bulk stores are complete
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns: thread t gets lane (base+t), columns
// [col, col+32).  The warp must own the lane quarter (warp_id % 4).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 16 consecutive fp32 columns (as tmem_ld32).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- operand staging ----------------------------------------------------------
// Byte offset of element (r, k) in a K-major SWIZZLE_NONE tile of `rows` rows
// whose 8-element K blocks are `kb_stride` bytes apart: core (r/8, k/8).
__device__ __forceinline__ uint32_t kmajor_off(int r, int kb, int kb_stride)
{
    return (uint32_t)(kb * kb_stride + (r >> 3) * 128 + (r & 7) * 16);
}

// Splits up to 8 consecutive fp32 values (scaled by s) into fp16 hi / lo
// halves and stores them as one 16-byte core-matrix row in each tile.
// `n` valid elements (0..8); `vec` allows two float4 loads (16-byte aligned).
__device__ __forceinline__ void split_store8(const float *src, float s, uint8_t *hi, uint8_t *lo,
                                             uint32_t off, int n, bool vec)
{
    float f[8];
    if (n == 8 && vec) {
        const float4 a = *reinterpret_cast<const float4 *>(src);
        const float4 b = *reinterpret_cast<const float4 *>(src + 4);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
        f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = e < n ? src[e] : 0.f;
    }
    __align__(16) __half h[8];
    __align__(16) __half l[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float v = f[e] * s;
        h[e] = __float2half_rn(v);
        l[e] = __float2half_rn(v - __half2float(h[e]));
    }
    *reinterpret_cast<uint4 *>(hi + off) = *reinterpret_cast<const uint4 *>(h);
    *reinterpret_cast<uint4 *>(lo + off) = *reinterpret_cast<const uint4 *>(l);
}

// split_store8 from registers (8 values already loaded).
__device__ __forceinline__ void split_store8_regs(const float4 (&v)[2], float s, uint8_t *hi, uint8_t *lo, uint32_t off)
{
    const float f[8] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w};
    __align__(16) __half h[8];
    __align__(16) __half l[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float w = f[e] * s;
        h[e] = __float2half_rn(w);
        l[e] = __float2half_rn(w - __half2float(h[e]));
    }
    *reinterpret_cast<uint4 *>(hi + off) = *reinterpret_cast<const uint4 *>(h);
    *reinterpret_cast<uint4 *>(lo + off) = *reinterpret_cast<const uint4 *>(l);
}

}  // namespace tc

// Power-of-two operand scales: |x * sx| <= 2^14, and 1/(sx sy).  absmax
// points at ONE pair's [max|x|, max|y|] (absmax[2 b], absmax[2 b + 1]): the
// split, and so every fp32 cost, depends only on that pair's own series, so
// a pair's results do not change with its batch-mates (sdtw(batch)[b] ==
// sdtw(batch[b:b+1]) bit for bit).
struct SplitScale {
    float sx, sy, inv;
};
__device__ __forceinline__ SplitScale split_scale(const unsigned *absmax)
{
    const float mx = fmaxf(__uint_as_float(absmax[0]), 1e-30f);
    const float my = fmaxf(__uint_as_float(absmax[1]), 1e-30f);
    int ex, ey;
    frexpf(mx, &ex);  // mx < 2^ex
    frexpf(my, &ey);
    SplitScale s;
    s.sx = ldexpf(1.0f, 14 - ex);
    s.sy = ldexpf(1.0f, 14 - ey);
    s.inv = ldexpf(1.0f, ex + ey - 28);
    return s;
}

// Norms in double, rounded once (the cost epilogue's largest terms), and the
// operand-scale maximum max|v| of each pair in the same pass: one warp per
// row, a fixed butterfly reduction (deterministic); row r belongs to pair
// r / rpp and its maximum goes to absmax[2 (r / rpp) + which].  Each CTA
// owns a contiguous row range, so a warp's rows mostly share one pair and it
// flushes its running maximum with one atomic per pair it touched.
template <int kTU = 0>
__global__ void __launch_bounds__(256) norms_absmax_f32_kernel(const float *__restrict__ x, int rows, int D,
                                                               float *__restrict__ out, unsigned *absmax, int rpp,
                                                               int which)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = (rows + gridDim.x - 1) / gridDim.x;
    const int r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
    float mx = 0.f;
    int pair = -1;
    int r = r0 + w;
    if ((D & 3) == 0 && D <= 128) {
        // four rows per warp iteration, their loads issued together (one
        // load latency per four rows instead of per row)
        for (; r + 24 < r1; r += 32) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                v[u] = 4 * lane < D ? __ldg(reinterpret_cast<const float4 *>(x + (size_t)(r + 8 * u) * D + 4 * lane))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int ru = r + 8 * u;
                if (ru / rpp != pair) {
                    if (pair >= 0 && lane == 0 && mx > 0.f) atomicMax(absmax + 2 * pair + which, __float_as_uint(mx));
                    pair = ru / rpp;
                    mx = 0.f;
                }
                double sd = 0.0;
                sd = fma((double)v[u].x, (double)v[u].x, sd);
                sd = fma((double)v[u].y, (double)v[u].y, sd);
                sd = fma((double)v[u].z, (double)v[u].z, sd);
                sd = fma((double)v[u].w, (double)v[u].w, sd);
                float m = fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w)));
                for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(kFull, sd, o);
                for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
                mx = fmaxf(mx, m);
                if (lane == 0) out[ru] = (float)sd;
            }
        }
    }
    for (; r < r1; r += 8) {
        if (r / rpp != pair) {
            if (pair >= 0 && lane == 0 && mx > 0.f) atomicMax(absmax + 2 * pair + which, __float_as_uint(mx));
            pair = r / rpp;
            mx = 0.f;
        }
        const float *e = x + (size_t)r * D;
        double s = 0.0;
        float m = 0.f;
        if ((D & 3) == 0) {
            for (int k = 4 * lane; k < D; k += 128) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(e + k));
                s = fma((double)v.x, (double)v.x, s);
                s = fma((double)v.y, (double)v.y, s);
                s = fma((double)v.z, (double)v.z, s);
                s = fma((double)v.w, (double)v.w, s);
                m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            }
        } else {
            for (int k = lane; k < D; k += 32) {
                const float v = e[k];
                s = fma((double)v, (double)v, s);
                m = fmaxf(m, fabsf(v));
            }
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
        mx = fmaxf(mx, m);
        if (lane == 0) out[r] = (float)s;
    }
    if (pair >= 0 && lane == 0 && mx > 0.f) atomicMax(absmax + 2 * pair + which, __float_as_uint(mx));
}

__device__ __forceinline__ void named_bar_cg(int id, int threads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// The cost epilogue shared by all tensor-core paths (the unfused GEMM, the
// fused forward and the fused backward recompute): accumulator acc of row i,
// column j; d = ||x_i||^2 + ||y_j||^2 - 2 <x_i, y_j>, clamped at 0
// (cost.hpp:63-78); 0 outside the matrix / band.
__device__ __forceinline__ float tc_cost(float acc, float xi, float yj, float m2, bool ok)
{
    float v = fmaf(m2, acc, xi + yj);
    v = v < 0.f ? 0.f : v;
    return ok ? v : 0.f;
}

// ----------------------------------------------------------------------------
// Operand packing for the unfused GEMM: rows [B][R][D] fp32 -> blocks
// [B][nblk][hi|lo][dpad/8][rpb][8] fp16, the SWIZZLE_NONE K-major image of an
// rpb-row operand tile (K-block stride rpb * 16 bytes); rows >= R and
// features >= D zero.  One thread per 16-byte core-matrix row, split exactly
// as split_store8.  which = 0: x (scale sx), 1: y (scale sy).
// ----------------------------------------------------------------------------
// Block k covers rows [k rstride + roff, + rpb) (rstride = rpb, roff = 0 for
// a plain tiling; the GEMM's B operand uses overlapping 160-row blocks).
template <int kTU = 0>
__global__ void pack_split_kernel(const float *__restrict__ src, int B, int R, int D, int dpad, int rpb,
                                  const unsigned *absmax, int which, uint8_t *__restrict__ dst, int rstride = 0,
                                  int roff = 0)
{
    if (rstride == 0) rstride = rpb;
    const int nblk = (R + rstride - 1) / rstride;  // blocks start at k rstride + roff (roff <= 0)
    const int kbn = dpad / 8;
    const size_t total = (size_t)B * nblk * rpb * kbn;
    const bool vec = (D & 7) == 0;
    for (size_t u = (size_t)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(u % rpb);        // row within the block (fastest: coalesced stores)
        const size_t rest = u / rpb;
        const int kb = (int)(rest % kbn);
        const size_t bb = rest / kbn;        // b * nblk + blk
        const int blk = (int)(bb % nblk);
        const int b = (int)(bb / nblk);
        const int row = blk * rstride + roff + r;
        const SplitScale sc = split_scale(absmax + 2 * b);
        const float s = which == 0 ? sc.sx : sc.sy;
        uint8_t *hi = dst + bb * (size_t)rpb * dpad * 4;
        uint8_t *lo = hi + (size_t)rpb * dpad * 2;
        const int k = kb * 8;
        const int nk = (row >= 0 && row < R) ? max(0, min(8, D - k)) : 0;
        const float *p = src + ((size_t)b * R + min(max(row, 0), R - 1)) * D + min(k, D - 1);
        tc::split_store8(p, s, hi, lo, tc::kmajor_off(r, kb, rpb * 16), nk, vec && nk == 8);
    }
}

// ----------------------------------------------------------------------------
// Unfused cost tensor on tcgen05 (materialize_costs, cost.hpp:82-99): one CTA
// per (pair, 128-row block, 128-column block).  Operands come from the packed
// fp16 hi/lo images by bulk copies (TMA engine), 32 features per round and
// four rounds in flight (a load warp and an MMA warp): A =
// the 128 x rows, B = five 32-column y chunks [j0 - 32, j0 + 128) (N = 32
// MMAs into TMEM columns 32 z).  The extra chunk on the left lets the CTA
// write whole rows of the DP's skewed strip layout
//   dsk[b][s][kk][t] = d(32 s + t, kk - t)   (0-based, kk in [0, KK))
// for kk in [j0, j0 + 128) with no row shared between CTAs: the epilogue
// writes each strip's costs into a shared-memory image of those skewed rows
// (bank-conflict free) and sends the image, contiguous in dsk, to HBM with one
// bulk store (TMA engine) that overlaps the next tile's epilogue.  The last
// column block also writes the tail rows up to KK.
// ----------------------------------------------------------------------------
constexpr int kCgStageRows = 160;                             // skewed rows per strip image (KK - j0 <= 160)
constexpr int kCgKR = 32;                                     // features per operand round
constexpr int kCgStages = 4;                                  // operand rounds in flight
constexpr int kCgABytes = 128 * kCgKR * 2;                    // 128 x rows, one fp16 half (8 KB)
constexpr int kCgBBytes = 160 * kCgKR * 2;                    // 160 y rows, one fp16 half (10 KB)
constexpr int kCgStageBytes = 2 * kCgABytes + 2 * kCgBBytes;  // one round's operands: A hi|lo + B hi|lo (36 KB)
constexpr int kCgXHalf = 128 * 128 * 2;                       // resident x rows, one fp16 half (dpad <= 128)
static_assert(2 * kCgXHalf + kCgStages * 2 * kCgBBytes <= kCgStages * kCgStageBytes,
              "resident x + the y ring must fit the operand ring");
constexpr int kCgEpiBytes = 4 * kCgStageRows * 32 * 4;        // four strip images (80 KB)
constexpr int kCgSmem = kCgStages * kCgStageBytes + kCgEpiBytes;  // 224 KB: four operand stages + staging
#ifndef CG_EPI_WARPS
#define CG_EPI_WARPS 12  // measured: 8 -> 0.808, 12 -> 0.772, 16 -> 0.804 ms at C3
#endif
constexpr int kCgEpiWarps = CG_EPI_WARPS;                     // epilogue warps (3 per TMEM lane quarter)
constexpr int kCgThreads = 32 * (kCgEpiWarps + 2);            // + MMA warp + load warp

struct CgShared {
    uint64_t st_full[kCgStages], st_empty[kCgStages], acc_full[2], acc_empty[2], x_full, x_empty;
    uint32_t tmem_base;
};

// Persistent and pipelined: TMEM kernels run one CTA per SM, so each CTA
// walks tiles (b, ib, jb) with the producer warp loading round g + 1 while
// the MMAs of round g run, and the epilogue warps draining tile n - 1
// from the other TMEM accumulator (2 x 160 columns) while tile n is computed.
template <int kTU = 0>
__global__ void __launch_bounds__(kCgThreads, 1)
    cost_gemm_tc_kernel(const uint8_t *__restrict__ xp, const uint8_t *__restrict__ yp, const float *__restrict__ xn,
                        const float *__restrict__ yn, const unsigned *absmax, int B, int N, int M, int S, int C,
                        int KK, int bw, int dpad, float *__restrict__ dsk)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ CgShared sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NB = (N + 127) / 128, JB = (M + 127) / 128;
    const int ntiles = B * NB * JB;
    const int rounds = dpad / kCgKR;
    if (tid == 0) {
        for (int k = 0; k < kCgStages; ++k) {
            tc::mbar_init(&sh.st_full[k], 1);
            tc::mbar_init(&sh.st_empty[k], 1);
        }
        tc::mbar_init(&sh.x_full, 1);
        tc::mbar_init(&sh.x_empty, 1);
        for (int k = 0; k < 2; ++k) {
            tc::mbar_init(&sh.acc_full[k], 1);
            tc::mbar_init(&sh.acc_empty[k], kCgEpiWarps);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(&sh.tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = sh.tmem_base;
    // a contiguous range of tiles per CTA (jb fastest): consecutive tiles
    // share the 128 x rows, which stay resident in shared memory when
    // dpad <= 128 (xres; the ring then carries y only)
    const int t0 = (int)((long long)blockIdx.x * ntiles / gridDim.x);
    const int t1 = (int)((long long)(blockIdx.x + 1) * ntiles / gridDim.x);
    const bool xres = dpad <= 128;
    auto tile_of = [&](int n, int &b, int &ib, int &jb) {
        jb = n % JB;
        const int r = n / JB;
        ib = r % NB;
        b = r / NB;
    };

    if (warp == kCgEpiWarps + 1) {
        // ---------------------------------------------------------------- loads
        // one bulk copy per operand half and round, kCgStages rounds ahead of
        // the MMAs (the ring runs across tile boundaries)
        if (lane == 0) {
            int g = 0, xr = 0;
            for (int n = t0; n < t1; ++n) {
                int b, ib, jb;
                tile_of(n, b, ib, jb);
                const uint8_t *xa = xp + ((size_t)b * NB + ib) * (size_t)128 * dpad * 4;
                const uint8_t *ya = yp + ((size_t)b * JB + jb) * (size_t)160 * dpad * 4;
                if (xres && (n == t0 || n / JB != (n - 1) / JB)) {
                    // new x rows: wait until the MMAs on the previous ones are done
                    if (xr > 0) tc::mbar_wait(&sh.x_empty, (xr - 1) & 1);
                    const uint32_t xb = 128u * dpad * 2;
                    tc::mbar_expect_tx(&sh.x_full, 2 * xb);
                    tc::bulk_g2s(smem, xa, xb, &sh.x_full);
                    tc::bulk_g2s(smem + kCgXHalf, xa + xb, xb, &sh.x_full);
                    ++xr;
                }
                for (int kc = 0; kc < rounds; ++kc, ++g) {
                    const int sb = g % kCgStages;
                    tc::mbar_wait(&sh.st_empty[sb], ((g / kCgStages) & 1) ^ 1);
                    if (xres) {
                        uint8_t *st = smem + 2 * kCgXHalf + sb * 2 * kCgBBytes;
                        tc::mbar_expect_tx(&sh.st_full[sb], 2u * kCgBBytes);
                        tc::bulk_g2s(st, ya + (size_t)kc * kCgBBytes, kCgBBytes, &sh.st_full[sb]);
                        tc::bulk_g2s(st + kCgBBytes, ya + (size_t)160 * dpad * 2 + (size_t)kc * kCgBBytes, kCgBBytes,
                                     &sh.st_full[sb]);
                        continue;
                    }
                    uint8_t *st = smem + sb * kCgStageBytes;
                    tc::mbar_expect_tx(&sh.st_full[sb], (uint32_t)kCgStageBytes);
                    tc::bulk_g2s(st, xa + (size_t)kc * kCgABytes, kCgABytes, &sh.st_full[sb]);
                    tc::bulk_g2s(st + kCgABytes, xa + (size_t)128 * dpad * 2 + (size_t)kc * kCgABytes, kCgABytes,
                                 &sh.st_full[sb]);
                    tc::bulk_g2s(st + 2 * kCgABytes, ya + (size_t)kc * kCgBBytes, kCgBBytes, &sh.st_full[sb]);
                    tc::bulk_g2s(st + 2 * kCgABytes + kCgBBytes, ya + (size_t)160 * dpad * 2 + (size_t)kc * kCgBBytes,
                                 kCgBBytes, &sh.st_full[sb]);
                }
            }
        }
        __syncwarp();
    } else if (warp == kCgEpiWarps) {
        // ---------------------------------------------------------------- MMA
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_f16_f32(128, 160);
            int g = 0;   // global round counter of this CTA
            int li = 0;  // local tile index
            int xm = 0;  // x blocks consumed
            for (int n = t0; n < t1; ++n, ++li) {
                const int ab = li & 1;
                tc::mbar_wait(&sh.acc_empty[ab], ((li >> 1) & 1) ^ 1);  // epilogue done with tile li - 2
                tc::tc_fence_after();
                if (xres && (n == t0 || n / JB != (n - 1) / JB)) {
                    tc::mbar_wait(&sh.x_full, xm & 1);
                    tc::tc_fence_after();
                    ++xm;
                }
                for (int kc = 0; kc < rounds; ++kc, ++g) {
                    const int sb = g % kCgStages;
                    tc::mbar_wait(&sh.st_full[sb], (g / kCgStages) & 1);
                    tc::tc_fence_after();
                    // one M = 128, N = 160 MMA per K step and pass: B = the
                    // 160 y rows [j0 - 32, j0 + 128) (K-block stride 2560 B)
                    uint32_t ah, al, bh;
                    if (xres) {
                        ah = tc::smem_u32(smem) + kc * kCgABytes;
                        al = ah + kCgXHalf;
                        bh = tc::smem_u32(smem + 2 * kCgXHalf + sb * 2 * kCgBBytes);
                    } else {
                        ah = tc::smem_u32(smem + sb * kCgStageBytes);
                        al = ah + kCgABytes;
                        bh = ah + 2 * kCgABytes;
                    }
                    const uint32_t bl = bh + kCgBBytes;
                    const uint32_t d = tmem + 256u * ab;
#pragma unroll
                    for (int ks = 0; ks < kCgKR / 16; ++ks) {
                        const int kg = (kCgKR / 16) * kc + ks;
                        const uint32_t oa = ks * 4096, ob = ks * 5120;
                        const uint32_t acc0 = kg > 0 ? 1u : 0u;
                        tc::mma_f16(d, tc::smem_desc(ah + oa, 2048, 128), tc::smem_desc(bh + ob, 2560, 128), idesc, acc0);
                        tc::mma_f16(d, tc::smem_desc(ah + oa, 2048, 128), tc::smem_desc(bl + ob, 2560, 128), idesc, 1u);
                        tc::mma_f16(d, tc::smem_desc(al + oa, 2048, 128), tc::smem_desc(bh + ob, 2560, 128), idesc, 1u);
                    }
                    tc::mma_commit(&sh.st_empty[sb]);  // the stage is free once these MMAs finish
                }
                tc::mma_commit(&sh.acc_full[ab]);
                // last tile on these x rows: they may be replaced once its MMAs finish
                if (xres && n + 1 < t1 && (n + 1) / JB != n / JB) tc::mma_commit(&sh.x_empty);
            }
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------------- epilogue
        // warp w reads TMEM lane quarter q = w & 3 (rows i0 + 32 q + lane);
        // the G warps of a quarter split its five 32-column chunks and write
        // the costs straight into the skewed image of strip s = 4 ib + q
        // (stage[kk - j0][t] = d(32 s + t, kk - t): address 32 r + t, so a
        // warp's stores hit 32 distinct banks); the image of rows
        // [j0, rend) is contiguous in dsk and leaves with ONE bulk store
        constexpr int G = kCgEpiWarps / 4;  // warps per lane quarter
        const int q = warp & 3, hf = warp >> 2;
        float *stage = reinterpret_cast<float *>(smem + kCgStages * kCgStageBytes) + q * kCgStageRows * 32;
        const bool leader = hf == 0 && lane == 0;  // issues the quarter's bulk store
        // the cost stream must not push the operands (re-read per tile row) out of L2
        const uint64_t st_policy = tc::l2_evict_first_policy();
        const int zb = (5 * hf) / G, ze = (5 * (hf + 1)) / G;  // this warp's 32-column chunks
        int li = 0;
        for (int n = t0; n < t1; ++n, ++li) {
            int b, ib, jb;
            tile_of(n, b, ib, jb);
            const int i0 = 128 * ib, j0 = 128 * jb;
            const int ab = li & 1;
            const float m2 = -2.0f * split_scale(absmax + 2 * b).inv;
            const int i = i0 + 32 * q + lane;
            const bool row_ok = i < N;
            const float xi = row_ok ? xn[(size_t)b * N + i] : 0.f;
            const bool last = jb == JB - 1;
            const int rows = (last ? KK : min(j0 + 128, KK)) - j0;  // skewed rows of this tile (<= 160)
            float yv[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int j = j0 - 32 + 32 * (zb + u) + lane;
                yv[u] = (zb + u < ze && j >= 0 && j < M) ? yn[(size_t)b * M + j] : 0.f;
            }
            tc::mbar_wait(&sh.acc_full[ab], (li >> 1) & 1);
            tc::tc_fence_after();
            // the quarter's image is free once its previous bulk store has read it
            if (leader) tc::bulk_wait_read0();
            named_bar_cg(2 + q, 32 * G);
            const bool interior = j0 >= 32 && j0 + 128 <= M && bw == 0 && i0 + 128 <= N;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int z = zb + u;
                if (z >= ze) break;
                float acc[32];
                tc::tmem_ld32(tmem + 256u * ab + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * z), acc);
                const int jz = j0 - 32 + 32 * z;
                const int r0 = 32 * (z - 1) + lane;  // skewed row of element e: r0 + e
                float *st = stage + r0 * 32 + lane;
                if (interior) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float v = tc_cost(acc[e], xi, __shfl_sync(kFull, yv[u], e), m2, true);
                        if (r0 + e >= 0 && r0 + e < rows) st[e * 32] = v;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float yj = __shfl_sync(kFull, yv[u], e);
                        const int j = jz + e;
                        const bool ok = row_ok && j >= 0 && j < M && in_band(i + 1, j + 1, bw);
                        const float v = tc_cost(acc[e], xi, yj, m2, ok);
                        if (r0 + e >= 0 && r0 + e < rows) st[e * 32] = v;
                    }
                }
            }
            // this warp's TMEM reads are complete: release the accumulator
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sh.acc_empty[ab]);
            // last column block: skewed rows past the computed columns
            // (j = kk - t >= j0 + 128 >= M) are zero
            if (hf == 0 && rows > 128)
                for (int r = 128 + lane; r < rows; ++r) stage[r * 32 + lane] = 0.f;
            tc::fence_async_smem();  // generic-proxy writes -> the bulk copy engine
            named_bar_cg(2 + q, 32 * G);
            const int s = 4 * ib + q;
            if (leader && 32 * s < N)
                tc::bulk_s2g_hint(dsk + (((size_t)b * S + s) * (size_t)KK + j0) * 32, stage, (uint32_t)rows * 128u,
                                  st_policy);
        }
        if (leader) tc::bulk_wait0();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

}  // namespace sdtw
