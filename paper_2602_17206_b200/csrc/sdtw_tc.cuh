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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
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

// max |v| over a float array -> atomicMax on the bit pattern (non-negative floats
// order like their bits).
__global__ void absmax_kernel(const float *__restrict__ v, size_t n, unsigned *out)
{
    float m = 0.f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(v[i]));
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// Power-of-two operand scales: |x * sx| <= 2^14, and 1/(sx sy).
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

// Norms in double, rounded once (the cost epilogue's largest terms).
__global__ void norms_f32_kernel(const float *__restrict__ x, int rows, int D, float *__restrict__ out)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float *e = x + (size_t)r * D;
    double s = 0.0;
    for (int k = 0; k < D; ++k) s = fma((double)e[k], (double)e[k], s);
    out[r] = (float)s;
}

// ----------------------------------------------------------------------------
// Unfused cost tensor on tcgen05: one CTA per (pair, 128-row block, 128-column
// block).  Output in the DP's skewed strip layout dsk[b][s][kk][t] =
// d(32 s + t + 1, kk - t + 1) (0-based kk row of KK = row_pitch rows), so
// that every DP warp step reads one 128-byte line.  The epilogue stages the
// 32 x 128 block of each warp in shared memory and writes whole skewed rows
// (rows shared with a neighbouring CTA are lane-masked).
// ----------------------------------------------------------------------------
constexpr int kCgRows = 128, kCgCols = 128, kCgK = 64;
constexpr int kCgTile = kCgRows * kCgK * 2;  // bytes of one fp16 operand tile (16 KB)
constexpr int kCgStagePitch = kCgCols + 2;  // floats; odd bank step for skewed reads (2-way on writes)
constexpr int kCgSmem = 4 * 32 * kCgStagePitch * 4;  // >= 4 operand tiles (64 KB); reused by the staging

__global__ void __launch_bounds__(128, 1)
    cost_gemm_tc_kernel(const float *__restrict__ x, const float *__restrict__ y,
                        const float *__restrict__ xn, const float *__restrict__ yn, const unsigned *absmax,
                        int B, int N, int M, int D, int S, int KK, int bw, float *__restrict__ dsk)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *a_hi = smem, *a_lo = smem + kCgTile, *b_hi = smem + 2 * kCgTile, *b_lo = smem + 3 * kCgTile;
    __shared__ uint64_t mma_bar;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.z;
    const int i0 = blockIdx.y * kCgRows, j0 = blockIdx.x * kCgCols;
    const SplitScale sc = split_scale(absmax);

    if (warp == 0) tc::tmem_alloc<128>(&tmem_base);
    if (tid == 0) {
        tc::mbar_init(&mma_bar, 1);
        tc::fence_barrier_init();
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base;

    const float *xb = x + (size_t)b * N * D, *yb = y + (size_t)b * M * D;
    const uint32_t idesc = tc::idesc_f16_f32(128, kCgCols);
    const int kchunks = (D + kCgK - 1) / kCgK;
    const bool vec = (D & 7) == 0;
    uint32_t phase = 0;
    // Operand chunks (X rows [i0, i0+128), Y rows [j0, j0+128), features
    // [64 kc, 64 kc + 64)) go through registers: the loads of chunk kc + 1 are
    // in flight while the MMAs of chunk kc run.  Thread item i: row
    // (tid + 128 i) >> 3, K block (tid + 128 i) & 7.
    float4 px[8][2], py[8][2];
    auto load_chunk = [&](int kc) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int u = tid + 128 * i;
            const int r = u >> 3, kb = u & 7;
            const int k = kc * kCgK + kb * 8;
            const int nk = max(0, min(8, D - k));
            const int nx = i0 + r < N ? nk : 0, ny = j0 + r < M ? nk : 0;
            const float *sx = xb + (size_t)min(i0 + r, N - 1) * D + min(k, D - 1);
            const float *sy = yb + (size_t)min(j0 + r, M - 1) * D + min(k, D - 1);
            if (vec && nx == 8) {
                px[i][0] = __ldg(reinterpret_cast<const float4 *>(sx));
                px[i][1] = __ldg(reinterpret_cast<const float4 *>(sx) + 1);
            } else {
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = e < nx ? sx[e] : 0.f;
                px[i][0] = make_float4(f[0], f[1], f[2], f[3]);
                px[i][1] = make_float4(f[4], f[5], f[6], f[7]);
            }
            if (vec && ny == 8) {
                py[i][0] = __ldg(reinterpret_cast<const float4 *>(sy));
                py[i][1] = __ldg(reinterpret_cast<const float4 *>(sy) + 1);
            } else {
                float f[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = e < ny ? sy[e] : 0.f;
                py[i][0] = make_float4(f[0], f[1], f[2], f[3]);
                py[i][1] = make_float4(f[4], f[5], f[6], f[7]);
            }
        }
    };
    auto store_chunk = [&]() {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int u = tid + 128 * i;
            const uint32_t off = tc::kmajor_off(u >> 3, u & 7, 2048);
            tc::split_store8_regs(px[i], sc.sx, a_hi, a_lo, off);
            tc::split_store8_regs(py[i], sc.sy, b_hi, b_lo, off);
        }
    };
    load_chunk(0);
    for (int kc = 0; kc < kchunks; ++kc) {
        if (kc > 0) {
            // the previous chunk's MMAs still read the operand tiles
            tc::mbar_wait(&mma_bar, phase);
            phase ^= 1u;
            tc::tc_fence_after();
        }
        store_chunk();
        if (kc + 1 < kchunks) load_chunk(kc + 1);
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::tc_fence_after();
            const uint32_t ah = tc::smem_u32(a_hi), al = tc::smem_u32(a_lo);
            const uint32_t bh = tc::smem_u32(b_hi), bl = tc::smem_u32(b_lo);
#pragma unroll
            for (int ks = 0; ks < kCgK / 16; ++ks) {
                const uint32_t o = ks * 2 * 2048;
                const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
                tc::mma_f16(tmem, tc::smem_desc(ah + o, 2048, 128), tc::smem_desc(bh + o, 2048, 128), idesc, acc0);
                tc::mma_f16(tmem, tc::smem_desc(ah + o, 2048, 128), tc::smem_desc(bl + o, 2048, 128), idesc, 1u);
                tc::mma_f16(tmem, tc::smem_desc(al + o, 2048, 128), tc::smem_desc(bh + o, 2048, 128), idesc, 1u);
            }
            tc::mma_commit(&mma_bar);
        }
        __syncwarp();
    }
    tc::mbar_wait(&mma_bar, phase);
    phase ^= 1u;
    tc::tc_fence_after();

    // epilogue: warp w owns TMEM lanes 32w..32w+31 = rows i0 + 32w + lane
    float *stage = reinterpret_cast<float *>(smem) + warp * 32 * kCgStagePitch;  // [t][jj]
    const int i = i0 + 32 * warp + lane;  // 0-based row
    const bool row_ok = i < N;
    const float xi = row_ok ? xn[(size_t)b * N + i] : 0.f;
    const float m2 = -2.0f * sc.inv;
#pragma unroll 1
    for (int cc = 0; cc < kCgCols / 32; ++cc) {
        float acc[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * cc), acc);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int j = j0 + 32 * cc + e;
            float v = 0.f;
            if (row_ok && j < M && in_band(i + 1, j + 1, bw)) {
                v = fmaf(m2, acc[e], xi + yn[(size_t)b * M + j]);
                v = v < 0.f ? 0.f : v;
            }
            stage[lane * kCgStagePitch + 32 * cc + e] = v;
        }
    }
    __syncwarp();
    const int s = (i0 >> 5) + warp;
    if (32 * s < N) {
        float *ds = dsk + ((size_t)b * S + s) * (size_t)KK * 32;
        // skewed rows kk = j + t over this block's columns j in [j0, j0 + 128)
        const int kk_lo = j0, kk_hi = min(j0 + kCgCols, M) - 1 + 31;
        for (int kk = kk_lo; kk <= kk_hi; ++kk) {
            const int jl = kk - lane - j0;  // local column of this lane
            if (jl >= 0 && jl < kCgCols && j0 + jl < M) ds[(size_t)kk * 32 + lane] = stage[lane * kCgStagePitch + jl];
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

}  // namespace sdtw
