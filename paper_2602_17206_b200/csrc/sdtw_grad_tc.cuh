// sdtw_grad_tc.cuh — the input-gradient contraction on the tensor cores
// (fp32 engine).
//
// Reference: input_gradients (backward.hpp:208-266):
//   dX_i = 2 (x_i sum_j E_ij - sum_j E_ij y_j),  dY_j = 2 (y_j sum_i E_ij - sum_i E_ij x_i).
// The buckets and their fixed tile order are those of contract_ordered_kernel
// (sdtw_grad.cuh): a strip's own slots for dX, a chunk's tiles in strip order
// for dY.  Per work item (bucket, 128-feature block) the dot products
//   acc[d][o] = sum over the bucket's tiles, in order, of sum_m P[m][d] E(o, m)
// (o = output row, m = partner index, P = the partner rows: the y chunk for
// dX, the x strip for dY) are one tcgen05.mma chain into a 128 x 32 fp32 TMEM
// accumulator: A = P^T (M = 128 features, K = 32 partners), B = E (N = 32
// outputs, K = 32), both staged as K-major SWIZZLE_NONE fp16 images with the
// 3-pass hi/lo split of the cost GEMM (hi*hi + hi*lo + lo*hi, fp32
// accumulation; E scaled by 2^15, P by its pair's power-of-two scale), two
// stages so that tile e + 1 is staged while tile e's MMAs run, and tile
// e + 1's operands are loaded into registers while tile e is split and
// staged.  The kernel holds TMEM, so it runs one CTA per SM; the CTA carries
// kCtGroups independent 4-warp groups (own work items, accumulator columns,
// stages, barriers) to keep several items' loads in flight.  Marginals are
// fp64 sums of the fp32 E values; grad = 2 (v marg - acc) in fp64, as in the
// FMA kernel.  Deterministic: a fixed MMA sequence per work item, no atomics.
#pragma once
#include "sdtw_common.cuh"
#include "sdtw_dp2.cuh"
#include "sdtw_grad.cuh"
#include "sdtw_fused.cuh"
#include "sdtw_tc.cuh"

namespace sdtw {

constexpr int kCtListStrips = 2048;  // == max_list_strips<float>() (sdtw_grad.cuh)
constexpr int kCtGroups = 4;         // independent 4-warp groups per CTA
constexpr int kCtThreads = 128 * kCtGroups;
constexpr int kCtA = 128 * 32 * 2;   // one fp16 A image (128 features x 32 partners)
constexpr int kCtB = 32 * 32 * 2;    // one fp16 B image (32 outputs x 32 partners)
constexpr int kCtStage = 2 * kCtA + 2 * kCtB;  // hi + lo of both
constexpr int kCtGroupSmem = 2 * kCtStage;     // two stages per group

struct CtGroupShared {
    uint64_t mma_done[2];  // the MMAs that read stage s finished
    double marg[4][32];    // per-warp partial marginals
    int wcnt[4];
    int lst[kCtListStrips];
};

template <int kTU = 0>
__global__ void __launch_bounds__(kCtThreads, 1)
    contract_tc_kernel(const float *__restrict__ tiles, const int4 *__restrict__ meta, const int *__restrict__ strip_tiles,
                       int quota, const int *__restrict__ off, const int *__restrict__ ord, int which, int B, int S,
                       int C, int N, int M, int D, const float *__restrict__ vout, const float *__restrict__ vpart,
                       const unsigned *__restrict__ absmax, float *__restrict__ grad)
{
    extern __shared__ __align__(128) uint8_t ct_smem[];
    __shared__ CtGroupShared gsh[kCtGroups];
    __shared__ uint32_t tmem_base;
    const int gid = threadIdx.x >> 7;            // group
    const int tid = threadIdx.x & 127;           // thread within the group
    const int warp = tid >> 5, lane = tid & 31;  // warp within the group = TMEM lane quarter
    CtGroupShared &sh = gsh[gid];
    uint8_t *gsmem = ct_smem + (size_t)gid * kCtGroupSmem;
    if (tid == 0) {
        tc::mbar_init(&sh.mma_done[0], 1);
        tc::mbar_init(&sh.mma_done[1], 1);
        tc::fence_barrier_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc<32 * kCtGroups>(&tmem_base);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tmem_base + 32u * gid;  // this group's 32 accumulator columns
    auto gbar = [&]() { named_bar(1 + gid, 128); };
    const uint32_t idesc = tc::idesc_f16_f32(128, 32);
    uint32_t phase[2] = {0u, 0u};  // completed MMA batches per stage (parity)
    int pending[2] = {0, 0};       // stage s has MMAs in flight
    const int per_b = which == 0 ? S : C;
    const int Rout = which == 0 ? N : M, Rpart = which == 0 ? M : N;
    const int nkb = (D + 127) / 128;
    const int nitems = B * per_b * nkb;
    // items spread over the CTAs first (one group per SM before a second)
    for (int item = gid * gridDim.x + blockIdx.x; item < nitems; item += gridDim.x * kCtGroups) {
        const int key = item / nkb, kb = 128 * (item % nkb);
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
            // the chunk's tiles in strip order (each strip holds at most one
            // tile of a chunk), compacted 128 strips at a time
            int n = 0;
            for (int sb = 0; sb < S; sb += 128) {
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
                gbar();  // lst / wcnt of the previous round consumed
                if (lane == 0) sh.wcnt[warp] = __popc(bal);
                gbar();
                int pre = n;
                for (int q = 0; q < warp; ++q) pre += sh.wcnt[q];
                if (found >= 0) sh.lst[pre + __popc(bal & ((1u << lane) - 1u))] = found;
                for (int q = 0; q < 4; ++q) n += sh.wcnt[q];
            }
            gbar();
            lo = 0;
            hi = n;
            ordp = sh.lst;
        }
        const float *vo = vout + (size_t)b * Rout * D;
        const float *vp = vpart + (size_t)b * Rpart * D;
        float *g = grad + (size_t)b * Rout * D;
        const int kf = kb + tid;               // this thread's feature in the A staging
        const int ke = kb + 32 * warp + lane;  // and in the epilogue (TMEM lane)
        if (lo == hi) {
            // no non-zero E tile touches this block: the gradient is exactly 0
            if (ke < D)
                for (int o = 0; o < 32 && o0 + o < Rout; ++o) g[(size_t)(o0 + o) * D + ke] = 0.f;
            continue;
        }
        const SplitScale sc = split_scale(absmax + 2 * b);
        const float ps = which == 0 ? sc.sy : sc.sx;  // partner operand scale
        const float es = 32768.f;                     // E <= 1: 2^15 keeps small E in fp16's normal range
        double marg = 0.0;                            // thread (o = lane, partner group warp) partial
        // operands of one tile in registers: 32 partner values of feature kf,
        // 8 E values of (o = lane, partners 8 warp ..)
        float rp[32], re[8];
        auto load_tile = [&](int e) {
            const int idx = which == 0 ? e : ordp[e];
            const int4 m = meta[idx];
            const float *et = tiles + (size_t)idx * 1024;  // [r][jj]
            const int p0 = which == 0 ? 32 * m.z : 32 * m.y;
            const int np = which == 0 ? m.w : min(32, N - 32 * m.y);
#pragma unroll
            for (int mm = 0; mm < 32; ++mm) rp[mm] = (mm < np && kf < D) ? vp[(size_t)(p0 + mm) * D + kf] : 0.f;
#pragma unroll
            for (int r = 0; r < 8; ++r)
                re[r] = which == 0 ? et[lane * 32 + 8 * warp + r] : et[(8 * warp + r) * 32 + lane];
        };
        load_tile(lo);
        for (int e = lo; e < hi; ++e) {
            const int st = (e - lo) & 1;
            uint8_t *ah = gsmem + (size_t)st * kCtStage, *al = ah + kCtA;
            uint8_t *bh = al + kCtA, *bl = bh + kCtB;
            // the stage's previous MMAs (tile e - 2) must have read it
            if (pending[st]) {
                tc::mbar_wait(&sh.mma_done[st], phase[st] & 1u);
                ++phase[st];
                pending[st] = 0;
            }
            // A = P^T (feature kf, partners in 4 K-blocks of 8)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float4 v[2];
                v[0] = make_float4(rp[8 * q], rp[8 * q + 1], rp[8 * q + 2], rp[8 * q + 3]);
                v[1] = make_float4(rp[8 * q + 4], rp[8 * q + 5], rp[8 * q + 6], rp[8 * q + 7]);
                tc::split_store8_regs(v, ps, ah, al, tc::kmajor_off(tid, q, 2048));
            }
            // B = E as (output o, partner m): dX o = r, m = jj (rows of the
            // tile); dY o = jj, m = r (columns); thread = (o = lane, 8-partner group warp)
            {
                double s8 = 0.0;
#pragma unroll
                for (int r = 0; r < 8; ++r) s8 += (double)re[r];
                marg += s8;
                float4 v[2];
                v[0] = make_float4(re[0], re[1], re[2], re[3]);
                v[1] = make_float4(re[4], re[5], re[6], re[7]);
                tc::split_store8_regs(v, es, bh, bl, tc::kmajor_off(lane, warp, 512));
            }
            tc::fence_async_smem();
            gbar();
            if (e + 1 < hi) load_tile(e + 1);  // in flight during the MMAs
            if (tid == 0) {
                tc::tc_fence_after();
                const uint32_t a_h = tc::smem_u32(ah), a_l = tc::smem_u32(al);
                const uint32_t b_h = tc::smem_u32(bh), b_l = tc::smem_u32(bl);
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t oa = ks * 2 * 2048, ob = ks * 2 * 512;
                    const uint32_t acc0 = (e > lo || ks > 0) ? 1u : 0u;
                    tc::mma_f16(tmem, tc::smem_desc(a_h + oa, 2048, 128), tc::smem_desc(b_h + ob, 512, 128), idesc, acc0);
                    tc::mma_f16(tmem, tc::smem_desc(a_h + oa, 2048, 128), tc::smem_desc(b_l + ob, 512, 128), idesc, 1u);
                    tc::mma_f16(tmem, tc::smem_desc(a_l + oa, 2048, 128), tc::smem_desc(b_h + ob, 512, 128), idesc, 1u);
                }
                tc::mma_commit(&sh.mma_done[st]);
            }
            pending[st] = 1;
        }
        sh.marg[warp][lane] = marg;
        // the first half of the epilogue's v values, loaded while the last MMAs run
        float vv[16];
#pragma unroll
        for (int o = 0; o < 16; ++o) vv[o] = (o0 + o < Rout && ke < D) ? vo[(size_t)(o0 + o) * D + ke] : 0.f;
        // all MMAs of the item done
        for (int q = 0; q < 2; ++q) {
            if (pending[q]) {
                tc::mbar_wait(&sh.mma_done[q], phase[q] & 1u);
                ++phase[q];
                pending[q] = 0;
            }
        }
        tc::tc_fence_after();
        gbar();
        // epilogue: warp w holds features kb + 32 w + lane, outputs o = 0..31,
        // in two halves of 16 columns
        const float unscale = 1.0f / (ps * es);  // exact: powers of two
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float acc[16];
            tc::tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16u * h, acc);
            if (h == 1) {
#pragma unroll
                for (int o = 0; o < 16; ++o)
                    vv[o] = (o0 + 16 + o < Rout && ke < D) ? vo[(size_t)(o0 + 16 + o) * D + ke] : 0.f;
            }
            if (ke < D) {
#pragma unroll
                for (int o = 0; o < 16; ++o) {
                    const int oo = 16 * h + o;
                    if (o0 + oo >= Rout) break;
                    const double mg = ((sh.marg[0][oo] + sh.marg[1][oo]) + sh.marg[2][oo]) + sh.marg[3][oo];
                    g[(size_t)(o0 + oo) * D + ke] = (float)(2.0 * ((double)vv[o] * mg - (double)(acc[o] * unscale)));
                }
            }
        }
        tc::tc_fence_before();
        gbar();  // TMEM and marginals consumed before the next item overwrites them
    }
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc<32 * kCtGroups>(tmem_base);
}

}  // namespace sdtw
