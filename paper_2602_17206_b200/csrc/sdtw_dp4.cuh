// sdtw_dp4.cuh — backward DP with a short critical path.
//
// The v3 backward (sdtw_dp3.cuh) computed, per live 32x32 tile, the recompute
// (phase R, ~63 skewed steps on the MUFU chain) and then the reverse E sweep
// (phase E), and handed the tile's top-row S to the strip above only at the
// end: the critical path was (#live tiles on the band) x (R + E), ~25 us each.
// Here:
//   * each strip publishes a tile's LIVE/DEAD status as soon as it decides
//     it, so the strip above recomputes its own tile (phase R) while this one
//     still works;
//   * a live tile's recompute also recomputes the next tile to the left
//     speculatively (two independent tiles in one loop: ILP 2), because the
//     alignment band usually continues there;
//   * phase E hands S to the strip above every 8 columns, and consumes the
//     strip below's S every 8 columns (tagged entries, prefetched), so E
//     sweeps of consecutive strips overlap like the forward's strips do;
//   * runs of dead tiles are skipped 32 chunks per status load.
// Tile skipping, checkpoints and the gradient hand-off are those of v3.
#pragma once
#include <type_traits>
#include "sdtw_common.cuh"
#include "sdtw_dp2.cuh"
#include "sdtw_dp3.cuh"
#include "sdtw_fused.cuh"

namespace sdtw {

// Tile status (per strip, per chunk): DEAD = the tile passes no E upward (its
// top row's S is all zero; final), HINT = being processed (its S arrives per
// 8 columns; lets the strip above start recomputing), LIVE = final, non-zero S.
// COMMIT+k (k = 0, 1): the strip committed to the tile without evidence yet
// (k = 0) or is recomputing it speculatively because the strip below did
// (k = 1); strips above start their own recompute early on it, two levels
// deep at most, so the recompute leaves the critical path without
// cascading up whole columns.
enum : unsigned { kTileDead = 1u, kTileHint = 2u, kTileLive = 3u, kTileCommit = 4u };
#ifndef BWD_STATUS_SLEEP_NS
#define BWD_STATUS_SLEEP_NS 32
#endif
constexpr unsigned kSpecDepth = 2;

// Recompute window: tiles per recompute request (ILP of the helper's skewed
// loop); the probability cache holds two windows.  3 for the tensor-core
// fused path (TMEM limits it to one CTA per SM anyway), 2 otherwise: the
// 4-slot cache (51 KB) fits three workers per SM instead of two, so 1.5x
// more strips are in flight (the backward is occupancy-bound at C3 / C5:
// 4096 / 16384 strips against 296 workers).
template <bool kTc>
constexpr int bwd_window() { return kTc ? 3 : 2; }

template <class T, bool kFused, bool kTc = false, int kWin = bwd_window<kTc>()>
struct Bwd4Smem {
    // kTc: the strip's x rows as a packed fp16 hi/lo tensor-core operand
    // (32 rows x kFtcMaxD), placed first so that the unused rows 32..127 of
    // the M = 128 MMA read (harmlessly) into the probability slots after it
    static constexpr int kX = kTc ? kFtcMaxD * 32 * 4 / (int)sizeof(T) : 0;
    static constexpr int kSlot = 3 * 33 * 32;            // pd, pu, pl [jj][t], row 32 = dummy
    static constexpr int kP = 2 * kWin * kSlot;          // two windows of probability tiles
    static constexpr int kE = 32 * 34;                   // E tile [t][jj] (even stride: conflict-free), column 32 = dummy
    static constexpr int kRing = (kFused && !kTc) ? 0 : 4 * 1024;  // skewed cost row groups (slot g & 3)
    static constexpr int kHalo = 6 * 32;                 // 3 top halos (h), S in, S out (+dummy)
    static constexpr int kBar = kTc ? 16 / (int)sizeof(T) + 2 : 0;  // 2 mbarriers + TMEM base (kTc)
    static constexpr int kCtl = 64 / (int)sizeof(T);                 // 16 ints: warp hand-off block
    static constexpr int kPerWarp = kX + kP + kE + kRing + kHalo + kBar + kCtl;  // per worker (2 warps)
    // per-worker stride in bytes (operand images need 16-byte alignment)
    static constexpr size_t kWorkerBytes = ((size_t)kPerWarp * sizeof(T) + 1023) / 1024 * 1024;
};

// Status words: (epoch << 32) | status.
__device__ __forceinline__ void put_status(unsigned long long *p, unsigned v, unsigned tag)
{
    const unsigned long long w = ((unsigned long long)tag << 32) | v;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w));
}
__device__ __forceinline__ unsigned get_status(const unsigned long long *p, unsigned tag)
{
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p));
    return (unsigned)(w >> 32) == tag ? (unsigned)(w & 0xffffffffull) : 0u;
}

// Interior recompute cell: the forward softmin plus its three probabilities
// (3 ex2 + lg2 + rcp; one Newton step keeps pd + pu + pl = 1 within an ulp).
template <class T>
__device__ __forceinline__ void prob_cell(T d, T u, T l, T k, T gln2, T &v, T &h, T &pd, T &pu, T &pl)
{
    const T mn = tmin(tmin(u, l), T(0));
    const T e0 = Num<T>::ex2(mn * k);
    const T eu = Num<T>::ex2((mn - u) * k);
    const T el = Num<T>::ex2((mn - l) * k);
    const T s = (e0 + eu) + el;
    T r = Num<T>::rcp(s);
    r = r * (T(2) - s * r);
    const T sm = mn - gln2 * Num<T>::lg2(s);
    v = (d - u) + sm;
    h = (d - l) + sm;
    pd = e0 * r;
    pu = eu * r;
    pl = el * r;
}

template <class T, bool kFused>
__device__ __forceinline__ T bwd_cost(const DpArgs<T> &a, const T *ring, int b, int s, int t, int i, int j)
{
    if (kFused) return in_band(i, j, a.bw) ? load_cost<T, true>(a, b, s, t, i, j) : T(0);
    const int kk = (j - 1) + t;  // skewed row of (i, j)
    return ring[((kk >> 5) & 3) * 1024 + (kk & 31) * 32 + t];
}

// kTc (fp32 fused mode): the cost blocks of the recomputed tiles come from
// tcgen05.mma (sdtw_fused.cuh) into TMEM, through the same epilogue and into
// the same skewed ring the unfused path fills from the cost tensor.  The warp
// is warp 0 of its CTA, so it owns TMEM lanes 0..31: its strip's 32 rows are
// rows 0..31 of an M = 128 MMA whose other rows are don't-care.
// Workers: a worker = (recompute helper warp, E warp) on one strip at a time.
// kTc kernels hold TMEM, which limits them to one CTA per SM, so a kTc CTA
// carries two independent workers (helper w owns TMEM lane quarter w and the
// rows 32 w .. of its M = 128 MMAs); other variants run one worker per CTA.
template <bool kTc>
constexpr int bwd_workers() { return kTc ? 2 : 1; }

template <class T, bool kFused, bool kTc = false, int kWin = bwd_window<kTc>()>
__global__ void __launch_bounds__(64 * bwd_workers<kTc>(), 1) sdtw_backward4_kernel(Dp3Args<T> A,
                                                                                   unsigned long long *stat,
                                                                                   FusedTcArgs F)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __shared__ uint32_t tmem_slot;
    // band-cache rerun: nothing to do unless the banded pass missed the band
    // (uniform over the grid, before any barrier or TMEM allocation)
    if (A.band_gate && *reinterpret_cast<volatile unsigned *>(&A.stats[3]) == 0u) return;
    constexpr int kW = bwd_workers<kTc>();
    const DpArgs<T> &a = A.a;
    using SM = Bwd4Smem<T, kFused, kTc, kWin>;
    using TG = Tagged<T>;
    const int t = threadIdx.x & 31;
    const int wk = (threadIdx.x >> 5) % kW;    // worker
    const int warp = (threadIdx.x >> 5) / kW;  // role: 0 recompute helper, 1 E sweep
    uint8_t *wsm = smem_raw + (size_t)wk * SM::kWorkerBytes;
    uint8_t *xs = wsm;  // kTc: packed x rows of the strip
    T *base = reinterpret_cast<T *>(wsm) + SM::kX;
    // kTc: [0] MMA done, [1] operand copies landed; then the TMEM base
    uint64_t *tc_bar = reinterpret_cast<uint64_t *>(base + SM::kP + SM::kE + SM::kRing + SM::kHalo);
    uint32_t &tc_tmem = *reinterpret_cast<uint32_t *>(tc_bar + 2);
    uint32_t tc_ph[2] = {0u, 0u};
    uint32_t tmem = 0;
    float tc_m2 = 0.f;
    // warp hand-off block: [0] ticket, [1] requested window, [2] request
    // sequence, [3] strip done, [4] E position, [5..6] window start of slot
    // group g, [7..8] group state (0 empty, 1 computing, 2 ready)
    volatile int *ctl = reinterpret_cast<volatile int *>(base + SM::kP + SM::kE + SM::kRing + SM::kHalo + SM::kBar);
    (void)tc_tmem;
    if constexpr (kTc) {
        if (warp == 0 && t == 0) {
            tc::mbar_init(&tc_bar[0], 1);
            tc::mbar_init(&tc_bar[1], 1);
            tc::fence_barrier_init();
        }
        if (threadIdx.x < 32) tc::tmem_alloc<128 * kW>(&tmem_slot);
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
        tmem = tmem_slot + 128u * wk;  // this worker's 128 columns
    }
    const uint32_t tmem_lanes = (uint32_t)(32 * wk) << 16;  // lane quarter of the helper
    // probability tile slots k = 0..2 at base + kSlot k: pd, pu, pl [jj][t]
    constexpr int kSlot = SM::kSlot;
    T *et_s = base + SM::kP;
    T *ring = et_s + SM::kE;
    T *halo_s = ring + SM::kRing;  // [3][32] top halos of the recomputed tiles
    T *sin_s = halo_s + 96;
    T *sout_s = sin_s + 32;
    const unsigned epoch = A.epoch;
    const int total = a.B * a.S;
    const int ngroups_row = a.KK / 32;
    for (;;) {
        if (warp == 1) {
            const unsigned tk1 = warp_ticket(&a.tickets[1]);
            if (t == 0) {
                ctl[0] = (int)tk1;
                ctl[1] = -1;
                ctl[2] = 0;
                ctl[3] = 0;
                ctl[4] = a.C;
                ctl[5] = ctl[6] = -1000;
                ctl[7] = ctl[8] = 0;
            }
        }
        named_bar(1 + wk, 64);
        const unsigned tk = (unsigned)ctl[0];
        named_bar(1 + wk, 64);
        if ((int)tk >= total) break;
        const int s = a.S - 1 - (int)tk / a.B, b = (int)tk % a.B;
        const FxScales fx = fx_scales(A.absmax + 2 * b, a.N, a.M);
        if constexpr (kTc) tc_m2 = -2.0f * split_scale(A.absmax + 2 * b).inv;
        const int i = 32 * s + t + 1;
        const bool row_ok = i <= a.N;
        bool x_loaded = false;
        const float tc_xi = (kTc && row_ok) ? (float)a.xn[(size_t)b * a.N + i - 1] : 0.f;
        const bool bottom = s == a.S - 1;
        // unfused: the strip's skewed cost rows; band cache: its cached
        // groups [glo, glo + band_ng)
        const bool banded = !kFused && !kTc && A.band != nullptr;
        const int glo = banded ? band_lo(s, a.N, a.M, ngroups_row, A.band_ng) : 0;
        const T *dsrc = kFused ? nullptr
                        : banded ? A.band + ((size_t)b * a.S + s) * (size_t)A.band_ng * 1024
                                 : a.dsk + ((size_t)b * a.S + s) * (size_t)a.KK * 32;
        unsigned long long *stat_me = stat + ((size_t)b * a.S + s) * a.C;
        const unsigned long long *stat_below = stat + ((size_t)b * a.S + s + 1) * a.C;
        typename TG::Ent *sb_me = A.sbt + ((size_t)b * a.S + s) * a.M;
        const typename TG::Ent *sb_below = A.sbt + ((size_t)b * a.S + s + 1) * a.M;
        if (A.trace && t == 0 && warp == 1) A.trace[2 * ((size_t)a.B * a.S + (size_t)b * a.S + s)] = global_ns();
        int ntiles = 0;
        int nstored = 0;  // tiles of this strip in the store
        // cycle accounting (trace mode): [32 B S + 8 (b S + s) + e]: e = 0
        // recompute, 1 S wait, 2 E steps, 3 status waits, 4 tile epilogue, 5 other
        long long cyc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long c_mark = A.trace ? clock64() : 0;
        auto lap = [&](int e) {
            if (A.trace) {
                const long long now = clock64();
                cyc[e] += now - c_mark;
                c_mark = now;
            }
        };
        // event log (trace mode): up to 16 (time, chunk, kind) records per
        // strip at [40 B S + 48 (b S + s) + 3 k]; kinds 1/2 recompute
        // start/end, 3/4 E phase start/end
        int nev = 0;
        auto ev = [&](int kind, int chunk) {
            if (A.trace && t == 0 && nev < 16) {
                // E warp: [40 B S ..), helper: [88 B S ..)
                unsigned long long *r = A.trace + (warp == 1 ? 40 : 88) * (size_t)a.B * a.S +
                                        48 * ((size_t)b * a.S + s) + 3 * nev;
                r[0] = global_ns();
                r[1] = (unsigned long long)chunk;
                r[2] = (unsigned long long)kind;
                ++nev;
            }
        };
        T e_right = T(0), pl_right = T(0), pd_right = T(0);
        int grp = 0;  // slot group the helper is filling
        // which group holds tile cf (state >= 1), -1 if none
        auto group_of = [&](int cf) {
            for (int g = 0; g < 2; ++g) {
                const int w0 = ctl[5 + g];
                if (ctl[7 + g] != 0 && cf <= w0 && cf >= ctl[9 + g] && cf >= 0) return g;
            }
            return -1;
        };
        // kTc: cost blocks of chunks cr, cr-1, .. (nt of them) -> skewed ring.
        // Operands: the strip's x rows (loaded once per strip) and the y
        // chunks, staged K-half by K-half in the probability slots (free
        // until the recompute loop writes them).
        auto tc_costs = [&](int cr, int nt, bool &xl, int b_, int s_, int i_, bool rok, float xi) {
            if constexpr (kTc) {
                const int dpad = F.dpad;
                // operand staging inside the target group's own slots (free)
                uint8_t *stage = reinterpret_cast<uint8_t *>(base + kSlot * kWin * grp);
                const uint32_t idesc = tc::idesc_f16_f32(128, 32);
                const SplitScale sc = split_scale(A.absmax + 2 * b_);
                // raw fp32 staging after the three fp16 operand tiles (the
                // probability slots, E tile and ring are all free until the
                // recompute loop / epilogue)
                lap(5);
                // column norms of the (up to) three chunks, loaded first
                float yv3[3];
#pragma unroll
                for (int z = 0; z < 3; ++z) {
                    const int jz = 32 * (cr - z) + t;
                    yv3[z] = (z < nt && jz < a.M) ? (float)a.yn[(size_t)b_ * a.M + jz] : 0.f;
                }
                float *raw = reinterpret_cast<float *>(stage + 2 * 8192);  // <= 34 KB of the 38 KB group
                const bool async_ok = (a.D & 3) == 0;
                const float *xg = reinterpret_cast<const float *>(a.x) + (size_t)b_ * a.N * a.D;
                const float *yg = reinterpret_cast<const float *>(a.y) + (size_t)b_ * a.M * a.D;
                if (!xl) {
                    if (async_ok) {
                        raw_rows_async(raw, xg, a.D, 32 * s_, 32, a.N, 0, dpad, a.D, t);
                        cp_async_commit();
                        cp_async_wait<0>();
                        __syncwarp();
                        split_raw_rows(raw, 32, dpad, sc.sx, xs, xs + 32 * dpad * 2, 0, 512, t);
                        __syncwarp();
                    } else {
                        stage_split_rows(xg, a.D, 32 * s_, 32, a.N, a.D, dpad, sc.sx, xs, t);
                    }
                    xl = true;
                }
                // units u = (chunk z, K half kh): raw rows by cp.async one unit
                // ahead, split into one of two stage buffers, MMAs per unit
                // (the per-element instruction sequence is unchanged: for each
                // chunk the K halves in order, 4 K steps of hi.hi, hi.lo,
                // lo.hi each)
                const int KH = dpad / 64, U = nt * KH;
                // A = rows 32 wk .. 32 wk + 31 of an M = 128 operand: the
                // descriptor starts 4 wk 8-row groups (SBO = 128 B) before the
                // strip's rows; the other rows read neighbouring shared memory
                const uint32_t xh = tc::smem_u32(xs) - 512u * wk, xlo = xh + 32u * dpad * 2;
                auto unit_raw = [&](int u) {
                    const int z = u / KH, kh = u % KH;
                    raw_rows_async(raw + (u & 1) * 32 * 68, yg, a.D, 32 * (cr - z), 32, a.M, 64 * kh, 64, a.D, t);
                    cp_async_commit();
                };
                bool pend[2] = {false, false};
                if (async_ok) unit_raw(0);
                for (int u = 0; u < U; ++u) {
                    const int z = u / KH, kh = u % KH, sb = u & 1;
                    uint8_t *st = stage + sb * 8192;
                    if (pend[sb]) {  // the MMAs of unit u - 2 read this stage buffer
                        tc::mbar_wait(&tc_bar[sb], tc_ph[sb]);
                        tc_ph[sb] ^= 1u;
                        pend[sb] = false;
                        tc::tc_fence_after();
                    }
                    if (async_ok) {
                        if (u + 1 < U) {
                            unit_raw(u + 1);
                            cp_async_wait<1>();
                        } else {
                            cp_async_wait<0>();
                        }
                        __syncwarp();
                        split_raw_rows(raw + sb * 32 * 68, 32, 64, sc.sy, st, st + 4096, 0, 512, t);
                    } else {
                        stage_split_rows(yg + (size_t)64 * kh, a.D, 32 * (cr - z), 32, a.M, a.D - 64 * kh, 64, sc.sy, st, t);
                    }
                    tc::fence_async_smem();
                    __syncwarp();
                    tc::tc_fence_after();
                    if (t == 0) {
                        const uint32_t bh = tc::smem_u32(st), bl = bh + 4096;
                        const uint32_t d = tmem + 32u * z;
                        for (int ks = 0; ks < 4; ++ks) {
                            const int kg = 4 * kh + ks;
                            const uint32_t oa = kg * 1024, ob = ks * 1024;
                            const uint32_t acc0 = kg > 0 ? 1u : 0u;
                            tc::mma_f16(d, tc::smem_desc(xh + oa, 512, 128), tc::smem_desc(bh + ob, 512, 128), idesc, acc0);
                            tc::mma_f16(d, tc::smem_desc(xh + oa, 512, 128), tc::smem_desc(bl + ob, 512, 128), idesc, 1u);
                            tc::mma_f16(d, tc::smem_desc(xlo + oa, 512, 128), tc::smem_desc(bh + ob, 512, 128), idesc, 1u);
                        }
                        tc::mma_commit(&tc_bar[sb]);
                    }
                    __syncwarp();
                    pend[sb] = true;
                }
                lap(6);
                for (int sb = 0; sb < 2; ++sb)
                    if (pend[sb]) {
                        tc::mbar_wait(&tc_bar[sb], tc_ph[sb]);
                        tc_ph[sb] ^= 1u;
                    }
                tc::tc_fence_after();
                lap(7);
                for (int z = 0; z < nt; ++z) {
                    float acc[32];
                    tc::tmem_ld32(tmem + tmem_lanes + 32u * z, acc);
                    const int j0 = 32 * (cr - z);
                    const float yv = z == 0 ? yv3[0] : (z == 1 ? yv3[1] : yv3[2]);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const float yj = __shfl_sync(kFull, yv, e);
                        const int j = j0 + e;
                        const bool ok = rok && j < a.M && in_band(i_, j + 1, a.bw);
                        const int kk = j + t;
                        ring[((kk >> 5) & 3) * 1024 + (kk & 31) * 32 + t] = (T)tc_cost(acc[e], xi, yj, tc_m2, ok);
                    }
                }
                tc::tc_fence_before();
                lap(6);
            }
        };
        // recompute tile cr and, speculatively, cr-1 and cr-2 (independent
        // tiles in one skewed loop: ILP 3); tile cr - z lands in slot z of
        // group grp (helper warp only)
        auto recompute = [&](int cr) {
            ev(1, cr);
            lap(5);
            const int wr = min(32, a.M - 32 * cr);
            const int nt = min(kWin, cr + 1);
            if constexpr (kTc) {
                tc_costs(cr, nt, x_loaded, b, s, i, row_ok, tc_xi);
            } else if (!kFused) {
                for (int g = cr - (kWin - 1); g <= cr + 1; ++g) {
                    if (g < 0 || g >= ngroups_row) continue;
                    // left of the band: only the window's speculative tiles
                    // need it (they are cut off, ctl[9 + g]) unless the
                    // requested tile cr itself lies there
                    if (banded && g < glo && cr >= glo) continue;
                    if (banded && (g < glo || g >= glo + A.band_ng)) {
                        // outside the cached band: this pass's results are
                        // void, the tensor-core backward reruns the call
                        if (t == 0) atomicOr(&A.stats[3], 1u);
#ifdef SDTW_B5_DEBUG
                        if (t == 0 && atomicAdd(&A.stats[4], 1u) < 40u)
                            printf("band miss b=%d s=%d cr=%d nt=%d g=%d glo=%d ng=%d S=%d C=%d\n", b, s, cr, nt, g, glo,
                                   A.band_ng, a.S, a.C);
#endif
                        continue;
                    }
                    load_group(ring + (g & 3) * 1024, dsrc + (size_t)(g - glo) * 1024, t);
                }
                cp_async_commit();
            }
            T lc[kWin], hp[kWin];
#pragma unroll
            for (int z = 0; z < kWin; ++z) {
                const int cz = cr - z;
                lc[z] = (z < nt && cz > 0 && row_ok) ? a.vc[((size_t)b * a.C + (cz - 1)) * a.N + (i - 1)] : T(0);
                hp[z] = T(0);
                const int wz = z == 0 ? wr : 32;
                halo_s[z * 32 + t] = (z < nt && s > 0 && t < wz)
                                         ? TG::value(A.hbt + ((size_t)b * a.S + (s - 1)) * a.M + 32 * cz + t)
                                         : T(0);
            }
            if (!kFused && !kTc) cp_async_wait<0>();
            __syncwarp();
            // tiles touching row 1, column 1 or a band edge take the general
            // cell; all others a branch-free one (warp-uniform choice)
            const bool fix = (s == 0) || (cr - nt + 1 <= 1) || (a.bw != 0);
            // 8-step sub-groups (64 steps; the last is a no-op): costs and top
            // halos of the sub-group loaded up front, branch-free steps
            for (int q8 = 0; q8 < 64; q8 += 8) {
                T d8[kWin][8], hs8[kWin][8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int q = q8 + kk;
#pragma unroll
                    for (int z = 0; z < kWin; ++z) {
                        hs8[z][kk] = halo_s[z * 32 + (q & 31)];
                        // skewed row 32 (cr - z) + q of the ring
                        // (fused: the SIMT cost up front, off the step chain)
                        if (kFused) {
                            const int jj = q - t, wz = z == 0 ? wr : 32;
                            const bool act = z < nt && row_ok && jj >= 0 && jj < wz;
                            d8[z][kk] = act ? bwd_cost<T, kFused>(a, ring, b, s, t, i, 32 * (cr - z) + 1 + jj) : T(0);
                        } else {
                            d8[z][kk] = ring[((cr - z + (q >> 5)) & 3) * 1024 + (q & 31) * 32 + t];
                        }
                    }
                }
                auto rsteps = [&](auto fix_tag) {
                    constexpr bool kFix = decltype(fix_tag)::value;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int q = q8 + kk;
                        T src[kWin], u[kWin];
#pragma unroll
                        for (int z = 0; z < kWin; ++z) src[z] = (t == 31) ? hs8[z][kk] : hp[z];
#pragma unroll
                        for (int z = 0; z < kWin; ++z) u[z] = __shfl_sync(kFull, src[z], (t + 31) & 31);
                        const int jj = q - t;
#pragma unroll
                        for (int z = 0; z < kWin; ++z) {
                            const int wz = z == 0 ? wr : 32;
                            const bool act = z < nt && row_ok && jj >= 0 && jj < wz;
                            const int j = 32 * (cr - z) + 1 + jj;
                            const T d = d8[z][kk];
                            T v, h, pd, pu, pl;
                            if constexpr (kFix) {
                                const Cell<T> cc = dp_cell<T, true>(i, j, a.bw, d, u[z], lc[z], a.k, a.gln2);
                                v = cc.v; h = cc.h; pd = cc.pd; pu = cc.pu; pl = cc.pl;
                            } else {
                                prob_cell<T>(d, u[z], lc[z], a.k, a.gln2, v, h, pd, pu, pl);
                            }
                            // inactive lanes write the dummy row: no divergent branch
                            T *Pz = base + kSlot * (kWin * grp + z) + (act ? jj : 32) * 32 + t;
                            Pz[0] = pd;
                            Pz[1056] = pu;
                            Pz[2112] = pl;
                            lc[z] = act ? v : lc[z];
                            hp[z] = act ? h : hp[z];
                        }
                    }
                };
                if (fix) rsteps(std::true_type{});
                else rsteps(std::false_type{});
            }
            __syncwarp();
            lap(0);
            ev(2, cr);
        };
        // ---- helper side: serve a window request / extend the cache leftwards
        auto pick_group = [&]() {
            const int e_pos = ctl[4];
            for (int g = 0; g < 2; ++g)
                if (ctl[7 + g] == 0 || ctl[5 + g] - (kWin - 1) > e_pos) return g;  // empty or passed by E
            return ctl[5] < ctl[6] ? 0 : 1;                                 // else the leftmost (speculative)
        };
        auto serve = [&](int cr) {
            int g = -1;
            if (t == 0) g = group_of(cr) >= 0 ? -1 : pick_group();
            g = __shfl_sync(kFull, g, 0);
            if (g < 0) return false;
            if (t == 0) {
                ctl[7 + g] = 0;
                __threadfence_block();
                ctl[5 + g] = cr;
                // lowest valid tile of the window: a band-cache window stops
                // at the band's left edge (its tiles further left are never
                // loaded; E requests them afresh, which then misses the band)
                ctl[9 + g] = (banded && cr >= glo) ? max(cr - (kWin - 1), glo) : cr - (kWin - 1);
                __threadfence_block();
                ctl[7 + g] = 1;
            }
            __syncwarp();
            grp = g;
            recompute(cr);
            __threadfence_block();
            __syncwarp();
            if (t == 0) ctl[7 + g] = 2;
            return true;
        };
        auto speculate = [&]() {
            int cn = -1;
            if (t == 0) {
                int w = 1 << 30;
                for (int g = 0; g < 2; ++g)
                    if (ctl[7 + g] != 0) w = min(w, ctl[5 + g]);
                const int e_pos = ctl[4];
                if (w != (1 << 30) && w - kWin >= 0 && w - kWin <= e_pos) {
                    // only into a group E no longer needs
                    bool free_g = false;
                    for (int g = 0; g < 2; ++g)
                        free_g |= ctl[7 + g] == 0 || ctl[5 + g] - (kWin - 1) > e_pos;
                    if (free_g) cn = w - kWin;
                }
            }
            cn = __shfl_sync(kFull, cn, 0);
            if (banded && cn < glo) return false;  // left of the cached band: not speculatively
            return cn >= 0 && serve(cn);
        };
        // ---- E side: ask for a window / wait for a tile's probabilities
        auto request = [&](int cr) {
            int have = 0;
            if (t == 0) have = group_of(cr) >= 0;
            if (__shfl_sync(kFull, have, 0)) return;
            if (t == 0) {
                ctl[1] = cr;
                __threadfence_block();
                ctl[2] = ctl[2] + 1;
            }
            __syncwarp();
        };
        auto tile_P = [&](int cf) -> T * {
            bool requested = false;
            unsigned polls = 0;
            for (;;) {
                int g = -1, st = 0, w0 = 0;
                if (t == 0) {
                    g = group_of(cf);
                    if (g >= 0) {
                        st = ctl[7 + g];
                        w0 = ctl[5 + g];
                    }
                }
                g = __shfl_sync(kFull, g, 0);
                st = __shfl_sync(kFull, st, 0);
                w0 = __shfl_sync(kFull, w0, 0);
                if (g >= 0 && st == 2) {
                    __threadfence_block();
                    return base + kSlot * (kWin * g + (w0 - cf));
                }
                // (re-)request while the tile is in no group: a window the
                // helper placed may be evicted before this warp saw it
                if (g < 0 && (!requested || (polls & 255u) == 255u)) {
                    request(cf);
                    requested = true;
                }
                __nanosleep(20);
                if (++polls > (1u << 26)) {
                    if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                    return base;
                }
            }
        };
        auto advance = [&](int) {};
        auto dead_chunk = [&](int cd) {
            const int w = min(32, a.M - 32 * cd);
            if (t < w) TG::store(sb_me + 32 * cd + t, T(0), epoch);
            if (t == 0) put_status(stat_me + cd, kTileDead, epoch);
        };
        if (warp == 0) {
            // ---- recompute helper: serve requests, speculate one window ahead
            int my_seq = 0;
            unsigned idle = 0;
            for (;;) {
                int seq = 0, done = 0, req = -1;
                if (t == 0) {
                    seq = ctl[2];
                    done = ctl[3];
                    req = ctl[1];
                }
                seq = __shfl_sync(kFull, seq, 0);
                done = __shfl_sync(kFull, done, 0);
                req = __shfl_sync(kFull, req, 0);
                if (seq != my_seq) {
                    my_seq = seq;
                    serve(req);
                    idle = 0;
                    continue;
                }
                if (done) break;
                if (speculate()) {
                    idle = 0;
                    continue;
                }
                __nanosleep(64);
                if (++idle > (1u << 26)) {
                    if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                    break;
                }
            }
        }
        int c = warp == 1 ? a.C - 1 : -1;
        while (c >= 0) {
            if (t == 0) ctl[4] = c;
            const bool has_end = bottom && c == a.C - 1;
            const bool live_right = has_end || __any_sync(kFull, e_right != T(0));
            if (!live_right) {
                if (bottom) {
                    dead_chunk(c);
                    pl_right = T(0);
                    pd_right = T(0);
                    advance(c);
                    --c;
                    continue;
                }
                // statuses of chunks c, c-1, ..., c-31 of the strip below
                const int cc = c - t;
                unsigned st = kTileHint;  // lanes past chunk 0 never stop a dead run
                if (cc >= 0) st = get_status(stat_below + cc, epoch);
                unsigned polls = 0;
                lap(5);
                while (!__shfl_sync(kFull, st, 0)) {  // chunk c's status must be known
                    if (BWD_STATUS_SLEEP_NS > 0) __nanosleep(BWD_STATUS_SLEEP_NS);
                    if (cc >= 0 && st == 0) st = get_status(stat_below + cc, epoch);
                    if (++polls > (1u << 26)) {
                        if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                        break;
                    }
                }
                lap(3);
                const unsigned stop = __ballot_sync(kFull, st != kTileDead);
                const int run = stop ? __ffs(stop) - 1 : 32;  // leading dead chunks
                if (run > 0) {
                    for (int q = 0; q < run; ++q) dead_chunk(c - q);
                    pl_right = T(0);
                    pd_right = T(0);
                    advance(c);
                    c -= run;
                    continue;
                }
                unsigned st0 = __shfl_sync(kFull, st, 0);
                if (st0 >= kTileCommit && c <= diag_chunk(s, a.N, a.M) + A.spec_right) {
                    // near the diagonal (where the alignment band lies): sweep
                    // right behind the strip below, whose S arrives per 8
                    // columns (zeros if the tile turns out dead), instead of
                    // waiting for its verdict; the diagonal bound keeps these
                    // sweeps from cascading over dead tiles
                    request(c);
                } else if (st0 >= kTileCommit) {
                    // the strip below has no evidence yet: recompute early (and
                    // say so one level up), then wait for its verdict
                    request(c);
                    if (st0 + 1 < kTileCommit + kSpecDepth && t == 0) put_status(stat_me + c, st0 + 1, epoch);
                    polls = 0;
                    lap(5);
                    while (st0 >= kTileCommit) {
                        if (BWD_STATUS_SLEEP_NS > 0) __nanosleep(2 * BWD_STATUS_SLEEP_NS);
                        st0 = __shfl_sync(kFull, get_status(stat_below + c, epoch), 0);
                        if (++polls > (1u << 26)) {
                            if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                            break;
                        }
                    }
                    lap(3);
                    if (st0 == kTileDead) {
                        dead_chunk(c);
                        pl_right = T(0);
                        pd_right = T(0);
                        --c;
                        continue;
                    }
                }
                // chunk c below is HINT or LIVE: commit to this tile; its S
                // arrives per 8 columns during phase E
            }
            // ---- candidate tile c.  HINT is published only with evidence that
            // E enters it (E from the right now, or a non-zero S from below
            // during phase E), so hints cannot cascade over zero tiles.
            bool hinted = live_right;
            if (t == 0) put_status(stat_me + c, hinted ? kTileHint : kTileCommit, epoch);
            const int j0 = 32 * c + 1;
            const int width = min(32, a.M - 32 * c);
            // the whole tile's S from below in one load per lane, issued before
            // the probability wait: when the strip below has already finished
            // this tile, the sweep then polls L2 once per tile, not once per
            // 8 columns (fp32; otherwise per 8 columns as below)
            unsigned long long s_all = 0;
            if constexpr (sizeof(T) == 4)
                if (!bottom && t < width) s_all = TG::load_raw(sb_below + (j0 - 1) + t);
            T *Pc = tile_P(c);
            bool s_all_ok = false;
            if constexpr (sizeof(T) == 4)
                s_all_ok = !bottom && __all_sync(kFull, t >= width || (unsigned)(s_all >> 32) == epoch);
            // ---- phase E with 8-column hand-offs --------------------------
            const bool has_end_tile = bottom && c == a.C - 1;
            T s_prev = T(0);
            unsigned long long pf_w = 0;
            int pf_q = -1;
            lap(5);
            // 8-step sub-groups: S from below polled once per sub-group, the
            // sub-group's probabilities loaded up front (no shared load on the
            // step chain), branch-free steps; S published as soon as lane 0
            // completes a group of 8 columns (after step 6 of a sub-group).
            ev(3, c);
            int pub_next = 0;  // next 8-column group (from the right) to publish
            auto publish = [&](int done) {
                // groups k with all columns done (or the tile's last partial group)
                while (8 * pub_next <= done && (8 * pub_next + 7 <= done || done >= width - 1)) {
                    __syncwarp();
                    const int hi = width - 1 - 8 * pub_next;
                    const int lo = max(0, hi - 7);
                    if (t <= hi - lo) TG::store(sb_me + (j0 - 1) + lo + t, sout_s[lo + t], epoch);
                    ++pub_next;
                }
            };
            for (int q8 = 0; q8 < width + 31; q8 += 8) {
                const int jj31 = width - 1 - q8;
                if (jj31 >= 0) {
                    lap(2);
                    // S from below for columns [jj31 - 7, jj31] of this chunk
                    const int lo = max(0, jj31 - 7);
                    const int n = jj31 - lo + 1;
                    T v = T(0);
                    if (!bottom) {
                        if constexpr (sizeof(T) == 4) {
                          if (s_all_ok) {
                            v = __uint_as_float((unsigned)(__shfl_sync(kFull, s_all, (lo + t) & 31) & 0xffffffffull));
                          } else {
                            bool ok = t >= n;
                            if (!ok) {
                                const unsigned long long w8 = (pf_q == q8) ? pf_w : TG::load_raw(sb_below + (j0 - 1) + lo + t);
                                ok = (unsigned)(w8 >> 32) == epoch;
                                v = __uint_as_float((unsigned)(w8 & 0xffffffffull));
                            }
                            if (!__all_sync(kFull, ok)) v = poll_entries<T>(sb_below + (j0 - 1) + lo, n, epoch, t);
                            // prefetch the next 8 columns
                            const int jn = jj31 - 8;
                            if (jn >= 0) {
                                const int lo2 = max(0, jn - 7);
                                if (t <= jn - lo2) pf_w = TG::load_raw(sb_below + (j0 - 1) + lo2 + t);
                                pf_q = q8 + 8;
                            }
                          }
                        } else {
                            v = poll_entries<T>(sb_below + (j0 - 1) + lo, n, epoch, t);
                        }
                    }
                    lap(1);
                    if (t < n) sin_s[lo + t] = v;
                    if (!hinted && __any_sync(kFull, v != T(0))) {
                        hinted = true;
                        if (t == 0) put_status(stat_me + c, kTileHint, epoch);
                    }
                    __syncwarp();
                }
                T pd8[8], pu8[8], pl8[8], si8[8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int q = q8 + kk;
                    const int jj = width - 1 - q + (31 - t);
                    const int jc = (jj >= 0 && jj < width) ? jj : 32;
                    pd8[kk] = Pc[jc * 32 + t];
                    pu8[kk] = Pc[1056 + jc * 32 + t];
                    pl8[kk] = Pc[2112 + jc * 32 + t];
                    const int j31 = width - 1 - q;
                    si8[kk] = sin_s[j31 >= 0 ? j31 : 0];
                }
                auto esteps = [&](auto fix_tag) {
                    constexpr bool kFix = decltype(fix_tag)::value;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int q = q8 + kk;
                        const int jj = width - 1 - q + (31 - t);
                        const T src = (t == 0) ? si8[kk] : s_prev;
                        const T s_in = __shfl_sync(kFull, src, (t + 1) & 31);
                        // branch-free step: inactive lanes write the dummy row
                        const bool act = jj >= 0 && jj < width;
                        const bool cell = act && row_ok;
                        const int jc = act ? jj : 32;
                        T e = fma(e_right, pl_right, s_in);
                        e = e < T(1) ? e : T(1);
                        if constexpr (kFix) {
                            const int j = j0 + jj;
                            e = (i == a.N && j == a.M) ? T(1) : e;
                            e = in_band(i, j, a.bw) ? e : T(0);
                        }
                        e = cell ? e : T(0);
                        const T s_out = cell ? fma(e, pu8[kk], e_right * pd_right) : s_prev;
                        e_right = cell ? e : e_right;
                        pl_right = cell ? pl8[kk] : pl_right;
                        pd_right = cell ? pd8[kk] : pd_right;
                        et_s[t * 34 + jc] = e;
                        if (t == 0) sout_s[jc] = s_out;
                        s_prev = s_out;
                        // lane 0 has now completed done + 1 columns: a full group
                        // of 8 ends at kk = 6 (q = 31 + 8 g + 7)
                        if (kk == 6) publish(q - 31);
                    }
                };
                if (has_end_tile || a.bw != 0) esteps(std::true_type{});
                else esteps(std::false_type{});
                publish(min(q8 + 7 - 31, width - 1));
            }
            __syncwarp();
            lap(2);
            ev(4, c);
            // final status: does any S go up?  (stops the spread of hints over
            // tiles whose inputs turned out to be exactly zero)
            const bool s_nz = __any_sync(kFull, t < width && sout_s[t] != T(0));
            if (t == 0) put_status(stat_me + c, s_nz ? kTileLive : kTileDead, epoch);
            bool e_nz = false;
            for (int r = 0; r < 32; ++r) e_nz |= (t < width && et_s[r * 34 + t] != T(0));
            if (!__any_sync(kFull, e_nz)) {
                // exactly-zero tile after all: nothing to contract or store
            } else {
            if (t == 0) atomicAdd(&A.stats[0], 1u);
            if (a.E) {
                for (int r = 0; r < 32; ++r) {
                    const int ir = 32 * s + r + 1;
                    if (ir <= a.N && t < width)
                        a.E[((size_t)b * a.N + (ir - 1)) * a.M + (j0 - 1) + t] = et_s[r * 34 + t];
                }
            }
            // queue the tile for the contraction (or contract here): the
            // k-th stored tile of a strip is fixed by the strip's own order,
            // so the split between the two paths is deterministic
            if (nstored < A.tile_quota) {
                const size_t slot = ((size_t)b * a.S + s) * A.tile_quota + nstored;
                T *dst = A.tiles + slot * 1024;
                for (int r = 0; r < 32; ++r) dst[r * 32 + t] = (t < width) ? et_s[r * 34 + t] : T(0);
                if (t == 0) A.tile_meta[slot] = make_int4(b, s, c, width);
                ++nstored;
            } else {
                if (t == 0) atomicAdd(&A.stats[2], 1u);
                // the speculative tile's probabilities live in the other slot;
                // use the E tile's storage neighbour as scratch (ring slot 3,
                // or P of tile c which is consumed)
                tile_contract_fx<T>(A, fx, b, s, c, width, et_s, Pc, t, 34);
            }
            }
            __syncwarp();
            lap(4);
            advance(c);
            ++ntiles;
            --c;
        }
        lap(5);
        if (warp == 1 && t == 0) ctl[3] = 1;  // strip done: release the helper
        named_bar(1 + wk, 64);
        if (warp == 0) continue;
        if (t == 0) A.strip_tiles[(size_t)b * a.S + s] = nstored;
        if (A.trace && t == 0)
            for (int e = 0; e < 8; ++e)
                A.trace[32 * (size_t)a.B * a.S + 8 * ((size_t)b * a.S + s) + e] = (unsigned long long)cyc[e];
        if (A.trace && t == 0) {
            A.trace[2 * ((size_t)a.B * a.S + (size_t)b * a.S + s) + 1] = global_ns();
            A.trace[4 * (size_t)a.B * a.S + (size_t)b * a.S + s] = (unsigned long long)ntiles;
        }
    }
    if constexpr (kTc) {
        tc::tc_fence_before();
        __syncthreads();
        if (threadIdx.x < 32) tc::tmem_dealloc<128 * kW>(tmem_slot);
    }
}

}  // namespace sdtw
