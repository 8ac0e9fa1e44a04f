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
#include "sdtw_common.cuh"
#include "sdtw_dp2.cuh"
#include "sdtw_dp3.cuh"

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
constexpr unsigned kSpecDepth = 2;

template <class T, bool kFused>
struct Bwd4Smem {
    static constexpr int kSlot = 3 * 33 * 32;            // pd, pu, pl [jj][t], row 32 = dummy
    static constexpr int kP = 3 * kSlot;                 // three probability tiles
    static constexpr int kE = 32 * 34;                   // E tile [t][jj] (even stride: conflict-free), column 32 = dummy
    static constexpr int kRing = kFused ? 0 : 4 * 1024;  // skewed cost row groups (slot g & 3)
    static constexpr int kHalo = 6 * 32;                 // 3 top halos (h), S in, S out (+dummy)
    static constexpr int kPerWarp = kP + kE + kRing + kHalo;
};

// Status words: (epoch << 32) | status.
__device__ __forceinline__ void put_status(unsigned long long *p, unsigned v, unsigned tag)
{
    const unsigned long long w = ((unsigned long long)tag << 32) | v;
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned get_status(const unsigned long long *p, unsigned tag)
{
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
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

template <class T, bool kFused>
__global__ void __launch_bounds__(32) sdtw_backward4_kernel(Dp3Args<T> A, unsigned long long *stat)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    const DpArgs<T> &a = A.a;
    using SM = Bwd4Smem<T, kFused>;
    using TG = Tagged<T>;
    const int t = threadIdx.x & 31;
    T *base = reinterpret_cast<T *>(smem_raw);
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
    const FxScales fx = fx_scales(A.absmax, a.N, a.M);
    for (;;) {
        const unsigned tk = warp_ticket(&a.tickets[1]);
        if ((int)tk >= total) return;
        const int s = a.S - 1 - (int)tk / a.B, b = (int)tk % a.B;
        const int i = 32 * s + t + 1;
        const bool row_ok = i <= a.N;
        const bool bottom = s == a.S - 1;
        const T *dsrc = kFused ? nullptr : a.dsk + ((size_t)b * a.S + s) * (size_t)a.KK * 32;
        unsigned long long *stat_me = stat + ((size_t)b * a.S + s) * a.C;
        const unsigned long long *stat_below = stat + ((size_t)b * a.S + s + 1) * a.C;
        typename TG::Ent *sb_me = A.sbt + ((size_t)b * a.S + s) * a.M;
        const typename TG::Ent *sb_below = A.sbt + ((size_t)b * a.S + s + 1) * a.M;
        if (A.trace && t == 0) A.trace[2 * ((size_t)a.B * a.S + (size_t)b * a.S + s)] = global_ns();
        int ntiles = 0;
        auto ev = [&](int e) {
            if (A.trace && t == 0 && e < 8)
                A.trace[5 * (size_t)a.B * a.S + 8 * ((size_t)b * a.S + s) + e] = global_ns();
        };
        T e_right = T(0), pl_right = T(0), pd_right = T(0);
        // P-tile cache: slot k holds chunk slot_c[k] (-1: none)
        int slot_c0 = -1, slot_c1 = -1, slot_c2 = -1;
        auto find_slot = [&](int cf) { return slot_c0 == cf ? 0 : slot_c1 == cf ? 1 : slot_c2 == cf ? 2 : -1; };
        // recompute tile cr and, speculatively, cr-1 and cr-2 (independent
        // tiles in one skewed loop: ILP 3); tile cr - z lands in slot z
        auto recompute = [&](int cr) {
            const int wr = min(32, a.M - 32 * cr);
            const int nt = min(3, cr + 1);
            if (!kFused) {
                for (int g = cr - 2; g <= cr + 1; ++g)
                    if (g >= 0 && g < ngroups_row) load_group(ring + (g & 3) * 1024, dsrc + (size_t)g * 1024, t);
                cp_async_commit();
            }
            T lc[3], hp[3];
#pragma unroll
            for (int z = 0; z < 3; ++z) {
                const int cz = cr - z;
                lc[z] = (z < nt && cz > 0 && row_ok) ? a.vc[((size_t)b * a.C + (cz - 1)) * a.N + (i - 1)] : T(0);
                hp[z] = T(0);
                const int wz = z == 0 ? wr : 32;
                halo_s[z * 32 + t] = (z < nt && s > 0 && t < wz)
                                         ? TG::value(A.hbt + ((size_t)b * a.S + (s - 1)) * a.M + 32 * cz + t)
                                         : T(0);
            }
            if (!kFused) cp_async_wait<0>();
            __syncwarp();
            // tiles touching row 1, column 1 or a band edge take the general
            // cell; all others a branch-free one (warp-uniform choice)
            const bool fix = (s == 0) || (cr - nt + 1 <= 1) || (a.bw != 0);
            for (int q = 0; q < 32 + 31; ++q) {
                T src[3], u[3];
#pragma unroll
                for (int z = 0; z < 3; ++z) src[z] = (t == 31) ? halo_s[z * 32 + (q & 31)] : hp[z];
#pragma unroll
                for (int z = 0; z < 3; ++z) u[z] = __shfl_sync(kFull, src[z], (t + 31) & 31);
                const int jj = q - t;
#pragma unroll
                for (int z = 0; z < 3; ++z) {
                    const int wz = z == 0 ? wr : 32;
                    const bool act = z < nt && row_ok && jj >= 0 && jj < wz;
                    const int j = 32 * (cr - z) + 1 + jj;
                    const T d = kFused ? (act ? bwd_cost<T, kFused>(a, ring, b, s, t, i, j) : T(0))
                                       : bwd_cost<T, kFused>(a, ring, b, s, t, i, j);
                    T v, h, pd, pu, pl;
                    if (fix) {
                        const Cell<T> cc = dp_cell<T, true>(i, j, a.bw, d, u[z], lc[z], a.k, a.gln2);
                        v = cc.v; h = cc.h; pd = cc.pd; pu = cc.pu; pl = cc.pl;
                    } else {
                        prob_cell<T>(d, u[z], lc[z], a.k, a.gln2, v, h, pd, pu, pl);
                    }
                    // inactive lanes write the dummy row: no divergent branch
                    T *Pz = base + kSlot * z + (act ? jj : 32) * 32 + t;
                    Pz[0] = pd;
                    Pz[1056] = pu;
                    Pz[2112] = pl;
                    lc[z] = act ? v : lc[z];
                    hp[z] = act ? h : hp[z];
                }
            }
            __syncwarp();
            slot_c0 = cr;
            slot_c1 = nt > 1 ? cr - 1 : -1;
            slot_c2 = nt > 2 ? cr - 2 : -1;
        };
        auto advance = [&](int) {};
        auto dead_chunk = [&](int cd) {
            const int w = min(32, a.M - 32 * cd);
            if (t < w) TG::store(sb_me + 32 * cd + t, T(0), epoch);
            if (t == 0) put_status(stat_me + cd, kTileDead, epoch);
        };
        int c = a.C - 1;
        while (c >= 0) {
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
                while (!__shfl_sync(kFull, st, 0)) {  // chunk c's status must be known
                    __nanosleep(32);
                    if (cc >= 0 && st == 0) st = get_status(stat_below + cc, epoch);
                    if (++polls > (1u << 26)) {
                        if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                        break;
                    }
                }
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
                if (st0 >= kTileCommit) {
                    // the strip below has no evidence yet: recompute early (and
                    // say so one level up), then wait for its verdict
                    if (find_slot(c) < 0) recompute(c);
                    if (st0 + 1 < kTileCommit + kSpecDepth && t == 0) put_status(stat_me + c, st0 + 1, epoch);
                    polls = 0;
                    while (st0 >= kTileCommit) {
                        __nanosleep(64);
                        st0 = __shfl_sync(kFull, get_status(stat_below + c, epoch), 0);
                        if (++polls > (1u << 26)) {
                            if (t == 0) atomicAdd(&g_sdtw_wait_timeouts, 1);
                            break;
                        }
                    }
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
            ev(3 + 2 * min(ntiles, 1));
            if (find_slot(c) < 0) recompute(c);
            ev(4 + 2 * min(ntiles, 1));
            T *Pc = base + kSlot * find_slot(c);
            // ---- phase E with 8-column hand-offs --------------------------
            const bool has_end_tile = bottom && c == a.C - 1;
            T s_prev = T(0);
            unsigned long long pf_w = 0;
            int pf_q = -1;
            for (int q = 0; q < width + 31; ++q) {
                const int jj31 = width - 1 - q;
                if (((q & 7) == 0) && jj31 >= 0) {
                    // S from below for columns [jj31 - 7, jj31] of this chunk
                    const int lo = max(0, jj31 - 7);
                    const int n = jj31 - lo + 1;
                    T v = T(0);
                    if (!bottom) {
                        if constexpr (sizeof(T) == 4) {
                            bool ok = t >= n;
                            if (!ok) {
                                const unsigned long long w8 = (pf_q == q) ? pf_w : TG::load_raw(sb_below + (j0 - 1) + lo + t);
                                ok = (unsigned)(w8 >> 32) == epoch;
                                v = __uint_as_float((unsigned)(w8 & 0xffffffffull));
                            }
                            if (!__all_sync(kFull, ok)) v = poll_entries<T>(sb_below + (j0 - 1) + lo, n, epoch, t);
                            // prefetch the next 8 columns
                            const int jn = jj31 - 8;
                            if (jn >= 0) {
                                const int lo2 = max(0, jn - 7);
                                if (t <= jn - lo2) pf_w = TG::load_raw(sb_below + (j0 - 1) + lo2 + t);
                                pf_q = q + 8;
                            }
                        } else {
                            v = poll_entries<T>(sb_below + (j0 - 1) + lo, n, epoch, t);
                        }
                    }
                    if (t < n) sin_s[lo + t] = v;
                    if (!hinted && __any_sync(kFull, v != T(0))) {
                        hinted = true;
                        if (t == 0) put_status(stat_me + c, kTileHint, epoch);
                    }
                    __syncwarp();
                }
                const int jj = width - 1 - q + (31 - t);
                const T src = (t == 0) ? sin_s[jj31 >= 0 ? jj31 : 0] : s_prev;
                const T s_in = __shfl_sync(kFull, src, (t + 1) & 31);
                // branch-free step: inactive lanes read / write the dummy row
                const bool act = jj >= 0 && jj < width;
                const bool cell = act && row_ok;
                const int jc = act ? jj : 32;
                const T pd = Pc[jc * 32 + t], pu = Pc[1056 + jc * 32 + t], pl = Pc[2112 + jc * 32 + t];
                const int j = j0 + jj;
                T e = fma(e_right, pl_right, s_in);
                e = e < T(1) ? e : T(1);
                if (has_end_tile || a.bw != 0) {  // warp-uniform
                    e = (i == a.N && j == a.M) ? T(1) : e;
                    e = in_band(i, j, a.bw) ? e : T(0);
                }
                e = cell ? e : T(0);
                const T s_out = cell ? fma(e, pu, e_right * pd_right) : s_prev;
                e_right = cell ? e : e_right;
                pl_right = cell ? pl : pl_right;
                pd_right = cell ? pd : pd_right;
                et_s[t * 34 + jc] = e;
                if (t == 0) sout_s[jc] = s_out;
                s_prev = s_out;
                // lane 0 finished column jj0 = width-1-(q-31): publish each
                // completed group of 8 columns
                const int done = q - 31;  // columns completed by lane 0 minus 1
                if (done >= 0 && (((done & 7) == 7) || done == width - 1)) {
                    __syncwarp();
                    const int hi = width - 1 - (done & ~7);
                    const int lo = width - 1 - done;
                    if (t <= hi - lo) TG::store(sb_me + (j0 - 1) + lo + t, sout_s[lo + t], epoch);
                }
            }
            __syncwarp();
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
            // queue the tile for the contraction kernel (or contract here)
            unsigned slot = 0;
            if (t == 0) slot = atomicAdd(&A.stats[1], 1u);
            slot = __shfl_sync(kFull, slot, 0);
            if (slot < A.tile_cap) {
                T *dst = A.tiles + (size_t)slot * 1024;
                for (int r = 0; r < 32; ++r) dst[r * 32 + t] = (t < width) ? et_s[r * 34 + t] : T(0);
                if (t == 0) A.tile_meta[slot] = make_int4(b, s, c, width);
            } else {
                if (t == 0) atomicAdd(&A.stats[2], 1u);
                // the speculative tile's probabilities live in the other slot;
                // use the E tile's storage neighbour as scratch (ring slot 3,
                // or P of tile c which is consumed)
                tile_contract_fx<T>(A, fx, b, s, c, width, et_s, Pc, t, 34);
            }
            }
            __syncwarp();
            advance(c);
            ++ntiles;
            --c;
        }
        if (A.trace && t == 0) {
            A.trace[2 * ((size_t)a.B * a.S + (size_t)b * a.S + s) + 1] = global_ns();
            A.trace[4 * (size_t)a.B * a.S + (size_t)b * a.S + s] = (unsigned long long)ntiles;
        }
    }
}

}  // namespace sdtw
