// sdtw_bwd5.cuh — backward DP as a per-pair pipeline inside one CTA.
//
// Reference: backward_sweep<T, Cost, kLog> (backward.hpp:29-177) and its
// callers backward_log / sdtw_with_gradients (backward.hpp:183-190, 276-304).
// The E recurrence is the engine's probability form (sdtw_common.cuh):
//     E(i,j) = E(i,j+1) P_l(i,j+1) + E(i+1,j) P_u(i+1,j) + E(i+1,j+1) P_d(i+1,j+1),
// E(N,M) = 1, out-of-band / outside cells 0, E <= 1 (the reference's Ebar <= 0
// clamp).  In fp32, E is exactly 0 outside a narrow band around the soft
// alignment path, so the backward's work is the band, and its
// time is the dependency chain along it: ~N + M anti-diagonal steps.
//
// Why one CTA per pair.  The v4 backward (sdtw_dp4.cuh) ran strips on
// persistent workers anywhere on the GPU and handed S (the E mass entering a
// strip from below) and tile statuses through L2: every strip hop paid L2
// round trips, and every live tile paid a 31-step skew fill/drain of its
// own.  Here the strips of a pair are processed bottom-up by NE "E warps" of
// one CTA in a pipeline, and everything on the chain stays in shared memory:
//   * S hand-off: strip s's lane 0 writes S(j) of its top row into a ring in
//     shared memory; strip s-1's lane 31 reads it (8 columns per sub-group).
//   * Continuous sweeps: an E warp sweeps consecutive live tiles without
//     draining between them (lane 31 enters tile c-1 while lanes 0..30
//     finish tile c); it only drains where the band ends, and restarts if
//     E still leaves the drained tile on some row.
//   * Recompute off the chain: NH helper warps recompute tiles' softmin
//     probabilities P from the forward's checkpoints (hbt: h of every
//     strip's bottom row; vc: v at every 32nd column) into a per-CTA pool in
//     global memory (L2-resident), requested kB5Ahead strips ahead of the
//     strip that will need them, in windows of kB5Win tiles (ILP).
// Tiles: strip s = rows [32 s, 32 s + 32), chunk c = columns [32 c, 32 c + 32)
// (0-based).  A lane t of strip s owns row 32 s + t; an E sweep starting at
// column J gives lane t column J - k + 31 - t at step k (lane 31 first), so at
// every step all lanes read the same rotated row r = (j + t) & 31 of their
// tiles' P, stored as Pt[r][t] = P(t, (r - t) & 31) (coalesced, and written
// by the recompute one row per step as well).
#pragma once
#include <climits>
#include <cstdio>
#include <type_traits>
#include "sdtw_common.cuh"
#include "sdtw_dp.cuh"
#include "sdtw_dp2.cuh"
#include "sdtw_dp3.cuh"
#include "sdtw_dp4.cuh"

namespace sdtw {

constexpr int kB5Ring = 256;   // S ring per producer slot (columns)
constexpr int kB5NQ = 8;       // strip slots (P-tile coverage), >= 2 NE
constexpr int kB5JQ = 64;      // recompute job queue (speculative requests)
constexpr int kB5UQ = 16;      // urgent job queue (a strip waiting for its own tile)
constexpr int kB5Win = 3;      // tiles per recompute job (independent tiles: ILP)
constexpr int kB5Ahead = 3;    // a strip entering chunk c requests strips s-1 .. s-kB5Ahead
constexpr int kB5MaxC = 4096;  // chunks per pair the coverage bitmaps hold (M <= 131072)

template <class T, int NE, int NH>
struct Bwd5Shared {
    T sring[NE][2][kB5Ring];   // S of the top row of the strip in (warp, slot)
    T et[NE][3][32][33];       // E tile staging, rotated rows (three tiles in flight)
    T hhalo[NH][kB5Win][32];   // helper: top halos of the window's tiles
    int ring_strip[NE][2];     // strip the ring serves
    int zero_above[NE][2];     // columns >= zero_above: S = 0 (-1 until the producer knows: its
                               // first sweep starts there, or it is dead: 0)
    int prod_pos[NE][2];       // columns >= prod_pos: decided (ring or zero)
    int intent_pos[NE][2];     // lowest column the producer is writing or has written
    int zero_below[NE][2];     // columns < zero_below: S = 0 (decided)
    int cons_pos[NE][2];       // INT_MIN: ring free (its consumer finished)
    int slot_strip[kB5NQ];
    unsigned cov[kB5NQ][kB5MaxC / 32];  // requested P tiles of the slot's strip (bitmap over chunks)
    unsigned rdy[kB5NQ][kB5MaxC / 32];  // P tiles in the pool
    int e_pos[kB5NQ];                   // tiles > e_pos no longer read by the strip's E warp
    int lock[kB5NQ];
    int outstanding[kB5NQ];             // queued or running recompute jobs of the slot's strip
    int4 jobs[2][kB5JQ];                // [0] speculative, [1] urgent (kB5UQ used)
    int job_seq[2][kB5JQ], job_rd[2][kB5JQ];
    int job_tail[2], job_head[2];
    int done;                           // the pair's strips are finished: helpers leave
    int4 hjob[NH];                      // a helper's current job (lane 0 -> warp)
    int pair;
};

#ifdef SDTW_B5_DEBUG
#define B5_CHECK(cond, tag, a, b)                                                                     \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("B5_CHECK %s failed: blk %d warp %d lane %d a=%lld b=%lld\n", tag, blockIdx.x,      \
                   threadIdx.x >> 5, threadIdx.x & 31, (long long)(a), (long long)(b));               \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define B5_CHECK(cond, tag, a, b) \
    do {                          \
    } while (0)
#endif

__device__ __forceinline__ int vld(const int &p) { return *(const volatile int *)&p; }
__device__ __forceinline__ unsigned vldu(const unsigned &p) { return *(const volatile unsigned *)&p; }
__device__ __forceinline__ void vst(int &p, int v) { *(volatile int *)&p = v; }
__device__ __forceinline__ void vstu(unsigned &p, unsigned v) { *(volatile unsigned *)&p = v; }
__device__ __forceinline__ unsigned b5_tag(int s, int c) { return ((unsigned)s << 16 | (unsigned)c) + 1u; }

// Bounded spin (a scheduling bug must surface as an error, not a hang).
// (trace mode: a timed-out wait also records (site, CTA, a, b) in g_b5_dbg)
static __device__ int g_b5_dbg[4 + 4 * 64];
static __device__ unsigned g_b5_spin_limit = 1u << 24;  // experiments: set through knob[2]
struct B5Spin {
    unsigned n = 0;
    int *timeouts;
    int site, a, b;
    __device__ explicit B5Spin(int *to, int site_ = 0, int a_ = 0, int b_ = 0) : timeouts(to), site(site_), a(a_), b(b_)
    {
    }
    __device__ __forceinline__ bool go(int lane)
    {
        if (++n > g_b5_spin_limit) {
            if (lane == 0) {
                atomicAdd(timeouts, 1);
                const int k = atomicAdd(&g_b5_dbg[0], 1);
                if (k < 64) {
                    g_b5_dbg[4 + 4 * k] = site;
                    g_b5_dbg[5 + 4 * k] = blockIdx.x;
                    g_b5_dbg[6 + 4 * k] = a;
                    g_b5_dbg[7 + 4 * k] = b;
                }
            }
            return false;
        }
        return true;
    }
};

// Diagnostics (trace mode only, A.trace != nullptr): A.stats[4..15]
//   4 jobs enqueued, 5 jobs skipped, 6 tiles recomputed, 7 E tile-wait
//   kcycles, 8 E below-wait kcycles, 9 E request kcycles, 10 E strip
//   kcycles, 11 runs, 12 tiles entered, 13 helper busy kcycles, 14 helper
//   queue-wait kcycles, 15 E start-wait kcycles
__device__ __forceinline__ void b5_count(const unsigned long long *trace, unsigned *stats, int i, long long v)
{
    if (trace && v) atomicAdd(&stats[i], (unsigned)v);
}

template <class T>
__device__ __forceinline__ T ldcg(const T *p)
{
    if constexpr (sizeof(T) == 4) {
        float v;
        asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
        return v;
    } else {
        double v;
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
        return v;
    }
}

// ----------------------------------------------------------------------------
// Recompute requests (lane 0 of an E warp): chunks [lo, hi] of strip s.  The
// pool holds a P tile per (strip slot, chunk), so requests in any order
// never collide; a bitmap marks what was requested, and unmarked runs are
// queued as jobs of <= kB5Win tiles (urgent: the strip's own E warp waits).
// ----------------------------------------------------------------------------
__device__ __forceinline__ bool b5_bit(const unsigned *bm, int c)
{
    return (*(const volatile unsigned *)&bm[c >> 5] >> (c & 31)) & 1u;
}

template <class T, int NE, int NH>
__device__ void b5_enqueue(Bwd5Shared<T, NE, NH> &sh, int qu, int4 job, int *timeouts)
{
    const int cap = qu ? kB5UQ : kB5JQ;
    const int slot = atomicAdd(&sh.job_tail[qu], 1);
    const int p = slot % cap;
    B5Spin sq(timeouts, 3, job.x, slot);
    while (vld(sh.job_rd[qu][p]) != slot - cap)  // previous occupant taken by a helper
        if (!sq.go(0)) break;
    B5_CHECK(job.z >= 1 && job.z <= kB5Win, "enqueue", (long long)slot * 1000 + qu * 100 + p,
             (long long)job.x * 1000000 + job.y * 1000 + job.z);
    sh.jobs[qu][p] = job;
    __threadfence_block();
    vst(sh.job_seq[qu][p], slot + 1);
}

template <class T, int NE, int NH>
__device__ void b5_request(Bwd5Shared<T, NE, NH> &sh, int s, int lo, int hi, int C, bool urgent, int *timeouts,
                           const unsigned long long *trace = nullptr, unsigned *stats = nullptr)
{
    lo = max(lo, 0);
    hi = min(hi, C - 1);
    if (s < 0 || lo > hi) return;
    const int q = s % kB5NQ;
    // lock-free fast path: every chunk already requested
    if (vld(sh.slot_strip[q]) == s) {
        bool all = true;
        for (int c = lo; c <= hi && all; ++c) all = b5_bit(sh.cov[q], c);
        if (all) return;
    }
    B5Spin sp(timeouts, 1, s, lo);
    while (atomicCAS(&sh.lock[q], 0, 1) != 0)
        if (!sp.go(0)) return;
    __threadfence_block();
    if (vld(sh.slot_strip[q]) != s) {
        // first request for strip s: the slot's previous strip (s + kB5NQ)
        // finished long ago (the pipeline holds at most 2 NE strips), but
        // speculative jobs of it may still be queued or running: they skip
        // themselves or finish into the pool before the slot is reused
        {
            B5Spin so(timeouts, 2, s, vld(sh.slot_strip[q]));
            while (vld(sh.outstanding[q]) != 0)
                if (!so.go(0)) break;
        }
        for (int w = 0; w < (C + 31) / 32; ++w) {
            sh.cov[q][w] = 0u;
            sh.rdy[q][w] = 0u;
        }
        vst(sh.e_pos[q], INT_MAX);
        __threadfence_block();
        vst(sh.slot_strip[q], s);
    }
    // unmarked runs, highest chunk first (the order the E warp needs them)
    int c = hi;
    while (c >= lo) {
        if (b5_bit(sh.cov[q], c)) {
            --c;
            continue;
        }
        int n = 0;
        while (n < kB5Win && c - n >= lo && !b5_bit(sh.cov[q], c - n)) {
            sh.cov[q][(c - n) >> 5] |= 1u << ((c - n) & 31);
            ++n;
        }
        atomicAdd(&sh.outstanding[q], 1);
        b5_count(trace, stats, 4, 1);
        __threadfence_block();
        b5_enqueue(sh, urgent ? 1 : 0, make_int4(s, c, n, 0), timeouts);
        c -= n;
    }
    __threadfence_block();
    atomicExch(&sh.lock[q], 0);
}

// ----------------------------------------------------------------------------
// Helper: recompute a window of tiles (strip s, chunks hi, hi-1, .., hi-n+1)
// from the checkpoints and write their P into the pool (rotated rows).
// kCost: 0 = skewed cost tensor (unfused), 1 = SIMT cost (fused, non-tensor-core).
// ----------------------------------------------------------------------------
template <class T, int kCost, int NE, int NH>
__device__ void b5_recompute(Bwd5Shared<T, NE, NH> &sh, const Dp3Args<T> &A, T *mypool, int b, int s, int cr,
                             int nt, int h, int t)
{
    const DpArgs<T> &a = A.a;
    using TG = Tagged<T>;
    const int q = s % kB5NQ;
    const int i = 32 * s + t + 1;
    const bool row_ok = i <= a.N;
    const int wr = min(32, a.M - 32 * cr);
    T *halo = &sh.hhalo[h][0][0];
    T lc[kB5Win], hp[kB5Win];
    T *dst[kB5Win];
#pragma unroll
    for (int z = 0; z < kB5Win; ++z) {
        const int cz = cr - z;
        lc[z] = (z < nt && cz > 0 && row_ok) ? a.vc[((size_t)b * a.C + (cz - 1)) * a.N + (i - 1)] : T(0);
        hp[z] = T(0);
        const int wz = z == 0 ? wr : 32;
        halo[z * 32 + t] = (z < nt && s > 0 && t < wz) ? TG::value(A.hbt + ((size_t)b * a.S + (s - 1)) * a.M + 32 * cz + t)
                                                       : T(0);
        dst[z] = mypool + ((size_t)q * a.C + max(cz, 0)) * 3 * 1024 + t;
    }
    __syncwarp();
    const bool fix = (s == 0) || (cr - nt + 1 <= 1) || (a.bw != 0);
    const T *dbase = (kCost == 0) ? a.dsk + ((size_t)b * a.S + s) * (size_t)a.KK * 32 + t : nullptr;
    // costs of 8 steps per tile, loaded one sub-group ahead
    T dn[kB5Win][8];
    auto load_d = [&](int q8, T (&d)[kB5Win][8]) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int z = 0; z < kB5Win; ++z) {
                const int kkr = 32 * (cr - z) + q8 + kk;  // skewed row of the step
                d[z][kk] = (kCost == 0 && z < nt && kkr < a.KK) ? dbase[(size_t)kkr * 32] : T(0);
            }
    };
    if (kCost == 0) load_d(0, dn);
    for (int q8 = 0; q8 < 64; q8 += 8) {
        T d8[kB5Win][8], hs8[kB5Win][8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
#pragma unroll
            for (int z = 0; z < kB5Win; ++z) {
                d8[z][kk] = dn[z][kk];
                hs8[z][kk] = halo[z * 32 + ((q8 + kk) & 31)];
            }
        if (kCost == 0 && q8 + 8 < 64) load_d(q8 + 8, dn);
        auto rsteps = [&](auto fix_tag) {
            constexpr bool kFix = decltype(fix_tag)::value;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int qq = q8 + kk;
                T src[kB5Win], u[kB5Win];
#pragma unroll
                for (int z = 0; z < kB5Win; ++z) src[z] = (t == 31) ? hs8[z][kk] : hp[z];
#pragma unroll
                for (int z = 0; z < kB5Win; ++z) u[z] = __shfl_sync(kFull, src[z], (t + 31) & 31);
                const int jj = qq - t;
#pragma unroll
                for (int z = 0; z < kB5Win; ++z) {
                    const int wz = z == 0 ? wr : 32;
                    const bool act = z < nt && row_ok && jj >= 0 && jj < wz;
                    const int j = 32 * (cr - z) + 1 + jj;
                    T d = d8[z][kk];
                    if (kCost == 1) d = act ? load_cost<T, true>(a, b, s, t, i, j) : T(0);
                    T v, hh, pd, pu, pl;
                    if constexpr (kFix) {
                        const Cell<T> cc = dp_cell<T, true>(i, j, a.bw, d, u[z], lc[z], a.k, a.gln2);
                        v = cc.v; hh = cc.h; pd = cc.pd; pu = cc.pu; pl = cc.pl;
                    } else {
                        prob_cell<T>(d, u[z], lc[z], a.k, a.gln2, v, hh, pd, pu, pl);
                    }
                    if (act) {
                        B5_CHECK(cr - z >= 0 && cr - z < a.C && s >= 0 && s < a.S, "recompute tile", s, cr - z);
                        T *p = dst[z] + (qq & 31) * 32;
                        p[0] = pd;
                        p[1024] = pu;
                        p[2048] = pl;
                    }
                    lc[z] = act ? v : lc[z];
                    hp[z] = act ? hh : hp[z];
                }
            }
        };
        if (fix) rsteps(std::true_type{});
        else rsteps(std::false_type{});
    }
    __syncwarp();
}

template <class T, int kCost, int NE, int NH>
__device__ void b5_helper(Bwd5Shared<T, NE, NH> &sh, const Dp3Args<T> &A, T *mypool, int b, int h, int t,
                          int *timeouts)
{
    const bool tr = A.trace != nullptr;
    for (;;) {
        int4 job = make_int4(-1, 0, 0, 0);
        const long long tw0 = tr ? clock64() : 0;
        if (t == 0) {
            // take a job: urgent queue first; leave when the pair is done
            B5Spin sp(timeouts, 4, h, 0);
            for (;;) {
                bool got = false;
                for (int qu = 1; qu >= 0 && !got; --qu) {
                    const int hd = vld(sh.job_head[qu]);
                    if (hd < vld(sh.job_tail[qu]) && atomicCAS(&sh.job_head[qu], hd, hd + 1) == hd) {
                        const int cap = qu ? kB5UQ : kB5JQ;
                        const int p = hd % cap;
                        B5Spin sw(timeouts, 10, hd, qu);
                        bool ok = true;
                        while (vld(sh.job_seq[qu][p]) != hd + 1)
                            if (!sw.go(0)) {
                                ok = false;
                                break;
                            }
                        __threadfence_block();
                        job = sh.jobs[qu][p];
                        B5_CHECK(job.z >= 1, "job read", (long long)hd * 1000 + qu * 100 + p,
                                 (long long)job.x * 1000000 + job.y * 1000 + job.z);
                        if (!ok) job = make_int4(-1, 0, 0, 0);  // never run a half-published job
                        __threadfence_block();
                        vst(sh.job_rd[qu][p], hd);
                        got = true;
                    }
                }
                if (got) break;
                if (vld(sh.done)) break;  // job.x stays -1
                __nanosleep(32);
                if (!sp.go(0)) break;
            }
        }
        // broadcast through shared memory behind a warp barrier (lane 0 may
        // have spun in its own loop above)
        if (t == 0) sh.hjob[h] = job;
        __syncwarp();
        job = sh.hjob[h];
        __syncwarp();
        if (job.x < 0) return;
        B5_CHECK(job.x < A.a.S && job.y >= 0 && job.y < A.a.C && job.z >= 1 && job.z <= kB5Win && job.y - job.z + 1 >= 0,
                 "job", job.x * 65536 + job.y, job.z);
        const int q = job.x % kB5NQ;
        // skip a window its strip's E warp is already past (wasted work);
        // decided by lane 0 (e_pos moves under us: every lane must agree,
        // the recompute is full of warp collectives)
        bool live = false;
        if (t == 0) live = vld(sh.e_pos[q]) >= job.y - job.z + 1;
        live = __shfl_sync(kFull, live, 0);
        const long long tw1 = tr ? clock64() : 0;
        if (live) b5_recompute<T, kCost, NE, NH>(sh, A, mypool, b, job.x, job.y, job.z, h, t);
        if (tr && t == 0) {
            b5_count(A.trace, A.stats, live ? 6 : 5, live ? job.z : 1);
            b5_count(A.trace, A.stats, 13, (clock64() - tw1) >> 10);
            b5_count(A.trace, A.stats, 14, (tw1 - tw0) >> 10);
        }
        // the E warp reads the pool through L2 (ld.global.cg): the tiles must
        // be visible there before the ready bits are
        __threadfence();
        __syncwarp();
        if (t == 0) {
            for (int z = 0; z < job.z; ++z) {
                const int c = job.y - z;
                atomicOr(&sh.rdy[q][c >> 5], 1u << (c & 31));
            }
            __threadfence_block();
            atomicSub(&sh.outstanding[q], 1);
        }
    }
}

// ----------------------------------------------------------------------------
// E warp: one strip.
// ----------------------------------------------------------------------------
template <class T, int kCost, int NE, int NH>
__device__ void b5_strip(Bwd5Shared<T, NE, NH> &sh, const Dp3Args<T> &A, T *mypool, T *myspill, int b, int s, int k,
                         int seq, int t, int *timeouts, const FxScales &fx)
{
    const DpArgs<T> &a = A.a;
    const int q = s % kB5NQ;
    const int rme = seq & 1;
    const bool bottom = s == a.S - 1;
    const bool top = s == 0;
    // producer of my S input: strip s + 1
    const int kb = (k + NE - 1) % NE;
    const int rb = (k >= 1 ? seq : seq - 1) & 1;
    const int i = 32 * s + t + 1;
    const bool row_ok = i <= a.N;
    const int M = a.M;
    // S rings: the shared-memory ring holds the last kB5Ring columns; every
    // value also goes to the ring's full-width copy in global memory (L2),
    // read by a consumer that fell more than kB5Ring columns behind.  So a
    // producer never waits for its consumer (no back-pressure: the pipeline
    // holds only NE strips, and a full ring could otherwise wait on a strip
    // not yet started, whatever the band width).
    T *ring_me = sh.sring[k][rme];
    const T *ring_b = sh.sring[kb][rb];
    T *spill_me = myspill + (size_t)(2 * k + rme) * M;
    const T *spill_b = myspill + (size_t)(2 * kb + rb) * M;

    const bool tr = A.trace != nullptr;
    long long cy_tile = 0, cy_below = 0, cy_req = 0, n_runs = 0, n_tiles = 0;
    const long long cy_start = tr ? clock64() : 0;
    // ---- 1. my ring slot free (its previous consumer finished)
    if (t == 0) {
        B5Spin sp(timeouts, 5, s, k);
        while (vld(sh.cons_pos[k][rme]) != INT_MIN)
            if (!sp.go(0)) break;
    }
    // ---- 2. start chunk: the producer's upper bound of non-zero S
    int c0 = a.C - 1;
    int zab = M;  // producer's zero_above
    if (!bottom) {
        if (t == 0) {
            B5Spin sp(timeouts, 6, s, vld(sh.ring_strip[kb][rb]));
            while (vld(sh.ring_strip[kb][rb]) != s + 1 || vld(sh.zero_above[kb][rb]) < 0)
                if (!sp.go(0)) break;
            __threadfence_block();
            zab = vld(sh.zero_above[kb][rb]);
        }
        __syncwarp();  // lane 0 spun alone above: reconverge before the broadcast
        zab = __shfl_sync(kFull, zab, 0);
        c0 = zab > 0 ? (zab - 1) >> 5 : -1;
    }
    if (tr && t == 0) b5_count(A.trace, A.stats, 15, (clock64() - cy_start) >> 10);
    // ---- 3. publish my ring; its upper bound (zero_above) follows when this
    // strip's first sweep starts (everything right of it is dead for the
    // strip above, which then starts right there instead of scanning)
    if (t == 0) {
        vst(sh.zero_above[k][rme], -1);
        vst(sh.prod_pos[k][rme], M);
        vst(sh.intent_pos[k][rme], M);
        vst(sh.zero_below[k][rme], 0);
        vst(sh.cons_pos[k][rme], top ? INT_MIN : M);
        __threadfence_block();
        vst(sh.ring_strip[k][rme], s);
    }
    bool za_known = false;
    auto publish_top = [&](int za) {  // no S >= za from this strip
        if (!za_known && t == 0) {
            vst(sh.prod_pos[k][rme], za);
            vst(sh.intent_pos[k][rme], za);
            __threadfence_block();
            vst(sh.zero_above[k][rme], za);
        }
        za_known = true;
    };
    // S from below for columns [jl, jh] decided?  (bottom strip: all zero)
    auto wait_below = [&](int jl, int jh) -> int {
        int zb = 0;
        if (bottom) return INT_MAX;
        const long long c0_ = tr ? clock64() : 0;
        if (t == 0) {
            B5Spin sp(timeouts, 7, s, jl);
            for (;;) {
                zb = vld(sh.zero_below[kb][rb]);
                if (zb > jh || vld(sh.prod_pos[kb][rb]) <= jl) break;
                if (!sp.go(0)) break;
            }
            __threadfence_block();
        }
        if (tr) cy_below += clock64() - c0_;
        __syncwarp();  // lane 0 spun alone above: reconverge before the broadcast
        return __shfl_sync(kFull, zb, 0);
    };
    // (valid once the producer decided column j: wait_below).  Read the
    // ring first, then check that the producer had not started writing
    // column j - kB5Ring (which overwrites the slot): else the global copy.
    auto s_below = [&](int j, int zb) -> T {
        if (bottom || j >= zab || j < zb) return T(0);
        B5_CHECK(j >= 0 && j < M, "s_below", j, zb);
        const T v = ring_b[j & (kB5Ring - 1)];
        __threadfence_block();
        if (vld(sh.intent_pos[kb][rb]) > j - kB5Ring) return v;
        return ldcg(spill_b + j);
    };
    // the 8 columns hi, hi-1, .., hi-7 (>= lo) at once: one validation
    auto s_below8 = [&](int hi, int lo, int zb, T (&o)[8]) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int j = hi - kk;
            o[kk] = (bottom || j < lo || j >= zab || j < zb) ? T(0) : ring_b[j & (kB5Ring - 1)];
        }
        if (bottom) return;
        __threadfence_block();
        const int ip = vld(sh.intent_pos[kb][rb]);
        if (ip <= hi - kB5Ring) {  // rare: fell behind the ring
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int j = hi - kk;
                if (j >= lo && j < zab && j >= zb && ip <= j - kB5Ring) o[kk] = ldcg(spill_b + j);
            }
        }
    };

    T e_right = T(0), pl_right = T(0), pd_right = T(0), s_prev = T(0);
    int nstored = 0;
    int c = c0;
    // Speculative recompute for the strips above: the band of strip s - d
    // is predicted around chunk cc - d sigma (sigma = chunks per strip along
    // the diagonal, M / N), +-1 tile; requested kB5Ahead strips ahead, as a
    // tile's recompute (63 dependent steps) takes a few strip hops.
    const float sigma = (float)a.M / (float)a.N;
    auto request_up = [&](int cc) {
        const long long c0_ = tr ? clock64() : 0;
        if (t == 0)
            for (int d = 1, ahead = A.knob[0] ? A.knob[0] : kB5Ahead; d <= ahead; ++d) {
                const int ch = cc - __float2int_rn(d * sigma);
                b5_request(sh, s - d, ch - 1, ch + 1, a.C, false, timeouts, A.trace, A.stats);
            }
        if (tr) cy_req += clock64() - c0_;
    };
    auto tile_ready = [&](int cc) {
        const long long c0_ = tr ? clock64() : 0;
        if (t == 0) {
            if (!b5_bit(sh.cov[q], cc)) b5_request(sh, s, cc - (kB5Win - 1), cc, a.C, true, timeouts, A.trace, A.stats);
            b5_request(sh, s, cc - kB5Win, cc - 1, a.C, false, timeouts, A.trace, A.stats);
        }
        const long long c1_ = tr ? clock64() : 0;
        if (t == 0) {
            B5Spin sp(timeouts, 8, s, cc);
            while (!b5_bit(sh.rdy[q], cc))
                if (!sp.go(0)) break;
            __threadfence_block();
        }
        __syncwarp();
        if (tr) {
            cy_req += c1_ - c0_;
            cy_tile += clock64() - c1_;
            ++n_tiles;
        }
    };
    // flush a completed E tile: store it for the contraction if non-zero
    auto flush = [&](int cc) {
        T *et = &sh.et[k][cc % 3][0][0];
        const int width = min(32, M - 32 * cc);
        T v[32];
        bool nz = false;
#pragma unroll
        for (int r = 0; r < 32; ++r) {  // lane = column jj, v[r] = E(row r, jj)
            v[r] = et[((t + r) & 31) * 33 + r];
            nz |= v[r] != T(0);
        }
        if (!__any_sync(kFull, nz)) return;
        if (t == 0) atomicAdd(&A.stats[0], 1u);
        const int j0 = 32 * cc;
        if (a.E) {
            for (int r = 0; r < 32; ++r) {
                const int ir = 32 * s + r + 1;
                if (ir <= a.N && t < width) a.E[((size_t)b * a.N + (ir - 1)) * a.M + j0 + t] = v[r];
            }
        }
        B5_CHECK(cc >= 0 && cc < a.C && nstored <= a.C, "flush", cc, nstored);
        if (nstored < A.tile_quota) {
            const size_t slot = ((size_t)b * a.S + s) * A.tile_quota + nstored;
            T *dt = A.tiles + slot * 1024;
#pragma unroll
            for (int r = 0; r < 32; ++r) dt[r * 32 + t] = (t < width) ? v[r] : T(0);
            if (t == 0) A.tile_meta[slot] = make_int4(b, s, cc, width);
            ++nstored;
        } else {
            // rare: the capped tile store is full; contract here into the
            // fixed-point accumulators (natural layout in place, the tile's
            // P slot in the pool as scratch: its E warp is past it)
            if (t == 0) atomicAdd(&A.stats[2], 1u);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 32; ++r) et[r * 33 + t] = v[r];
            __syncwarp();
            T *scratch = mypool + ((size_t)q * a.C + cc) * 3 * 1024;
            tile_contract_fx<T>(A, fx, b, s, cc, width, et, scratch, t, 33);
        }
        __syncwarp();
    };

    if (c0 >= 0) {
        if (t == 0) b5_request(sh, s, c0, c0, a.C, false, timeouts);
    }
    bool carry = false;  // E leaves the last drained tile on some row: sweep on
    while (c >= 0) {
        // ---------------- idle at chunk c: no E from the right ----------------
        const bool end_tile = bottom && c == a.C - 1;
        const int jl = 32 * c, jh = min(M, 32 * c + 32) - 1;
        if (t == 0) vst(sh.e_pos[q], c);  // tiles > c are never read again
        if (!carry && !end_tile) {
            if (bottom) break;  // bottom strip: nothing enters from below
            const int zb = wait_below(jl, jh);
            if (zb > jh) break;  // everything from here left is dead
            const T sv = (jl + t <= jh) ? s_below(jl + t, zb) : T(0);
            if (__any_sync(kFull, sv != T(0))) goto sweep;
            // dead chunk: zero S for the strip above (nothing to write while
            // no sweep has started: it is above this strip's zero_above)
            if (!top && za_known) {
                if (t == 0) vst(sh.intent_pos[k][rme], jl);
                __syncwarp();
                __threadfence_block();
                if (jl + t <= jh) {
                    ring_me[(jl + t) & (kB5Ring - 1)] = T(0);
                    spill_me[jl + t] = T(0);
                }
                __syncwarp();
                if (t == 0) {
                    __threadfence_block();
                    vst(sh.prod_pos[k][rme], jl);
                }
            }
            --c;
            continue;
        }
    sweep:
        // ---------------- sweep from chunk c ----------------
        publish_top(min(M, 32 * c + 32));
        const int J = 32 * c + 31;
        int Jstop = INT_MIN;  // columns < Jstop are outside the run (set when it ends)
        int lowest = c;       // lowest chunk lane 31 entered
        int flush_next = c;
        ++n_runs;
        request_up(c);
        tile_ready(c);
        if (t == 0) vst(sh.e_pos[q], c);
        bool nz_tile = false;  // any E != 0 in the newest tile so far
        // probabilities of a sub-group's cells (rotated rows r, uniform),
        // loaded from the pool one sub-group ahead; only tiles >= lowest are
        // known ready, so an entry sub-group reloads its new tile's cells
        T pd8[8], pu8[8], pl8[8], pdn[8], pun[8], pln[8];
        auto load_p = [&](int l31x, int lowx, T (&pd)[8], T (&pu)[8], T (&pl)[8], bool only_new, int newc) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int j = l31x - kk + 31 - t;
                bool ld = j >= Jstop && j <= J && j >= 32 * lowx && j >= 0;
                if (only_new) ld = ld && (j >> 5) == newc;
                if (ld) {
                    const int cj = j >> 5;
                    B5_CHECK(cj >= 0 && cj < a.C, "P load", cj, j);
                    const T *pt = mypool + ((size_t)q * a.C + cj) * 3 * 1024 + ((l31x - kk + 31) & 31) * 32 + t;
                    pd[kk] = ldcg(pt);
                    pu[kk] = ldcg(pt + 1024);
                    pl[kk] = ldcg(pt + 2048);
                } else if (!only_new) {
                    pd[kk] = T(0);
                    pu[kk] = T(0);
                    pl[kk] = T(0);
                }
            }
        };
        load_p(J, lowest, pdn, pun, pln, false, 0);
        for (int g = 0;; ++g) {
            const int k0 = 8 * g;
            const int l31 = J - k0;  // lane 31's column at the sub-group's first step
            if (g > 0 && l31 >= Jstop && (l31 & 31) == 31) {
                // lane 31 enters chunk cn: continue the run?
                const int cn = l31 >> 5;
                const int zb2 = wait_below(l31 - 7, l31);
                T s8 = T(0);
                if (t < 8) s8 = s_below(l31 - t, zb2);
                const bool cont = cn >= 0 && (__any_sync(kFull, s8 != T(0)) || __any_sync(kFull, nz_tile));
                if (!cont) {
                    Jstop = 32 * cn + 32;
                } else {
                    request_up(cn);
                    tile_ready(cn);
                    lowest = cn;
                    nz_tile = false;
                    load_p(l31, lowest, pdn, pun, pln, true, cn);  // the new tile's cells of this sub-group
                }
            }
            const int l0 = l31 + 31;  // lane 0's column at the first step
            if (l0 < Jstop) break;    // lane 0 has left the run
            const bool l31_on = l31 >= Jstop;
            // S from below for lane 31's columns this sub-group
            T si8[8];
            if (l31_on) {
                const int lo = max(l31 - 7, Jstop);
                const int zb2 = wait_below(lo, l31);
                s_below8(l31, lo, zb2, si8);
            } else {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) si8[kk] = T(0);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                pd8[kk] = pdn[kk];
                pu8[kk] = pun[kk];
                pl8[kk] = pln[kk];
            }
            load_p(l31 - 8, lowest, pdn, pun, pln, false, 0);  // next sub-group (tiles already ready)
            T so8[8];
            bool nzg = false;
            const bool fixg = a.bw != 0 || (bottom && l31 - 7 <= M - 1 && M - 1 <= l0);
            auto esteps = [&](auto fix_tag) {
                constexpr bool kFix = decltype(fix_tag)::value;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int j = l31 - kk + 31 - t;  // this lane's column (0-based)
                    const bool in_run = j >= Jstop && j <= J && j >= 32 * lowest;
                    const bool cell = in_run && row_ok && j < M;
                    // lane 31 takes S from below through lane 0 (whose own s_prev
                    // goes to the ring, not down the warp)
                    const T src = (t == 0) ? si8[kk] : s_prev;
                    const T s_in = __shfl_sync(kFull, src, (t + 1) & 31);
                    T e = fma(e_right, pl_right, s_in);
                    e = e < T(1) ? e : T(1);
                    if constexpr (kFix) {
                        e = (i == a.N && j + 1 == a.M) ? T(1) : e;
                        e = in_band(i, j + 1, a.bw) ? e : T(0);
                    }
                    e = cell ? e : T(0);
                    const T s_out = cell ? fma(e, pu8[kk], e_right * pd_right) : s_prev;
                    e_right = cell ? e : e_right;
                    pl_right = cell ? pl8[kk] : pl_right;
                    pd_right = cell ? pd8[kk] : pd_right;
                    if (in_run) sh.et[k][(j >> 5) % 3][(j + t) & 31][t] = e;
                    nzg |= e != T(0);
                    so8[kk] = s_out;
                    s_prev = s_out;
                }
            };
            if (fixg) esteps(std::true_type{});
            else esteps(std::false_type{});
            nz_tile |= nzg;
            // lane 0's S output for columns l0 - kk (those inside the run)
            if (!top) {
                const int lo0 = max(l0 - 7, max(Jstop, 32 * lowest));
                if (l0 >= lo0 && l0 <= J + 31) {
                    if (t == 0) {
                        vst(sh.intent_pos[k][rme], lo0);
                        __threadfence_block();
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const int j = l0 - kk;
                            if (j >= lo0 && j <= J) {
                                B5_CHECK(j >= 0 && j < M, "spill write", j, lo0);
                                ring_me[j & (kB5Ring - 1)] = so8[kk];
                                spill_me[j] = so8[kk];
                            }
                        }
                        __threadfence_block();
                        if (lo0 <= J) vst(sh.prod_pos[k][rme], lo0);
                    }
                }
            }
            __syncwarp();
            // flush tiles lane 0 has completed (it processed their column 32 cc)
            const int l0_last = l0 - 7;
            while (flush_next >= lowest && 32 * flush_next >= l0_last && flush_next >= (Jstop == INT_MIN ? 0 : (Jstop >> 5))) {
                flush(flush_next);
                --flush_next;
            }
            if (t == 0) vst(sh.e_pos[q], max(l0_last, 0) >> 5);
        }
        // flush what the drain completed
        while (flush_next >= lowest && flush_next >= (Jstop >> 5)) {
            flush(flush_next);
            --flush_next;
        }
        c = (Jstop >> 5) - 1;
        carry = __any_sync(kFull, e_right != T(0));  // E leaves the drained tile on some row
    }
    // ---- strip done: everything left of chunk c + 1 carries no S upward
    publish_top(0);  // never swept: the whole strip is dead
    if (t == 0) {
        const int zbme = 32 * (c + 1);
        __threadfence_block();
        vst(sh.zero_below[k][rme], max(zbme, 0));
        vst(sh.prod_pos[k][rme], max(zbme, 0));
        if (!bottom) vst(sh.cons_pos[kb][rb], INT_MIN);  // release the producer's ring
        vst(sh.e_pos[q], -1);                            // no tile of this strip is needed any more
        A.strip_tiles[(size_t)b * a.S + s] = nstored;
        if (tr) {
            b5_count(A.trace, A.stats, 7, cy_tile >> 10);
            b5_count(A.trace, A.stats, 8, cy_below >> 10);
            b5_count(A.trace, A.stats, 9, cy_req >> 10);
            b5_count(A.trace, A.stats, 10, (clock64() - cy_start) >> 10);
            b5_count(A.trace, A.stats, 11, n_runs);
            b5_count(A.trace, A.stats, 12, n_tiles);
        }
    }
    __syncwarp();
}

// ----------------------------------------------------------------------------
// The kernel: persistent CTAs over pair tickets (a.tickets[1]).
// ----------------------------------------------------------------------------
template <class T, int kCost, int NE, int NH>
__global__ void __launch_bounds__(32 * (NE + NH), 1) sdtw_backward5_kernel(Dp3Args<T> A, T *pool, T *spill,
                                                                          int *timeouts)
{
    extern __shared__ __align__(16) uint8_t smem_raw[];
    auto &sh = *reinterpret_cast<Bwd5Shared<T, NE, NH> *>(smem_raw);
    const DpArgs<T> &a = A.a;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    T *mypool = pool + (size_t)blockIdx.x * kB5NQ * a.C * 3 * 1024;
    T *myspill = spill + (size_t)blockIdx.x * 2 * NE * a.M;
    for (;;) {
        if (threadIdx.x == 0) sh.pair = (int)atomicAdd(&a.tickets[1], 1u);
        for (int e = threadIdx.x; e < NE * 2; e += blockDim.x) {
            (&sh.ring_strip[0][0])[e] = -1;
            (&sh.cons_pos[0][0])[e] = INT_MIN;
            (&sh.zero_above[0][0])[e] = 0;
            (&sh.prod_pos[0][0])[e] = INT_MAX;
            (&sh.intent_pos[0][0])[e] = INT_MAX;
            (&sh.zero_below[0][0])[e] = 0;
        }
        for (int e = threadIdx.x; e < kB5NQ; e += blockDim.x) {
            sh.slot_strip[e] = -1;
            sh.lock[e] = 0;
            sh.outstanding[e] = 0;
            sh.e_pos[e] = INT_MAX;
        }
        for (int e = threadIdx.x; e < kB5JQ; e += blockDim.x) {
            sh.jobs[0][e] = make_int4(-3, -3, -3, -3);
            sh.jobs[1][e] = make_int4(-3, -3, -3, -3);
            sh.job_seq[0][e] = 0;
            sh.job_rd[0][e] = e - kB5JQ;
            sh.job_seq[1][e] = 0;
            sh.job_rd[1][e] = e - kB5UQ;
        }
        if (threadIdx.x == 0) {
            sh.job_tail[0] = sh.job_tail[1] = 0;
            sh.job_head[0] = sh.job_head[1] = 0;
            sh.done = 0;
        }
        __syncthreads();
        const int b = sh.pair;
        if (b >= a.B) break;
        if (warp < NE) {
            const FxScales fx = fx_scales(A.absmax + 2 * b, a.N, a.M);
            int seq = 0;
            for (int s = a.S - 1 - warp; s >= 0; s -= NE, ++seq)
                b5_strip<T, kCost, NE, NH>(sh, A, mypool, myspill, b, s, warp, seq, t, timeouts, fx);
            // the top strip is the last to finish: release the helpers (they
            // drain what is queued, skipping windows no strip needs)
            if (a.S - 1 - warp >= 0 && ((a.S - 1 - warp) % NE) == 0 && t == 0) {
                __threadfence_block();
                vst(sh.done, 1);
            }
        } else {
            b5_helper<T, kCost, NE, NH>(sh, A, mypool, b, warp - NE, t, timeouts);
        }
        __syncthreads();
    }
}

}  // namespace sdtw
