/*
 * sdtw_capi.h — the C-ABI boundary of the B200 Soft-DTW engine.
 *
 * The reference (arxiv/paper_2602_17206, /root/reference/proj) has no FFI
 * layer: its boundary is the header-only C++ template API in namespace
 * softdtw.  This C-ABI is what that API's bodies call in the drop-in headers
 * under include/softdtw/ (see INTEGRATION.md), and what the Python tests and
 * bench bind with ctypes.  Plain pointers and sizes only; no torch or CUDA
 * types in any signature (streams are passed as void*).
 *
 * Each entry point names the reference interface it replaces.  Reference
 * paths are relative to /root/reference/proj/include/softdtw/.
 *
 * Layouts (identical to the reference's containers):
 *   x  B x N x D, y  B x M x D  row-major                (types.hpp:160-209)
 *   costs  B x N x M row-major                            (types.hpp:247-276)
 *   R / E tables  B x (N+2) x (M+2), interior 1-based     (types.hpp:278-378)
 *   grad_x B x N x D, grad_y B x M x D                    (types.hpp:381-385)
 *
 * Pointer residency: every call takes `ptr_kind`; SDTW_PTR_HOST means all
 * array arguments are host memory (copies happen inside the call, on the
 * context's stream), SDTW_PTR_DEVICE means they are device pointers on the
 * context's device.  Calls are stream-ordered on the context stream and
 * return after the results are valid for the caller (host: copied back;
 * device: stream synchronized unless SDTW_FLAG_ASYNC is or-ed into ptr_kind).
 *
 * Errors: every call returns an sdtw_status; sdtw_last_error() returns a
 * thread-local message, sdtw_last_oom_bytes() the refused byte count for
 * SDTW_ENOMEM.  The C++ drop-in maps them back to the reference exception
 * types (types.hpp:17-54).
 */
#ifndef SDTW_CAPI_H
#define SDTW_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDTW_CAPI_VERSION 1

typedef enum sdtw_status {
    SDTW_OK = 0,
    SDTW_EINVAL = 1,       /* ValidationError        types.hpp:22-25   */
    SDTW_ENOMEM = 2,       /* OutOfMemoryError       types.hpp:29-41   */
    SDTW_EUNREACHABLE = 3, /* UnreachableEndError    types.hpp:45-48   */
    SDTW_EINCOMPLETE = 4,  /* IncompleteTableError   types.hpp:51-54   */
    SDTW_ECUDA = 5,        /* Error (device failure)                   */
    SDTW_ENCCL = 6         /* Error (collective failure)               */
} sdtw_status;

enum { SDTW_COST_UNFUSED = 0, SDTW_COST_FUSED = 1 };     /* CostMode      types.hpp:218 */
enum { SDTW_BWD_LOG = 0, SDTW_BWD_LINEAR = 1 };          /* BackwardSpace types.hpp:219 */
enum { SDTW_PTR_HOST = 0, SDTW_PTR_DEVICE = 1, SDTW_FLAG_ASYNC = 0x100 };

/* SdtwConfig (types.hpp:222-228).  `normalized` is handled by the caller
 * (forward_normalized, forward.hpp:85-102) and must be 0 here. */
typedef struct sdtw_config {
    double gamma;
    size_t bandwidth;
    int cost_mode;
    int backward_space;
    int normalized;
} sdtw_config;

typedef struct sdtw_ctx sdtw_ctx;

/* ---- context, stream, memory ledger (AllocationLedger types.hpp:60-88) -- */
int sdtw_ctx_create(int device, sdtw_ctx **out);
int sdtw_ctx_destroy(sdtw_ctx *ctx);
/* cudaStream_t as void*; NULL = the context's own stream. */
int sdtw_ctx_set_stream(sdtw_ctx *ctx, void *stream);
void *sdtw_ctx_stream(sdtw_ctx *ctx);
int sdtw_ctx_synchronize(sdtw_ctx *ctx);
/* Live and peak device bytes held by the engine's allocator. */
int sdtw_mem_stats(sdtw_ctx *ctx, size_t *live_bytes, size_t *peak_bytes);
int sdtw_mem_reset_peak(sdtw_ctx *ctx);
/* 0 = unlimited; over-limit allocations fail with SDTW_ENOMEM. */
int sdtw_set_mem_limit(sdtw_ctx *ctx, size_t limit_bytes);
/* Releases cached device blocks (live allocations are untouched). */
int sdtw_mem_trim(sdtw_ctx *ctx);
/* Number of kernel launches this context issued since the last reset. */
uint64_t sdtw_launch_count(sdtw_ctx *ctx);
void sdtw_reset_launch_count(sdtw_ctx *ctx);

/* Per-phase device timing of the most recent call on this context, taken
 * with CUDA events on the context stream (off by default).  Phases:
 * 0 norms, 1 cost tensor (unfused), 2 forward DP, 3 backward DP,
 * 4 input-gradient contraction.  ms[i] = -1 when a phase did not run. */
#define SDTW_NUM_PHASES 5
int sdtw_ctx_enable_timing(sdtw_ctx *ctx, int enable);
int sdtw_phase_times(sdtw_ctx *ctx, float *ms, int n);

/* Diagnostics: when trace_dev (device, 2 * B * S uint64) is non-NULL, the
 * forward DP records %globaltimer at each strip's start and end. */
int sdtw_debug_set_trace(sdtw_ctx *ctx, void *trace_dev);
/* Diagnostics (timing enabled): per phase 0 = not started, 1 = started,
 * 3 = finished (non-blocking event queries; -1 = phase did not run). */
int sdtw_debug_phase_status(sdtw_ctx *ctx, int *out, int n);
/* Diagnostics: fp32 fused-mode backward passes of this context (and its
 * host-call sub-contexts) that read the forward's band cache (out[0]) and,
 * of those, the ones whose alignment left the band and reran on the tensor
 * cores (out[1]).  Synchronises the context's stream. */
int sdtw_debug_band_stats(sdtw_ctx *ctx, unsigned long long *out);

const char *sdtw_last_error(void);
size_t sdtw_last_oom_bytes(void);

/* ---- the hot path: sdtw_with_gradients (backward.hpp:276-304) ----------
 * loss: B, grad_x: B*N*D, grad_y: B*M*D.  grad_x/grad_y may be NULL to skip
 * the input gradients (loss + E only). */
int sdtw_fwd_bwd_f32(sdtw_ctx *ctx, const float *x, const float *y, size_t B,
                     size_t N, size_t M, size_t D, const sdtw_config *cfg,
                     int ptr_kind, float *loss, float *grad_x, float *grad_y);
int sdtw_fwd_bwd_f64(sdtw_ctx *ctx, const double *x, const double *y,
                     size_t B, size_t N, size_t M, size_t D,
                     const sdtw_config *cfg, int ptr_kind, double *loss,
                     double *grad_x, double *grad_y);

/* ---- forward (forward.hpp:43-81) ----------------------------------------
 * loss: B.  R_out (nullable): the padded accumulated-cost table
 * B*(N+2)*(M+2) with the reference's +inf boundary and R[b,0,0] = 0.
 * cfg->normalized = 1: forward_normalized (forward.hpp:85-102), loss =
 *   sdtw(x,y) - (sdtw(x,x) + sdtw(y,y)) / 2 (requires N == M; R_out /
 *   costs_out / norms_out then describe the (x, y) pass).
 * costs_out (nullable): the B*N*M cost tensor (unfused mode only).
 * norms_out (nullable): B*N then B*M squared norms (NormCache, cost.hpp:12-20). */
int sdtw_forward_f32(sdtw_ctx *ctx, const float *x, const float *y, size_t B,
                     size_t N, size_t M, size_t D, const sdtw_config *cfg,
                     int ptr_kind, float *loss, float *R_out, float *costs_out,
                     float *norms_out);
int sdtw_forward_f64(sdtw_ctx *ctx, const double *x, const double *y,
                     size_t B, size_t N, size_t M, size_t D,
                     const sdtw_config *cfg, int ptr_kind, double *loss,
                     double *R_out, double *costs_out, double *norms_out);

/* ---- standalone backward over a padded R table
 *      (backward_log :183-190 / backward_linear :196-203) --------------------
 * R: B*(N+2)*(M+2) as produced by forward.  The cost source is either the
 * B*N*M tensor `costs` (MaterializedCosts, cost.hpp:102-109) or, when costs
 * is NULL, x/y (FusedCosts, cost.hpp:112-121).  E_out: B*(N+2)*(M+2), linear
 * space, 0 outside the in-band interior (backward.hpp:161-176).
 * Arithmetic follows the reference recurrence on the given R values. */
int sdtw_backward_table_f32(sdtw_ctx *ctx, const float *R, const float *costs,
                            const float *x, const float *y, size_t B,
                            size_t N, size_t M, size_t D,
                            const sdtw_config *cfg, int ptr_kind,
                            float *E_out);
int sdtw_backward_table_f64(sdtw_ctx *ctx, const double *R,
                            const double *costs, const double *x,
                            const double *y, size_t B, size_t N, size_t M,
                            size_t D, const sdtw_config *cfg, int ptr_kind,
                            double *E_out);

/* ---- loss + alignment-gradient table E from the engine's own forward
 *      (forward + backward_log in one call, CS3 fast path) ---------------- */
int sdtw_forward_backward_E_f32(sdtw_ctx *ctx, const float *x, const float *y,
                                size_t B, size_t N, size_t M, size_t D,
                                const sdtw_config *cfg, int ptr_kind,
                                float *loss, float *E_out);
int sdtw_forward_backward_E_f64(sdtw_ctx *ctx, const double *x,
                                const double *y, size_t B, size_t N, size_t M,
                                size_t D, const sdtw_config *cfg,
                                int ptr_kind, double *loss, double *E_out);

/* ---- input_gradients (backward.hpp:208-266) ---------------------------- */
int sdtw_input_grads_f32(sdtw_ctx *ctx, const float *E, const float *x,
                         const float *y, size_t B, size_t N, size_t M,
                         size_t D, int ptr_kind, float *grad_x,
                         float *grad_y);
int sdtw_input_grads_f64(sdtw_ctx *ctx, const double *E, const double *x,
                         const double *y, size_t B, size_t N, size_t M,
                         size_t D, int ptr_kind, double *grad_x,
                         double *grad_y);

/* ---- barycenter_objective (barycenter.hpp:60-86) ------------------------
 * z: Lz*D, members: K*L*D (equal lengths), weights: K or NULL (all ones).
 * value: sum_k w_k * sdtw(z, x_k) accumulated in double; grad: Lz*D.
 * All members run as one batch on the device (z broadcast). */
int sdtw_barycenter_objective_f32(sdtw_ctx *ctx, const float *z, size_t Lz,
                                  const float *members, size_t K, size_t L,
                                  size_t D, double gamma, size_t bandwidth,
                                  const double *weights, int ptr_kind,
                                  double *value, float *grad);
int sdtw_barycenter_objective_f64(sdtw_ctx *ctx, const double *z, size_t Lz,
                                  const double *members, size_t K, size_t L,
                                  size_t D, double gamma, size_t bandwidth,
                                  const double *weights, int ptr_kind,
                                  double *value, double *grad);

/* ---- Adam step (barycenter.hpp:181-191): fp64 moments, z updated in place.
 * All arrays of length n, device or host per ptr_kind. */
int sdtw_adam_step_f32(sdtw_ctx *ctx, float *z, const float *grad, double *m1,
                       double *m2, size_t n, size_t t, double lr,
                       double beta1, double beta2, double eps, int ptr_kind);
int sdtw_adam_step_f64(sdtw_ctx *ctx, double *z, const double *grad,
                       double *m1, double *m2, size_t n, size_t t, double lr,
                       double beta1, double beta2, double eps, int ptr_kind);

/* ---- multi-GPU barycenter (NCCL allreduce over NVLink) ------------------
 * One rank per process/GPU.  `uid` is a 128-byte ncclUniqueId produced by
 * sdtw_nccl_get_unique_id on rank 0 and broadcast by the caller. */
int sdtw_nccl_get_unique_id(void *uid128);
int sdtw_nccl_init(sdtw_ctx *ctx, const void *uid128, int nranks, int rank);
int sdtw_nccl_finalize(sdtw_ctx *ctx);
/* In-place sum over ranks: grad (n floats) and value (1 double). */
int sdtw_allreduce_grad_f32(sdtw_ctx *ctx, float *grad_dev, size_t n,
                            double *value_dev);

/* ---- multi-GPU, one process ----------------------------
 * G contexts, normally one per device (sdtw_ctx_create(g)).  The batch is
 * split into G contiguous pair shards [g B / G, (g+1) B / G) (the layout of
 * backward.hpp:276-304: pairs are independent), shard g runs on ctxs[g]
 * (its device, stream and allocator) from its own host thread, all shards
 * concurrently, with no collective; the results are bit for bit those of a
 * single context (per-pair operand scales).  Host pointers only
 * (ptr_kind = SDTW_PTR_HOST): each shard stages its own slice.  Replaces the
 * reference's single-host sdtw_with_gradients (backward.hpp:276-304) when
 * more than one GPU is visible. */
/* Number of visible CUDA devices (0 when none). */
int sdtw_device_count(int *n);
int sdtw_fwd_bwd_multi_f32(sdtw_ctx *const *ctxs, int G, const float *x,
                           const float *y, size_t B, size_t N, size_t M,
                           size_t D, const sdtw_config *cfg, int ptr_kind,
                           float *loss, float *grad_x, float *grad_y);
int sdtw_fwd_bwd_multi_f64(sdtw_ctx *const *ctxs, int G, const double *x,
                           const double *y, size_t B, size_t N, size_t M,
                           size_t D, const sdtw_config *cfg, int ptr_kind,
                           double *loss, double *grad_x, double *grad_y);
/* One NCCL communicator over the G contexts' devices of this process
 * (ncclCommInitAll); the devices must be distinct. */
int sdtw_nccl_init_all(sdtw_ctx *const *ctxs, int G);
/* barycenter_objective (barycenter.hpp:60-86) over G devices: members in
 * G contiguous shards, each device computes its shard's weighted objective
 * and grad_z, one NCCL allreduce(sum) of grad_z (fp32) and of the objective
 * (fp64) over the communicator of sdtw_nccl_init_all (the only collective,
 * replacing the sequential member loop at barycenter.hpp:77-84); every
 * device ends with the full sum, which is returned from ctxs[0] (host
 * pointers).  Deterministic for a fixed G. */
int sdtw_barycenter_objective_multi_f32(sdtw_ctx *const *ctxs, int G,
                                        const float *z, size_t Lz,
                                        const float *members, size_t K,
                                        size_t L, size_t D, double gamma,
                                        size_t bandwidth,
                                        const double *weights, int ptr_kind,
                                        double *value, float *grad);

#ifdef __cplusplus
}
#endif

#endif /* SDTW_CAPI_H */
