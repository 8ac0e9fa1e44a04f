/*
 * sdtw_oracle.c — plain-C restatement of the reference Soft-DTW path.
 *
 * TEST INFRASTRUCTURE ONLY (see sdtw_oracle.h).  Follows the reference's
 * arithmetic order operation for operation so that, compiled without FMA
 * contraction (oracle/Makefile: -ffp-contract=off, no -march), it reproduces
 * the reference's T=double results bit for bit.  That claim is checked
 * against the golden vectors in tests/golden/ by tests/test_oracle.py.
 *
 * Reference paths are relative to /root/reference/proj/include/softdtw/.
 */
#include "sdtw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static double dmin(double a, double b) { return b < a ? b : a; } /* std::min */
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */

/* softmin.hpp:22-31 — min-shifted softmin, total on +/-inf */
double oracle_softmin(double a, double b, double c, double gamma)
{
    const double mn = dmin(a, dmin(b, c));
    if (isinf(mn)) return mn;
    const double g = gamma;
    const double s = exp(-(a - mn) / g) + exp(-(b - mn) / g) +
                     exp(-(c - mn) / g);
    return mn - g * log(s);
}

/* softmin.hpp:41-47 — max-shifted three-way logsumexp */
double oracle_logsumexp3(double a, double b, double c)
{
    const double m = dmax(a, dmax(b, c));
    if (isinf(m)) return m;
    return m + log(exp(a - m) + exp(b - m) + exp(c - m));
}

/* cost.hpp:22-56 — sequential k loop per element */
void oracle_norms(const double *x, const double *y, size_t B, size_t N,
                  size_t M, size_t D, double *xn, double *yn)
{
    for (size_t b = 0; b < B; ++b) {
        for (size_t i = 0; i < N; ++i) {
            const double *e = x + (b * N + i) * D;
            double s = 0;
            for (size_t k = 0; k < D; ++k) s += e[k] * e[k];
            xn[b * N + i] = s;
        }
        for (size_t j = 0; j < M; ++j) {
            const double *e = y + (b * M + j) * D;
            double s = 0;
            for (size_t k = 0; k < D; ++k) s += e[k] * e[k];
            yn[b * M + j] = s;
        }
    }
}

/* cost.hpp:63-78 — norm expansion clamped at 0, 1-based (i, j) */
double oracle_cost_at(const double *x, const double *y, const double *xn,
                      const double *yn, size_t N, size_t M, size_t D,
                      size_t b, size_t i, size_t j)
{
    const double *xe = x + (b * N + (i - 1)) * D;
    const double *ye = y + (b * M + (j - 1)) * D;
    double dot = 0;
    for (size_t k = 0; k < D; ++k) dot += xe[k] * ye[k];
    const double v = xn[b * N + (i - 1)] - 2 * dot + yn[b * M + (j - 1)];
    return v < 0.0 ? 0.0 : v;
}

/* cost.hpp:82-99 — materialize_costs */
void oracle_costs(const double *x, const double *y, size_t B, size_t N,
                  size_t M, size_t D, double *d)
{
    double *xn = (double *)malloc(sizeof(double) * B * N);
    double *yn = (double *)malloc(sizeof(double) * B * M);
    oracle_norms(x, y, B, N, M, D, xn, yn);
    for (size_t b = 0; b < B; ++b)
        for (size_t i = 1; i <= N; ++i)
            for (size_t j = 1; j <= M; ++j)
                d[(b * N + (i - 1)) * M + (j - 1)] =
                    oracle_cost_at(x, y, xn, yn, N, M, D, b, i, j);
    free(xn);
    free(yn);
}

/* wavefront.hpp:31-36 */
int oracle_in_band(size_t i, size_t j, size_t bandwidth)
{
    if (bandwidth == 0) return 1;
    const size_t diff = i > j ? i - j : j - i;
    return diff <= bandwidth;
}

#define TAB(b, i, j) ((((b) * (N + 2) + (i)) * (M + 2)) + (j))

/*
 * forward.hpp:43-81.  The serial branch of sweep_forward
 * (wavefront.hpp:86-93) visits cells row-major; the parallel branch only
 * reorders write-disjoint cells, so both give these exact values.
 */
int oracle_forward(const double *x, const double *y, size_t B, size_t N,
                   size_t M, size_t D, double gamma, size_t bandwidth,
                   double *R, double *loss)
{
    double *d = (double *)malloc(sizeof(double) * B * N * M);
    oracle_costs(x, y, B, N, M, D, d);
    /* types.hpp:287-294: +inf fill, R[b,0,0] = 0 */
    const size_t cells = B * (N + 2) * (M + 2);
    for (size_t t = 0; t < cells; ++t) R[t] = INFINITY;
    for (size_t b = 0; b < B; ++b) R[TAB(b, 0, 0)] = 0.0;
    /* forward.hpp:25-37 */
    for (size_t b = 0; b < B; ++b)
        for (size_t ci = 0; ci < N; ++ci)
            for (size_t cj = 0; cj < M; ++cj) {
                if (!oracle_in_band(ci, cj, bandwidth)) continue;
                const size_t i = ci + 1, j = cj + 1;
                const double sm =
                    oracle_softmin(R[TAB(b, i - 1, j - 1)],
                                   R[TAB(b, i - 1, j)],
                                   R[TAB(b, i, j - 1)], gamma);
                R[TAB(b, i, j)] = d[(b * N + ci) * M + cj] + sm;
            }
    free(d);
    int rc = 0;
    for (size_t b = 0; b < B; ++b) {
        loss[b] = R[TAB(b, N, M)];
        if (!isfinite(loss[b])) rc = -1; /* forward.hpp:72-79 */
    }
    return rc;
}

/*
 * backward.hpp:29-177.  The reference walks anti-diagonals in reverse and
 * stages R of diagonals p, p+1, p+2 in a ring before overwriting the slab
 * with Ebar/E.  Reverse row-major order respects the same dependencies and
 * performs the same per-cell arithmetic; a full copy of R replaces the ring.
 */
int oracle_backward(double *slab, const double *d, size_t B, size_t N,
                    size_t M, double gamma, size_t bandwidth, int log_space)
{
    const size_t cells = B * (N + 2) * (M + 2);
    double *R = (double *)malloc(sizeof(double) * cells);
    memcpy(R, slab, sizeof(double) * cells);
    int incomplete = 0;
#define COST(b, i, j) d[((b) * N + ((i) - 1)) * M + ((j) - 1)]
    for (size_t b = 0; b < B; ++b) slab[TAB(b, 0, 0)] = INFINITY; /* :56 */
    for (size_t b = 0; b < B; ++b)
        for (size_t ci = N; ci-- > 0;)
            for (size_t cj = M; cj-- > 0;) {
                if (!oracle_in_band(ci, cj, bandwidth)) continue;
                const size_t i = ci + 1, j = cj + 1;
                if (ci == N - 1 && cj == M - 1) { /* :95-98 */
                    slab[TAB(b, i, j)] = log_space ? 0.0 : 1.0;
                    continue;
                }
                const double r_self = R[TAB(b, i, j)];
                if (isinf(r_self)) { /* :99-103 */
                    incomplete = 1;
                    continue;
                }
                /* :105-121 — a successor is dead if outside the grid or
                 * its staged R is +inf (out of band) */
                double down = -INFINITY, right = -INFINITY, diag = -INFINITY;
                if (ci + 1 < N) {
                    const double rs = oracle_in_band(ci + 1, cj, bandwidth)
                                          ? R[TAB(b, i + 1, j)]
                                          : INFINITY;
                    if (!isinf(rs))
                        down = (rs - r_self - COST(b, i + 1, j)) / gamma;
                }
                if (cj + 1 < M) {
                    const double rs = oracle_in_band(ci, cj + 1, bandwidth)
                                          ? R[TAB(b, i, j + 1)]
                                          : INFINITY;
                    if (!isinf(rs))
                        right = (rs - r_self - COST(b, i, j + 1)) / gamma;
                }
                if (ci + 1 < N && cj + 1 < M) {
                    const double rs = oracle_in_band(ci + 1, cj + 1, bandwidth)
                                          ? R[TAB(b, i + 1, j + 1)]
                                          : INFINITY;
                    if (!isinf(rs))
                        diag = (rs - r_self - COST(b, i + 1, j + 1)) / gamma;
                }
                if (log_space) { /* :123-137, Ebar = min(0, lse3) */
                    const double td =
                        isinf(down) ? -INFINITY : slab[TAB(b, i + 1, j)] + down;
                    const double tr = isinf(right)
                                          ? -INFINITY
                                          : slab[TAB(b, i, j + 1)] + right;
                    const double tg = isinf(diag)
                                          ? -INFINITY
                                          : slab[TAB(b, i + 1, j + 1)] + diag;
                    slab[TAB(b, i, j)] = dmin(0.0, oracle_logsumexp3(td, tr, tg));
                } else { /* :138-146 */
                    double acc = 0;
                    if (!isinf(down)) acc += exp(down) * slab[TAB(b, i + 1, j)];
                    if (!isinf(right))
                        acc += exp(right) * slab[TAB(b, i, j + 1)];
                    if (!isinf(diag))
                        acc += exp(diag) * slab[TAB(b, i + 1, j + 1)];
                    slab[TAB(b, i, j)] = acc;
                }
            }
#undef COST
    free(R);
    if (incomplete) return -2;
    /* :161-174 epilogue: in-band interior -> exp (log space), else 0 */
    for (size_t b = 0; b < B; ++b)
        for (size_t i = 0; i < N + 2; ++i)
            for (size_t j = 0; j < M + 2; ++j) {
                double *v = &slab[TAB(b, i, j)];
                const int interior = i >= 1 && i <= N && j >= 1 && j <= M &&
                                     oracle_in_band(i - 1, j - 1, bandwidth);
                if (!interior)
                    *v = 0.0;
                else if (log_space)
                    *v = exp(*v);
            }
    return 0;
}

/* backward.hpp:208-266 — row then column marginal reductions */
void oracle_input_gradients(const double *E, const double *x,
                            const double *y, size_t B, size_t N, size_t M,
                            size_t D, double *grad_x, double *grad_y)
{
    double *acc = (double *)malloc(sizeof(double) * D);
    for (size_t row = 0; row < B * N; ++row) {
        const size_t b = row / N, i = row % N;
        double marginal = 0;
        for (size_t k = 0; k < D; ++k) acc[k] = 0;
        for (size_t j = 0; j < M; ++j) {
            const double w = E[TAB(b, i + 1, j + 1)];
            marginal += w;
            const double *ye = y + (b * M + j) * D;
            for (size_t k = 0; k < D; ++k) acc[k] += w * ye[k];
        }
        const double *xe = x + (b * N + i) * D;
        for (size_t k = 0; k < D; ++k)
            grad_x[row * D + k] = 2 * (xe[k] * marginal - acc[k]);
    }
    for (size_t col = 0; col < B * M; ++col) {
        const size_t b = col / M, j = col % M;
        double marginal = 0;
        for (size_t k = 0; k < D; ++k) acc[k] = 0;
        for (size_t i = 0; i < N; ++i) {
            const double w = E[TAB(b, i + 1, j + 1)];
            marginal += w;
            const double *xe = x + (b * N + i) * D;
            for (size_t k = 0; k < D; ++k) acc[k] += w * xe[k];
        }
        const double *ye = y + (b * M + j) * D;
        for (size_t k = 0; k < D; ++k)
            grad_y[col * D + k] = 2 * (ye[k] * marginal - acc[k]);
    }
    free(acc);
}
#undef TAB

/* backward.hpp:276-304 */
int oracle_sdtw_with_gradients(const double *x, const double *y, size_t B,
                               size_t N, size_t M, size_t D, double gamma,
                               size_t bandwidth, int log_space, double *loss,
                               double *grad_x, double *grad_y)
{
    const size_t cells = B * (N + 2) * (M + 2);
    double *slab = (double *)malloc(sizeof(double) * cells);
    double *d = (double *)malloc(sizeof(double) * B * N * M);
    int rc = oracle_forward(x, y, B, N, M, D, gamma, bandwidth, slab, loss);
    if (rc == 0) {
        oracle_costs(x, y, B, N, M, D, d);
        rc = oracle_backward(slab, d, B, N, M, gamma, bandwidth, log_space);
    }
    if (rc == 0) oracle_input_gradients(slab, x, y, B, N, M, D, grad_x, grad_y);
    free(d);
    free(slab);
    return rc;
}

/* barycenter.hpp:60-86 — members sequential, value in double */
double oracle_barycenter_objective(const double *z, size_t Lz,
                                   const double *members, size_t K, size_t L,
                                   size_t D, double gamma, size_t bandwidth,
                                   const double *weights, double *grad)
{
    double value = 0;
    double *gx = (double *)malloc(sizeof(double) * Lz * D);
    double *gy = (double *)malloc(sizeof(double) * L * D);
    for (size_t i = 0; i < Lz * D; ++i) grad[i] = 0;
    for (size_t k = 0; k < K; ++k) {
        const double w = weights ? weights[k] : 1.0;
        if (w == 0) continue;
        double loss;
        oracle_sdtw_with_gradients(z, members + k * L * D, 1, Lz, L, D, gamma,
                                   bandwidth, 1, &loss, gx, gy);
        value += w * loss;
        for (size_t i = 0; i < Lz * D; ++i) grad[i] += w * gx[i];
    }
    free(gx);
    free(gy);
    return value;
}

/* barycenter.hpp:181-191 */
void oracle_adam_step(double *z, const double *grad, double *m1, double *m2,
                      size_t n, size_t t, double lr, double beta1,
                      double beta2, double eps)
{
    const double bc1 = 1.0 - pow(beta1, (double)t);
    const double bc2 = 1.0 - pow(beta2, (double)t);
    for (size_t i = 0; i < n; ++i) {
        const double g = grad[i];
        m1[i] = beta1 * m1[i] + (1.0 - beta1) * g;
        m2[i] = beta2 * m2[i] + (1.0 - beta2) * g * g;
        const double step = lr * (m1[i] / bc1) / (sqrt(m2[i] / bc2) + eps);
        z[i] -= step;
    }
}
