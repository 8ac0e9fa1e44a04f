// numerics_emu.cpp — design experiment (not product, not oracle).
//
// Emulates, on the CPU and in fp32, the arithmetic the B200 kernels use:
//   * costs d by the norm expansion in fp32 (optionally with the dot product
//     rounded like a 1-pass fp16/TF32 tensor-core MMA, or a 3-pass split);
//   * the forward DP in "edge-difference" form: every cell keeps only
//     v = R(i,j) - R(i-1,j) and h = R(i,j) - R(i,j-1) in fp32 (never R), and
//     the softmin is taken over (0, u, l) with u = R(i-1,j) - R(i-1,j-1),
//     l = R(i,j-1) - R(i-1,j-1);  loss = sum of g = R(i,j) - R(i-1,j-1)
//     along the diagonal (+ the straight tail) accumulated in double;
//   * the backward as the LINEAR recurrence over the forward softmin
//     probabilities  E(i,j) = sum_s E(s) * P_s(i,j)  (all weights in [0,1]);
//   * MUFU ex2/lg2/rcp modelled with +-2^-22 relative noise.
// and compares loss and gradients with the reference's T=double path
// (oracle/_ref/libsdtw_ref.so).  Prints the evidence table in DESIGN.md.
//
//   g++ -O2 -std=c++20 experiments/numerics_emu.cpp -ldl -o /tmp/emu && /tmp/emu
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

typedef int (*ref_wg_f64)(const double *, const double *, size_t, size_t,
                          size_t, size_t, double, size_t, int, int, unsigned,
                          double *, double *, double *);
typedef void (*ref_inputs)(size_t, size_t, size_t, unsigned long long,
                           float *, float *);

static std::mt19937_64 noise_rng(99);
static float mufu(float v)
{
    static std::uniform_real_distribution<double> u(-1.0, 1.0);
    return (float)((double)v * (1.0 + u(noise_rng) * std::ldexp(1.0, -22)));
}

enum DotMode { DOT_FP32 = 0, DOT_FP16X1 = 1, DOT_FP16X3 = 2, DOT_F64 = 3 };

static float round_fp16(float v)  // RN to 11 significant bits (range ok here)
{
    if (v == 0) return 0;
    int e;
    std::frexp(v, &e);
    const double q = std::ldexp(1.0, e - 11);
    return (float)(std::nearbyint(v / q) * q);
}

struct Stats {
    double loss_rel = 0, grad_max = 0, grad_p99 = 0, e11 = 0;
};

static Stats run(const float *x, const float *y, size_t B, size_t N, size_t M,
                 size_t D, double gamma_d, DotMode dm, bool mufu_noise,
                 const double *rl, const double *rgx, const double *rgy)
{
    const float gamma = (float)gamma_d;
    const float k = (float)(1.4426950408889634 / gamma_d);  // log2e/gamma
    const float gln2 = (float)(gamma_d * 0.6931471805599453);
    std::vector<double> errs;
    Stats st;
    for (size_t b = 0; b < B; ++b) {
        const float *xb = x + b * N * D, *yb = y + b * M * D;
        std::vector<float> xn(N), yn(M);
        for (size_t i = 0; i < N; ++i) {
            float s = 0;
            for (size_t kk = 0; kk < D; ++kk)
                s = std::fma(xb[i * D + kk], xb[i * D + kk], s);
            xn[i] = s;
        }
        for (size_t j = 0; j < M; ++j) {
            float s = 0;
            for (size_t kk = 0; kk < D; ++kk)
                s = std::fma(yb[j * D + kk], yb[j * D + kk], s);
            yn[j] = s;
        }
        auto cost = [&](size_t i, size_t j) {  // 0-based
            if (dm == DOT_F64) {
                double s2 = 0;
                for (size_t kk = 0; kk < D; ++kk) {
                    const double df = (double)xb[i * D + kk] - (double)yb[j * D + kk];
                    s2 += df * df;
                }
                return (float)s2;
            }
            float dot = 0;
            for (size_t kk = 0; kk < D; ++kk) {
                const float a = xb[i * D + kk], c = yb[j * D + kk];
                if (dm == DOT_FP32) {
                    dot = std::fma(a, c, dot);
                } else {
                    const float ah = round_fp16(a), ch = round_fp16(c);
                    float p = ah * ch;
                    if (dm == DOT_FP16X3) {
                        const float al = round_fp16(a - ah),
                                    cl = round_fp16(c - ch);
                        p = p + (ah * cl + al * ch);
                    }
                    dot += p;
                }
            }
            float v = xn[i] - 2.0f * dot + yn[j];
            return v < 0 ? 0.0f : v;
        };
        // forward: v, h per cell (N x M), probabilities P (3 per cell)
        const float INF = INFINITY;
        std::vector<float> V(N * M), H(N * M), Pd(N * M), Pu(N * M),
            Pl(N * M);
        double diag_sum = 0;
        for (size_t i = 0; i < N; ++i)
            for (size_t j = 0; j < M; ++j) {
                const float d = cost(i, j);
                float g, v, h, pd = 0, pu = 0, pl = 0;
                if (i == 0 && j == 0) {
                    g = d; v = -INF; h = -INF;
                } else if (i == 0) {
                    g = NAN; h = d; v = -INF; pl = 1;
                } else if (j == 0) {
                    g = NAN; v = d; h = -INF; pu = 1;
                } else {
                    const float u = H[(i - 1) * M + j], l = V[i * M + j - 1];
                    const float mn = std::min(0.0f, std::min(u, l));
                    float e0 = std::exp2((0.0f - mn) * -k);
                    float eu = std::exp2((u - mn) * -k);
                    float el = std::exp2((l - mn) * -k);
                    if (mufu_noise) { e0 = mufu(e0); eu = mufu(eu); el = mufu(el); }
                    const float s = e0 + eu + el;
                    float lg = std::log2(s);
                    if (mufu_noise) lg = mufu(lg);
                    const float sm = std::fma(-gln2, lg, mn);
                    g = d + sm;
                    v = g - u;
                    h = g - l;
                    float r = 1.0f / s;
                    if (mufu_noise) r = mufu(r);
                    pd = e0 * r; pu = eu * r; pl = el * r;
                }
                V[i * M + j] = v; H[i * M + j] = h;
                Pd[i * M + j] = pd; Pu[i * M + j] = pu; Pl[i * M + j] = pl;
                if (i == j) diag_sum += (i == 0) ? (double)d : (double)g;
            }
        // straight tail
        double loss = diag_sum;
        if (M > N) for (size_t j = N; j < M; ++j) loss += H[(N - 1) * M + j];
        if (N > M) for (size_t i = M; i < N; ++i) loss += V[i * M + (M - 1)];
        // backward (linear, probabilities)
        std::vector<float> E(N * M, 0.0f);
        for (size_t i = N; i-- > 0;)
            for (size_t j = M; j-- > 0;) {
                if (i == N - 1 && j == M - 1) { E[i * M + j] = 1; continue; }
                float e = 0;
                if (i + 1 < N) e = std::fma(E[(i + 1) * M + j], Pu[(i + 1) * M + j], e);
                if (j + 1 < M) e = std::fma(E[i * M + j + 1], Pl[i * M + j + 1], e);
                if (i + 1 < N && j + 1 < M)
                    e = std::fma(E[(i + 1) * M + j + 1], Pd[(i + 1) * M + j + 1], e);
                E[i * M + j] = std::min(e, 1.0f);
            }
        // gradients, fp32 accumulation
        auto rel = [](double a, double r) {
            return std::fabs(a - r) / std::max(1.0, std::fabs(r));
        };
        st.loss_rel = std::max(st.loss_rel, rel(loss, rl[b]));
        if (b == 0) st.e11 = E[0];
        for (size_t i = 0; i < N; ++i) {
            std::vector<float> acc(D, 0.0f);
            float mg = 0;
            for (size_t j = 0; j < M; ++j) {
                const float w = E[i * M + j];
                mg += w;
                for (size_t kk = 0; kk < D; ++kk)
                    acc[kk] = std::fma(w, yb[j * D + kk], acc[kk]);
            }
            for (size_t kk = 0; kk < D; ++kk) {
                const float gx = 2.0f * (xb[i * D + kk] * mg - acc[kk]);
                errs.push_back(rel(gx, rgx[(b * N + i) * D + kk]));
            }
        }
        for (size_t j = 0; j < M; ++j) {
            std::vector<float> acc(D, 0.0f);
            float mg = 0;
            for (size_t i = 0; i < N; ++i) {
                const float w = E[i * M + j];
                mg += w;
                for (size_t kk = 0; kk < D; ++kk)
                    acc[kk] = std::fma(w, xb[i * D + kk], acc[kk]);
            }
            for (size_t kk = 0; kk < D; ++kk) {
                const float gy = 2.0f * (yb[j * D + kk] * mg - acc[kk]);
                errs.push_back(rel(gy, rgy[(b * M + j) * D + kk]));
            }
        }
    }
    std::sort(errs.begin(), errs.end());
    st.grad_max = errs.back();
    st.grad_p99 = errs[(size_t)(0.99 * (errs.size() - 1))];
    return st;
}

int main(int argc, char **argv)
{
    void *h = dlopen("oracle/_ref/libsdtw_ref.so", RTLD_NOW);
    if (!h) { std::fprintf(stderr, "%s\n", dlerror()); return 1; }
    auto wg = (ref_wg_f64)dlsym(h, "ref_sdtw_with_gradients_f64");
    auto gen = (ref_inputs)dlsym(h, "ref_bench_inputs");
    struct Case { size_t Bgen, Bkeep, L, D; double gamma; };
    std::vector<Case> cases = {
        {32, 2, 256, 128, 1.0},   {32, 2, 256, 128, 0.01},
        {32, 2, 256, 128, 1e-3},  {32, 1, 1024, 128, 0.1},
        {32, 1, 1024, 128, 1e-3}, {32, 1, 256, 1024, 1.0},
    };
    if (argc > 2) {  // emu <x.f32> <y.f32> B L D gamma : raw fp32 inputs
        cases.clear();
    }
    if (argc == 2) cases.push_back({32, 1, 4096, 128, 0.01});
    if (argc > 2) {
        const size_t B = atoi(argv[3]), L = atoi(argv[4]), D = atoi(argv[5]);
        const double g = atof(argv[6]);
        std::vector<float> xf(B * L * D), yf(B * L * D);
        FILE *fx = fopen(argv[1], "rb"), *fy = fopen(argv[2], "rb");
        fread(xf.data(), 4, xf.size(), fx); fread(yf.data(), 4, yf.size(), fy);
        std::vector<double> xd(xf.begin(), xf.end()), yd(yf.begin(), yf.end());
        std::vector<double> rl(B), rgx(xd.size()), rgy(yd.size());
        wg(xd.data(), yd.data(), B, L, L, D, g, 0, 0, 1, 0, rl.data(), rgx.data(), rgy.data());
        for (int noise = 0; noise < 4; ++noise) {
            Stats s = run(xf.data(), yf.data(), B, L, L, D, g, noise >= 2 ? DOT_F64 : DOT_FP32, noise & 1, rl.data(), rgx.data(), rgy.data());
            std::printf("file noise=%d loss %.2e p99 %.2e max %.2e E11 %.7f\n", noise, s.loss_rel, s.grad_p99, s.grad_max, s.e11);
        }
        return 0;
    }
    std::printf("%-24s %-9s %-10s %-10s %-10s %-10s\n", "case", "dot",
                "loss_rel", "grad_p99", "grad_max", "E11");
    for (const auto &c : cases) {
        std::vector<float> xf(c.Bgen * c.L * c.D), yf(c.Bgen * c.L * c.D);
        gen(c.Bgen, c.L, c.D, 42, xf.data(), yf.data());
        // slice the first Bkeep pairs (pairs are independent)
        const size_t n = c.Bkeep * c.L * c.D;
        std::vector<double> xd(xf.begin(), xf.begin() + n),
            yd(yf.begin(), yf.begin() + n);
        std::vector<double> rl(c.Bkeep), rgx(n), rgy(n);
        wg(xd.data(), yd.data(), c.Bkeep, c.L, c.L, c.D, c.gamma, 0, 0, 1, 0,
           rl.data(), rgx.data(), rgy.data());
        for (DotMode dm : {DOT_FP32, DOT_FP16X1, DOT_FP16X3}) {
            Stats s = run(xf.data(), yf.data(), c.Bkeep, c.L, c.L, c.D,
                          c.gamma, dm, true, rl.data(), rgx.data(), rgy.data());
            char name[64];
            std::snprintf(name, sizeof name, "L=%zu D=%zu g=%g", c.L, c.D,
                          c.gamma);
            std::printf("%-24s %-9s %-10.2e %-10.2e %-10.2e %-10.7f\n", name,
                        dm == DOT_FP32 ? "fp32" : dm == DOT_FP16X1 ? "fp16x1"
                                                                   : "fp16x3",
                        s.loss_rel, s.grad_p99, s.grad_max, s.e11);
        }
    }
    return 0;
}
