// mufu_rate.cu — measured MUFU (SFU) throughput on this GPU: ex2.approx,
// lg2.approx, rcp.approx (f32), and the forward cell's mix (2 ex2 + 1 lg2).
// The roofline denominator of the DP kernels (bench.py `roofline.peak`).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu
//   ./mufu_rate > profiles/mufu_r2.json
//
// Each thread runs 8 independent dependency chains of one MUFU op (plus a
// cheap FFMA to keep the chain's values finite and live); the kernel fills
// every SM with 32 warps.  Rate = lane-ops / (cycles of the slowest SM),
// cycles read with clock64 per CTA, so the result is in MUFU lane-ops per
// clock per SM, independent of the SM clock the run happened to get.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__device__ __forceinline__ float op(float a)
{
    float r;
    if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    if (OP == 1) asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}

template <int OP>
__global__ void __launch_bounds__(1024) mufu_kernel(float *out, long long *cyc, int iters)
{
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.5f + 0.01f * (threadIdx.x + k);
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 3) {  // forward-cell mix: 2 ex2 + 1 lg2 per cell
                const float e1 = op<0>(v[k] * -0.25f), e2 = op<0>(v[k] * -0.5f);
                v[k] = op<1>(1.0f + e1 + e2) + 0.5f;
            } else {
                v[k] = fmaf(op<OP>(v[k]), 0.25f, 0.5f);
            }
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
double run(int sms, int iters, float *out, long long *cyc, float *ms)
{
    const int blocks = sms;  // one 1024-thread CTA per SM
    mufu_kernel<OP><<<blocks, 1024>>>(out, cyc, iters);  // warm-up
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mufu_kernel<OP><<<blocks, 1024>>>(out, cyc, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    long long h[4096];
    cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    const double per_op = OP == 3 ? 3.0 : 1.0;
    const double lane_ops_per_sm = 1024.0 * 8.0 * iters * per_op;
    return lane_ops_per_sm / (double)mx;
}

int main()
{
    cudaDeviceProp p{};
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * 4096);
    const int iters = 4096;
    float ms[4];
    const double ex2 = run<0>(sms, iters, out, cyc, &ms[0]);
    const double lg2 = run<1>(sms, iters, out, cyc, &ms[1]);
    const double rcp = run<2>(sms, iters, out, cyc, &ms[2]);
    const double mix = run<3>(sms, iters, out, cyc, &ms[3]);
    const double ops = (double)sms * 1024 * 8 * iters;
    std::printf("{\"gpu\": \"%s\", \"sm_count\": %d, \"ex2_per_clk_sm\": %.3f, \"lg2_per_clk_sm\": %.3f, "
                "\"rcp_per_clk_sm\": %.3f, \"fwd_mix_per_clk_sm\": %.3f, "
                "\"ex2_gops_wall\": %.1f, \"lg2_gops_wall\": %.1f, \"rcp_gops_wall\": %.1f, "
                "\"fwd_mix_gops_wall\": %.1f, \"method\": \"8 independent chains per thread, 1024 threads x "
                "%d CTAs, clock64 per CTA (slowest SM); gops_wall from CUDA events\"}\n",
                p.name, sms, ex2, lg2, rcp, mix, ops / (ms[0] * 1e6), ops / (ms[1] * 1e6), ops / (ms[2] * 1e6),
                3 * ops / (ms[3] * 1e6), sms);
    return 0;
}
