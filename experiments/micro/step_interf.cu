// Step chain latency with 8 stepping warps per SM, plus spinning helper warps
// (mbarrier try_wait loop, or shared-memory polling), as in the fused forward.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float a){float r; asm("ex2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ float lg2(float a){float r; asm("lg2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ void cell(float d, float u, float l, float k, float gln2, float&g, float&v, float&h){
  const float lo=fminf(u,l), hi=fmaxf(u,l); const float mn=fminf(lo,0.f), mx=fmaxf(hi,0.f), md=fmaxf(lo,fminf(hi,0.f));
  const float e1=ex2((mn-md)*k), e2=ex2((mn-mx)*k); const float s=(e1+e2)+1.f;
  const float sm=mn-gln2*lg2(s); g=d+sm; v=(d-u)+sm; h=(d-l)+sm; }
__device__ __forceinline__ uint32_t su32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
template<int MODE>
__global__ void __launch_bounds__(384,1) k(const float* dsrc, unsigned long long* out, int steps, long long* cyc, float* sink, int nstep_warps){
  const int w=threadIdx.x>>5, t=threadIdx.x&31;
  __shared__ float dring[8][1024]; __shared__ float halo[8][32]; __shared__ uint64_t bar; __shared__ volatile unsigned flag;
  if(threadIdx.x==0){ asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(su32(&bar))); flag=0; }
  __syncthreads();
  if (w >= nstep_warps) {
    if (MODE==1) { // try_wait spin on a barrier that completes only at the end
      while (true) { uint32_t ok; asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0,1,0,P;}":"=r"(ok):"r"(su32(&bar)):"memory"); if(ok) break; }
    } else if (MODE==2) { // volatile smem polling
      while (flag == 0) {}
    }
    return;
  }
  for(int i=t;i<1024;i+=32) dring[w][i]=dsrc[i]; halo[w][t]=1.f; __syncwarp();
  float hp=0.f, lc=0.f; const float kk=1.4427f/0.1f, gl=0.1f*0.6931f;
  long long c0=clock64();
  #pragma unroll 8
  for(int s=0;s<steps;++s){
    const float hs=halo[w][s&31];
    const float src=(t==31)?hs:hp; const float u=__shfl_sync(0xffffffffu,src,(t+31)&31);
    const float d=dring[w][(s&31)*32+t];
    float g,v,h; cell(d,u,lc,kk,gl,g,v,h); lc=v; hp=h;
    unsigned long long wv=((unsigned long long)7<<32)|__float_as_uint(h);
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; @q st.relaxed.gpu.global.b64 [%0], %1;}"::"l"(out+s),"l"(wv),"r"((int)(t==31)):"memory");
  }
  long long c1=clock64();
  if(t==0 && blockIdx.x==0 && w==0) cyc[MODE]=(c1-c0);
  sink[blockIdx.x*blockDim.x+threadIdx.x]=hp+lc;
  __syncwarp();
  if (w==0 && t==0) { flag=1; asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"::"r"(su32(&bar)):"memory"); }
}
int main(){
  float* d; cudaMalloc(&d,4096*4); cudaMemset(d,0,4096*4);
  unsigned long long* o; cudaMalloc(&o,1<<20);
  long long* c; cudaMalloc(&c,64); float* sink; cudaMalloc(&sink,1<<24);
  const int steps=4096;
  for (int nsw : {1, 4, 8}) {
    for(int M=0;M<3;++M){
      auto kern = M==0?k<0>:M==1?k<1>:k<2>;
      int threads = M==0 ? 32*nsw : 384;
      kern<<<148,threads>>>(d,o,steps,c,sink,nsw); cudaDeviceSynchronize();
      kern<<<148,threads>>>(d,o,steps,c,sink,nsw); cudaDeviceSynchronize();
      long long h[3]; cudaMemcpy(h,c,24,cudaMemcpyDeviceToHost);
      printf("stepping warps %d, helpers %s: %.1f cycles/step\n", nsw, M==0?"none":M==1?"try_wait spin":"smem poll", (double)h[M]/steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
