// Per-step latency of forward-cell chain variants (one warp per SM).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float a){float r; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ float lg2(float a){float r; asm volatile("lg2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ float min3(float a,float b,float c){float r; asm("min.f32 %0, %1, %2, %3;":"=f"(r):"f"(a),"f"(b),"f"(c)); return r;}
__device__ __forceinline__ float max3(float a,float b,float c){float r; asm("max.f32 %0, %1, %2, %3;":"=f"(r):"f"(a),"f"(b),"f"(c)); return r;}
// V0: current cell
__device__ __forceinline__ void cell0(float d,float u,float l,float k,float gln2,float&v,float&h){
  const float lo=fminf(u,l), hi=fmaxf(u,l); const float mn=fminf(lo,0.f), mx=fmaxf(hi,0.f), md=fmaxf(lo,fminf(hi,0.f));
  const float e1=ex2((mn-md)*k), e2=ex2((mn-mx)*k); const float s=(e1+e2)+1.f;
  const float sm=mn-gln2*lg2(s); v=(d-u)+sm; h=(d-l)+sm; }
// V1: scaled domain, FMNMX3, folded epilogue
__device__ __forceinline__ void cell1(float d,float u,float l,float&v,float&h){
  const float mn=min3(u,l,0.f), mx=max3(u,l,0.f);
  const float md=min3(fmaxf(u,l),fmaxf(u,0.f),fmaxf(l,0.f));
  const float e1=ex2(mn-md), e2=ex2(mn-mx); const float s=(e1+e2)+1.f;
  const float L=lg2(s); v=((d-u)+mn)-L; h=((d-l)+mn)-L; }
// V2: scaled, 3 ex2 (no median)
__device__ __forceinline__ void cell2(float d,float u,float l,float&v,float&h){
  const float mn=min3(u,l,0.f);
  const float e0=ex2(mn), e1=ex2(mn-u), e2=ex2(mn-l); const float s=(e1+e2)+e0;
  const float L=lg2(s); v=((d-u)+mn)-L; h=((d-l)+mn)-L; }
template<int V>
__global__ void k(const float* dsrc, long long* cyc, float* sink, int steps, unsigned long long* gout){
  const int t=threadIdx.x&31; __shared__ float dring[1024]; __shared__ float halo[32]; __shared__ unsigned long long hx[128];
  for(int i=t;i<1024;i+=32) dring[i]=dsrc[i]*0.01f; halo[t]=0.5f; __syncwarp();
  float hp=0.f, lc=0.f; const float kk=1.4427f/0.1f, gl=0.1f*0.6931f;
  long long c0=clock64();
  #pragma unroll 8
  for(int s=0;s<steps;++s){
    const float hs=halo[s&31];
    const float src=(t==31)?hs:hp;
    float u;
    if (V==3) u = src; else u=__shfl_sync(0xffffffffu,src,(t+31)&31);
    const float d=dring[(s&31)*32+t];
    float v,h;
    if(V==0||V==3||V>=4) cell0(d,u,lc,kk,gl,v,h); else if(V==1) cell1(d,u,lc,v,h); else cell2(d,u,lc,v,h);
    lc=v; hp=h;
    if (V==4) { unsigned long long w=((unsigned long long)(s+7)<<32)|__float_as_uint(h);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.volatile.shared.u64 [%0], %1;\n\t}" :: "r"((unsigned)__cvta_generic_to_shared(&hx[s&127])), "l"(w), "r"((int)(t==31))); }
    if (V==5) { unsigned long long w=((unsigned long long)(s+7)<<32)|__float_as_uint(h);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.relaxed.gpu.global.b64 [%0], %1;\n\t}" :: "l"(gout+s), "l"(w), "r"((int)(t==31))); }
    if (V==6) { unsigned long long w=((unsigned long long)(s+7)<<32)|__float_as_uint(h);
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.relaxed.gpu.global.b64 [%0], %1;\n\t}" :: "l"(gout+s), "l"(w), "r"((int)(t==31)));
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.volatile.shared.u64 [%0], %1;\n\t}" :: "r"((unsigned)__cvta_generic_to_shared(&hx[s&127])), "l"(w), "r"((int)(t==31))); }
  }
  long long c1=clock64();
  if(threadIdx.x==0 && blockIdx.x==0) cyc[V]=(c1-c0);
  sink[blockIdx.x*blockDim.x+threadIdx.x]=hp+lc;
}
int main(){
  float* d; cudaMalloc(&d,4096*4); cudaMemset(d,0,4096*4);
  long long* c; cudaMalloc(&c,64); unsigned long long* go; cudaMalloc(&go, 8<<20); float* sink; cudaMalloc(&sink,1<<24);
  const int steps=8192;
  for(int warps : {1,8}){
    for(int V=0;V<7;++V){
      auto kern = V==0?k<0>:V==1?k<1>:V==2?k<2>:V==3?k<3>:V==4?k<4>:V==5?k<5>:k<6>;
      kern<<<148,32*warps>>>(d,c,sink,steps,go); kern<<<148,32*warps>>>(d,c,sink,steps,go); cudaDeviceSynchronize();
      long long h[8]; cudaMemcpy(h,c,64,cudaMemcpyDeviceToHost);
      printf("warps/SM %2d variant %d: %.1f cycles/step\n",warps,V,(double)h[V]/steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
