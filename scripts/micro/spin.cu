// One warp runs the forward-cell chain while 7 sibling warps of the CTA poll
// shared memory (tight / with nanosleep): does polling slow the worker?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float a){float r; asm volatile("ex2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ float lg2(float a){float r; asm volatile("lg2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ void cell0(float d,float u,float l,float k,float gln2,float&v,float&h){
  const float lo=fminf(u,l), hi=fmaxf(u,l); const float mn=fminf(lo,0.f), mx=fmaxf(hi,0.f), md=fmaxf(lo,fminf(hi,0.f));
  const float e1=ex2((mn-md)*k), e2=ex2((mn-mx)*k); const float s=(e1+e2)+1.f;
  const float sm=mn-gln2*lg2(s); v=(d-u)+sm; h=(d-l)+sm; }
template<int V>
__global__ void k(const float* dsrc, long long* cyc, float* sink, int steps){
  const int t=threadIdx.x&31, w=threadIdx.x>>5; __shared__ float dring[1024]; __shared__ float halo[32];
  __shared__ volatile unsigned long long flag[8];
  for(int i=threadIdx.x;i<1024;i+=blockDim.x) dring[i]=dsrc[i]*0.01f; if(threadIdx.x<32) halo[t]=0.5f; if (threadIdx.x<8) flag[threadIdx.x]=0; __syncthreads();
  if (w>0) {
    unsigned long long x=0; unsigned n=0;
    while (true) { x = flag[t&7]; if (__all_sync(0xffffffffu, x!=0)) break; if (V==1) __nanosleep(32); if (V==2) __nanosleep(200); ++n; }
    if (t==0 && blockIdx.x==0) cyc[8+w]=n;
    return;
  }
  float hp=0.f, lc=0.f; const float kk=1.4427f/0.1f, gl=0.1f*0.6931f;
  long long c0=clock64();
  #pragma unroll 8
  for(int s=0;s<steps;++s){
    const float hs=halo[s&31];
    const float src=(t==31)?hs:hp;
    float u=__shfl_sync(0xffffffffu,src,(t+31)&31);
    const float d=dring[(s&31)*32+t];
    float v,h; cell0(d,u,lc,kk,gl,v,h); lc=v; hp=h;
  }
  long long c1=clock64();
  if(t<8) flag[t]=1;
  if(threadIdx.x==0 && blockIdx.x==0) cyc[V]=(c1-c0);
  sink[blockIdx.x*blockDim.x+threadIdx.x]=hp+lc;
}
int main(){
  float* d; cudaMalloc(&d,4096*4); cudaMemset(d,0,4096*4);
  long long* c; cudaMalloc(&c,256); float* sink; cudaMalloc(&sink,1<<24);
  const int steps=8192;
  for (int warps : {1, 2, 4, 8}) for(int V=0;V<3;++V){
    auto kern = V==0?k<0>:V==1?k<1>:k<2>;
    kern<<<148,32*warps>>>(d,c,sink,steps); kern<<<148,32*warps>>>(d,c,sink,steps); cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h,c,128,cudaMemcpyDeviceToHost);
    printf("warps %d spin variant %d (0 tight, 1 sleep32, 2 sleep200): %.1f cycles/step\n",warps,V,(double)h[V]/steps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
