// Step-latency microbenchmark for the forward DP cell chain (one warp, or
// several warps per SM), variants of the per-step work.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float a){float r; asm("ex2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ float lg2(float a){float r; asm("lg2.approx.ftz.f32 %0, %1;":"=f"(r):"f"(a)); return r;}
__device__ __forceinline__ void cell(float d, float u, float l, float k, float gln2, float&g, float&v, float&h){
  const float lo=u<l?u:l, hi=u<l?l:u; const float mn=lo<0.f?lo:0.f, mx=hi>0.f?hi:0.f, hz=hi<0.f?hi:0.f, md=lo>hz?lo:hz;
  const float e1=ex2((mn-md)*k), e2=ex2((mn-mx)*k); const float s=(e1+e2)+1.f;
  g=d+(mn-gln2*lg2(s)); v=g-u; h=g-l; }
__device__ __forceinline__ void st_pred(unsigned long long* p, unsigned long long w, bool pr){
  asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; @q st.relaxed.gpu.global.b64 [%0], %1;}"::"l"(p),"l"(w),"r"((int)pr):"memory"); }
template<int V>
__global__ void k(const float* dsrc, unsigned long long* out, int steps, long long* cyc, float* sink){
  const int t=threadIdx.x&31; __shared__ float dring[1024]; __shared__ float halo[32];
  for(int i=t;i<1024;i+=32) dring[i]=dsrc[i]; halo[t]=1.f; __syncwarp();
  float hp=0.f, lc=0.f; const float kk=1.4427f/0.1f, gl=0.1f*0.6931f;
  long long c0=clock64();
  #pragma unroll 8
  for(int s=0;s<steps;++s){
    const float hs=halo[s&31];
    const float src=(t==31)?hs:hp; const float u=__shfl_sync(0xffffffffu,src,(t+31)&31);
    const float d=dring[(s&31)*32+t];
    float g,v,h; cell(d,u,lc,kk,gl,g,v,h); lc=v; hp=h;
    if(V==1){ if(t==31) { unsigned long long w=((unsigned long long)7<<32)|__float_as_uint(h); asm volatile("st.relaxed.gpu.global.b64 [%0], %1;"::"l"(out+s),"l"(w):"memory"); } }
    if(V==2){ unsigned long long w=((unsigned long long)7<<32)|__float_as_uint(h); st_pred(out+s,w,t==31); }
    if(V==3){ if(t==31) out[s]=__float_as_uint(h); }
  }
  long long c1=clock64();
  if(t==0 && blockIdx.x==0 && threadIdx.x==0) cyc[V]=(c1-c0);
  sink[blockIdx.x*blockDim.x+threadIdx.x]=hp+lc;
}
int main(){
  float* d; cudaMalloc(&d,4096*4); cudaMemset(d,0,4096*4);
  unsigned long long* o; cudaMalloc(&o,1<<20);
  long long* c; cudaMalloc(&c,64); float* sink; cudaMalloc(&sink,1<<24);
  const int steps=4096;
  for(int warps : {1,4,8,16}){
    for(int V=0;V<4;++V){
      auto kern = V==0?k<0>:V==1?k<1>:V==2?k<2>:k<3>;
      kern<<<148,32*warps>>>(d,o,steps,c,sink); cudaDeviceSynchronize();
      kern<<<148,32*warps>>>(d,o,steps,c,sink); cudaDeviceSynchronize();
      long long h[4]; cudaMemcpy(h,c,32,cudaMemcpyDeviceToHost);
      printf("warps/SM %2d variant %d: %.1f cycles/step\n",warps,V,(double)h[V]/steps);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
