
#include <cstdio>
__global__ void k(){ extern __shared__ float s[]; if (threadIdx.x == 9999) s[0] = 1; }
int main(){
  for (int kb = 90; kb <= 116; kb += 1) {
    int occ = 0; size_t sm = kb * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 64, sm);
    printf("%d KB -> %d\n", kb, occ);
  }
  int v; cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0); printf("max smem/SM %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); printf("max smem/block optin %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, 0); printf("reserved/block %d\n", v);
}
