#include <cstdio>
#include <cstdint>
__global__ void plain(){ extern __shared__ float s[]; if (threadIdx.x == 9999) s[0] = 1; }
__global__ void withtmem(int go){
  extern __shared__ float s[];
  __shared__ uint32_t tb;
  if (go && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"((uint32_t)__cvta_generic_to_shared(&tb)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tb) : "memory");
  }
  if (threadIdx.x == 9999) s[0] = 1;
}
int main(){
  for (int kb : {16, 48, 96}) {
    int o1 = 0, o2 = 0; size_t sm = kb * 1024;
    cudaFuncSetAttribute(plain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(withtmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, plain, 64, sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, withtmem, 64, sm);
    printf("%d KB: plain %d, with tcgen05.alloc %d\n", kb, o1, o2);
  }
}
