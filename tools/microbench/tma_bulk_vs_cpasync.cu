#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void issue1(uint64_t* bar, void* dst, const void* src, int bytes){
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(sa(bar)),"r"(bytes):"memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(dst)),"l"(src),"r"(bytes),"r"(sa(bar)):"memory");}
__device__ __forceinline__ void wait1(uint64_t* bar, uint32_t par){
  asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}"::"r"(sa(bar)),"r"(par):"memory");}
// mode 0: all threads wait + syncthreads, thread0 issues ; mode 1: thread 0 only waits/issues
__global__ void k_tma(const char* src, int chunk, int reps, int slots, int mode, unsigned long long* out){
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar=(uint64_t*)sm; unsigned char* buf=sm+256;
  if(threadIdx.x==0){for(int i=0;i<slots;i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;":::"memory");}
  __syncthreads();
  long long total=reps, qi=0;
  if(threadIdx.x==0) while(qi<slots&&qi<total){issue1(&bar[qi%slots], buf+(size_t)(qi%slots)*chunk, src+(size_t)(qi%6)*chunk, chunk);qi++;}
  unsigned long long t0=clock64();
  if(mode==0){
    for(long long q=0;q<total;q++){int s=q%slots; wait1(&bar[s],(q/slots)&1); __syncthreads();
      if(threadIdx.x==0&&qi<total){issue1(&bar[qi%slots], buf+(size_t)(qi%slots)*chunk, src+(size_t)(qi%6)*chunk, chunk);qi++;}}
  } else if(threadIdx.x==0){
    for(long long q=0;q<total;q++){int s=q%slots; wait1(&bar[s],(q/slots)&1);
      if(qi<total){issue1(&bar[qi%slots], buf+(size_t)(qi%slots)*chunk, src+(size_t)(qi%6)*chunk, chunk);qi++;}}
  }
  __syncthreads();
  unsigned long long t1=clock64();
  if(threadIdx.x==0) out[blockIdx.x]=t1-t0;
}
__global__ void k_cpa(const char* src, int chunk, int reps, unsigned long long* out){
  extern __shared__ __align__(128) unsigned char sm[];
  const int slots=4;
  unsigned long long t0=clock64();
  for(int q=0;q<reps+slots-1;q++){
    if(q<reps){int s=q%slots; const char* p=src+(size_t)(q%6)*chunk;
      for(int o=threadIdx.x*16;o<chunk;o+=blockDim.x*16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"::"r"(sa(sm+(size_t)s*chunk+o)),"l"(p+o):"memory");}
    asm volatile("cp.async.commit_group;":::"memory");
    if(q>=slots-1){asm volatile("cp.async.wait_group 3;":::"memory"); __syncthreads();}
  }
  unsigned long long t1=clock64();
  if(threadIdx.x==0) out[blockIdx.x]=t1-t0;
}
int main(){
  char* src; cudaMalloc(&src, 64<<20); cudaMemset(src,1,64<<20);
  unsigned long long* out; cudaMalloc(&out, 8*148);
  for(int mode: {0,1}) for(int chunk: {4096, 16384, 32768}) for(int slots: {2,6}) for(int blocks: {1,148}){
    int reps=300; int smem=256+chunk*slots; if(smem>220*1024) continue;
    cudaFuncSetAttribute(k_tma,cudaFuncAttributeMaxDynamicSharedMemorySize,smem);
    k_tma<<<blocks,256,smem>>>(src,chunk,reps,slots,mode,out); cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h,out,8,cudaMemcpyDeviceToHost);
    printf("TMA mode %d chunk %6d slots %d blocks %3d: %6.1f B/cyc/SM  %6.0f cyc/chunk %s\n",mode,chunk,slots,blocks,(double)chunk*reps/h,(double)h/reps,cudaGetErrorString(cudaGetLastError()));}
  for(int chunk: {4096,16384,32768}) for(int blocks: {1,148}){
    int reps=300; int smem=chunk*4; cudaFuncSetAttribute(k_cpa,cudaFuncAttributeMaxDynamicSharedMemorySize,smem);
    k_cpa<<<blocks,256,smem>>>(src,chunk,reps,out); cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h,out,8,cudaMemcpyDeviceToHost);
    printf("CPA chunk %6d blocks %3d: %6.1f B/cyc/SM %s\n",chunk,blocks,(double)chunk*reps/h,cudaGetErrorString(cudaGetLastError()));}
  return 0;
}
