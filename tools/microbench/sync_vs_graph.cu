// Cost of a cooperative grid.sync() vs a dependent kernel boundary in a CUDA graph (B200).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_sync(int n, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = n;
}
__global__ void k_empty(int* out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] += 1;
}
int main() {
  int* out; cudaMalloc(&out, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int threads : {256, 1024}) {
    int n = 2000; void* args[] = {&n, &out};
    cudaLaunchCooperativeKernel((void*)k_sync, sms, threads, args, 0, 0); cudaDeviceSynchronize();
    cudaEventRecord(a); cudaLaunchCooperativeKernel((void*)k_sync, sms, threads, args, 0, 0); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  grid=%d threads=%d: %.3f us per sync (%s)\n", sms, threads, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
  }
  cudaStream_t s; cudaStreamCreate(&s);
  for (int grid : {148, 1184}) {
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 100; ++i) k_empty<<<grid, 256, 0, s>>>(out);
    cudaStreamEndCapture(s, &gr); cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(a, s); for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(b, s);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph      grid=%d: %.3f us per dependent kernel\n", grid, ms * 1e3 / 2000);
  }
  return 0;
}
