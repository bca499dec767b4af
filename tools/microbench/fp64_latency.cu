#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, int n, double a, double b) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double x = out[threadIdx.x];
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);            // dependent DFMA
  unsigned long long t1 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < n; ++i) idx = (int)sm[idx] & 7;      // dependent LDS.64 + cvt
  unsigned long long t2 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  unsigned long long t3 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = __ddiv_rn(y, b);          // dependent IEEE division
  unsigned long long t4 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = z + a;                    // dependent DADD
  unsigned long long t5 = clock64();
  float fz = (float)x;
  for (int i = 0; i < n; ++i) fz = fmaf(fz, (float)a, (float)b);
  unsigned long long t6 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; }
  out[threadIdx.x] = x + idx + y + z + fz;
}
int main() {
  double* out; unsigned long long* t; cudaMalloc(&out, 8 * 1024); cudaMalloc(&t, 64); cudaMemset(out, 0, 8192);
  int n = 4096;
  for (int threads : {32, 256}) {
    k<<<1, threads, 8192>>>(out, t, n, 0.999, 1e-3); cudaDeviceSynchronize();
    unsigned long long h[6]; cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
    printf("threads %3d: DFMA %.1f  LDS-chain %.1f  syncthreads %.1f  DDIV %.1f  DADD %.1f  FFMA %.1f cycles/op\n", threads,
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n, (double)h[5] / n);
  }
  return 0;
}
