#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, int n, double a, double b) {
  double x = out[threadIdx.x] + 1.5;
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x) + 1.0;
  unsigned long long t1 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = __dsqrt_rn(y) + 1.0;
  unsigned long long t2 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) { double r = __drcp_rn(b); double q = z * r; double e = fma(-q, b, z); z = fma(e, r, q) + 1.0; }
  unsigned long long t3 = clock64();
  double w = x;
  for (int i = 0; i < n; ++i) w = (double)(int)(w * 0.5) + 3.0;  // int conversions
  unsigned long long t4 = clock64();
  int q = threadIdx.x + 7;
  int dv = (int)b + 240;
  for (int i = 0; i < n; ++i) q = q / dv + 1000 + i;  // runtime int division
  unsigned long long t5 = clock64();
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
  out[threadIdx.x] = x + y + z + w + q;
}
int main() {
  double* out; unsigned long long* t; cudaMalloc(&out, 8 * 1024); cudaMalloc(&t, 64); cudaMemset(out, 0, 8192);
  int n = 2048;
  k<<<1, 32>>>(out, t, n, 0.999, 3.0); cudaDeviceSynchronize();
  unsigned long long h[5]; cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
  printf("DRCP %.1f  DSQRT %.1f  RCP+Markstein(dep on z) %.1f  cvt-chain %.1f  idiv %.1f cycles/op\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  return 0;
}
