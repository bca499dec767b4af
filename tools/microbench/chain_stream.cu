// Access-pattern microbenchmark for the warp-per-chain down pass (C4 shape):
// per row a warp reads three row segments (912, 912, 512 B) and writes two
// (912, 512 B), one row ahead in registers, for 4096 chains x 24 rows.
// Layout 0: stage-major rows (row = t * nchain + chain, as the solver);
// layout 1: chain-major rows (row = chain * nrow + t).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_stream chain_stream.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NU = 114, NX = 64;

template <int LAYOUT>
__global__ void __launch_bounds__(128) k_stream(const double* __restrict__ L, const double* __restrict__ B,
                                                const double* __restrict__ G, double* U, double* X, int nchain,
                                                int nrow) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * 4 + warp;
  if (ci >= nchain) return;
  const int l2 = 2 * lane;
  const bool ok1 = 64 + l2 < NU;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0, ax0 = 0, ax1 = 0;
  auto row_of = [&](int t) -> size_t { return LAYOUT == 0 ? (size_t)t * nchain + ci : (size_t)ci * nrow + t; };
  double2 l0, l1, b0, b1, g;
  auto load = [&](int t) {
    const size_t r = row_of(t);
    l0 = __ldg(reinterpret_cast<const double2*>(L + r * NU + l2));
    l1 = ok1 ? __ldg(reinterpret_cast<const double2*>(L + r * NU + 64 + l2)) : make_double2(0, 0);
    b0 = __ldg(reinterpret_cast<const double2*>(B + r * NU + l2));
    b1 = ok1 ? __ldg(reinterpret_cast<const double2*>(B + r * NU + 64 + l2)) : make_double2(0, 0);
    g = __ldg(reinterpret_cast<const double2*>(G + r * NX + l2));
  };
  load(0);
  for (int t = 0; t < nrow; ++t) {
    double2 cl0 = l0, cl1 = l1, cb0 = b0, cb1 = b1, cg = g;
    if (t + 1 < nrow) load(t + 1);
    acc0 += cl0.x; acc1 += cl0.y; acc2 += cl1.x; acc3 += cl1.y;
    const size_t r = row_of(t);
    *reinterpret_cast<double2*>(U + r * NU + l2) = make_double2(cb0.x - acc0, cb0.y - acc1);
    if (ok1) *reinterpret_cast<double2*>(U + r * NU + 64 + l2) = make_double2(cb1.x - acc2, cb1.y - acc3);
    ax0 += cg.x + acc0; ax1 += cg.y + acc1;
    *reinterpret_cast<double2*>(X + r * NX + l2) = make_double2(ax0, ax1);
  }
}

int main() {
  const int nchain = 4096, nrow = 24;
  const size_t rows = (size_t)nchain * nrow;
  double *L, *B, *G, *U, *X;
  cudaMalloc(&L, rows * NU * 8); cudaMalloc(&B, rows * NU * 8); cudaMalloc(&G, rows * NX * 8);
  cudaMalloc(&U, rows * NU * 8); cudaMalloc(&X, rows * NX * 8);
  cudaMemset(L, 0, rows * NU * 8); cudaMemset(B, 0, rows * NU * 8); cudaMemset(G, 0, rows * NX * 8);
  double* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = (double)rows * (2 * NU * 8 + NX * 8) + (double)rows * (NU * 8 + NX * 8);
  for (int layout = 0; layout < 2; ++layout) {
    float best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(e0);
      if (layout == 0) k_stream<0><<<(nchain + 3) / 4, 128>>>(L, B, G, U, X, nchain, nrow);
      else k_stream<1><<<(nchain + 3) / 4, 128>>>(L, B, G, U, X, nchain, nrow);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("layout %s: %.1f us, %.0f GB/s\n", layout == 0 ? "stage-major" : "chain-major", best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
