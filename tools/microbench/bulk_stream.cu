// bulk_stream.cu — memory-stream model of the fused chain kernel (k_chain_dp):
// every warp walks whole chains bottom-up (stage-major rows: row = t*nchain + c),
// and per row reads 7 row segments (L, ut, g, y, y_prev, Ua, Xa = 7,600 B) and
// writes 4 (L, y_next, Ua, Xa = 4,256 B). Row segments reach shared memory
// either through a per-warp TMA bulk ring (cp.async.bulk + mbarrier, D stages,
// one elected lane issues) or as direct 16-byte loads one row ahead into
// registers. Reports achieved DRAM GB/s (loads + stores) at C4's shape
// (4,096 chains x 19 rows), for several warps-per-SM / ring depths. This is the
// ceiling the fused kernel can reach; it replaces tma_bulk_vs_cpasync.cu, whose
// ring kept only one copy outstanding.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_stream bulk_stream.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NSEG = 7;
__constant__ int c_seg_dbl[NSEG] = {114, 114, 64, 240, 240, 114, 64};  // row width in doubles
__constant__ int c_seg_off[NSEG] = {0, 114, 228, 292, 532, 772, 886};  // offset in the stage
constexpr int STAGE_DBL = 950;

struct Arrays {
  double* a[NSEG];
  double* yn;
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int D>
__global__ void k_bulk(Arrays A, int nchain, int nst, int cpw, int nw_total, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp * D;
  double* ring = reinterpret_cast<double*>(sm + (8 * D * wpc + 15) / 16 * 16 + 128) + (size_t)warp * D * STAGE_DBL;
  if (lane == 0) {
    for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int gw = blockIdx.x * wpc + warp;
  const int steps = cpw * nst;
  auto row_of = [&](int i) -> long long {
    const int c = gw + (i / nst) * nw_total;
    const int t = nst - 1 - (i % nst);
    return c < nchain ? (long long)t * nchain + c : -1;
  };
  auto issue = [&](int i) {
    if (lane != 0 || i >= steps) return;
    const long long r = row_of(i);
    if (r < 0) return;
    const int s = i % D;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar + s)), "r"(STAGE_DBL * 8)
                 : "memory");
    for (int k = 0; k < NSEG; ++k) {
      const double* src = A.a[k] + r * c_seg_dbl[k];
      double* dst = ring + s * STAGE_DBL + c_seg_off[k];
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(dst)),
                   "l"(src), "r"(c_seg_dbl[k] * 8), "r"(sa(bar + s))
                   : "memory");
    }
  };
  for (int i = 0; i < D; ++i) issue(i);
  double acc = 0.0;
  for (int i = 0; i < steps; ++i) {
    const long long r = row_of(i);
    if (r < 0) break;
    const int s = i % D;
    const uint32_t par = (i / D) & 1;
    asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(
                     sa(bar + s)),
                 "r"(par)
                 : "memory");
    const double* st = ring + s * STAGE_DBL;
    double v[NSEG][4];
#pragma unroll
    for (int k = 0; k < NSEG; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = lane + 32 * q;
        v[k][q] = e < c_seg_dbl[k] ? st[c_seg_off[k] + e] : 0.0;
      }
    __syncwarp();
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(i + D);
    // outputs: L (in place), y_next, Ua, Xa (in place)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = lane + 32 * q;
      if (e < 114) A.a[0][r * 114 + e] = v[0][q] + v[1][q];
      if (e < 114) A.a[5][r * 114 + e] = v[5][q] * 0.5 + v[6][q & 1];
      if (e < 64) A.a[6][r * 64 + e] = v[6][q] + v[2][q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane + 32 * q;
      if (e < 240) A.yn[r * 240 + e] = (q < 4 ? v[3][q] : v[4][q - 4]) * 0.99;
    }
    acc += v[3][0];
  }
  if (acc == 12345.678) sink[gw] = acc;
}

// direct loads one row ahead (registers), same stores
__global__ void k_direct(Arrays A, int nchain, int nst, int cpw, int nw_total, double* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  const int steps = cpw * nst;
  auto row_of = [&](int i) -> long long {
    const int c = gw + (i / nst) * nw_total;
    const int t = nst - 1 - (i % nst);
    return c < nchain ? (long long)t * nchain + c : -1;
  };
  double nx[NSEG][4];
  auto load = [&](double (&v)[NSEG][4], long long r) {
#pragma unroll
    for (int k = 0; k < NSEG; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = lane + 32 * q;
        v[k][q] = (r >= 0 && e < c_seg_dbl[k]) ? __ldcg(A.a[k] + r * c_seg_dbl[k] + e) : 0.0;
      }
  };
  load(nx, row_of(0));
  double acc = 0.0;
  for (int i = 0; i < steps; ++i) {
    const long long r = row_of(i);
    if (r < 0) break;
    double v[NSEG][4];
#pragma unroll
    for (int k = 0; k < NSEG; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[k][q] = nx[k][q];
    load(nx, i + 1 < steps ? row_of(i + 1) : -1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = lane + 32 * q;
      if (e < 114) A.a[0][r * 114 + e] = v[0][q] + v[1][q];
      if (e < 114) A.a[5][r * 114 + e] = v[5][q] * 0.5 + v[6][q & 1];
      if (e < 64) A.a[6][r * 64 + e] = v[6][q] + v[2][q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = lane + 32 * q;
      if (e < 240) A.yn[r * 240 + e] = (q < 4 ? v[3][q] : v[4][q - 4]) * 0.99;
    }
    acc += v[3][0];
  }
  if (acc == 12345.678) sink[gw] = acc;
}

int main() {
  const int nchain = 4096, nst = 19;
  const long long rows = (long long)nchain * nst;
  int hseg[NSEG] = {114, 114, 64, 240, 240, 114, 64};
  Arrays A;
  for (int k = 0; k < NSEG; ++k) {
    cudaMalloc(&A.a[k], rows * hseg[k] * 8);
    cudaMemset(A.a[k], 0, rows * hseg[k] * 8);
  }
  cudaMalloc(&A.yn, rows * 240 * 8);
  char* flush;
  const size_t fl = 512ull << 20;
  cudaMalloc(&flush, fl);
  double* sink;
  cudaMalloc(&sink, 1 << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)rows * (950 + 114 + 240 + 114 + 64) * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("rows %lld, bytes per pass %.1f MB (read 7600 B + write 4256 B per row)\n", rows, bytes / 1e6);
  for (int mode = 0; mode < 4; ++mode)
    for (int wps : {4, 7, 8, 12, 14, 16}) {
      const int D = mode == 0 ? 2 : (mode == 1 ? 3 : 4);
      const bool direct = mode == 3;
      int cpw = (nchain + sms * wps - 1) / (sms * wps);
      int nw = (nchain + cpw - 1) / cpw;
      int wpc = wps;
      int grid = (nw + wpc - 1) / wpc;
      nw = grid * wpc;
      size_t smem = direct ? 0 : (8 * D * wpc + 15) / 16 * 16 + 128 + (size_t)wpc * D * STAGE_DBL * 8;
      if (smem > 227 * 1024) continue;
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(flush, rep, fl);
        cudaEventRecord(e0);
        if (direct) k_direct<<<grid, wpc * 32>>>(A, nchain, nst, cpw, nw, sink);
        else if (D == 2) {
          cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          k_bulk<2><<<grid, wpc * 32, smem>>>(A, nchain, nst, cpw, nw, sink);
        } else if (D == 3) {
          cudaFuncSetAttribute(k_bulk<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          k_bulk<3><<<grid, wpc * 32, smem>>>(A, nchain, nst, cpw, nw, sink);
        } else {
          cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          k_bulk<4><<<grid, wpc * 32, smem>>>(A, nchain, nst, cpw, nw, sink);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("%s D=%d warps/SM %2d chains/warp %d grid %4d: %8.1f us  %7.1f GB/s  %s\n", direct ? "direct" : "bulk  ",
             direct ? 1 : D, wps, cpw, grid, best * 1e3, bytes / (best * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
