// wmpc_common.cuh — shared device view, exact-rounding helpers, reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace wmpc {

// Per-node factor state of the bound FactorCache, read through one device
// indirection so captured graphs survive rebinding.
struct NodePtrs {
  const double* e_off;  // n*nu
  const double* R;      // n*nu   sum_c -2 p_c e_off_c W
  const double* g;      // n*nt   demand_gd
  const double* shift;  // n*ns   demand Ed^T
  const double* ebar;   // n*nu   chain-local prefix of e_off (fast path; 0 off chains)
};

// Everything a kernel needs, passed by value (plain device pointers + dims).
struct DevView {
  int n, H, nt, nu, nd, ns, W, P;  // W = 2nt+nu (dual row), P = nu+nt (primal row)
  int lx;                          // row stride of state-sized arrays (nt rounded up to even)
  int ly;                          // row stride of the collapsed dual Yc = [Yx (lx) | Yu (nu)]
  int a_identity;                  // A == I exactly
  int w_scalar;                    // Wu == c I exactly
  double w_c;                      // c when w_scalar
  // tree
  const int* stage_of;  // n
  const int* anc;       // n, -1 at stage 1
  const int* cptr;      // n+1 CSR children (ascending child row)
  const int* cidx;
  const double* prob;   // n
  // model / factors
  const double* A;    // nt*nt
  const double* At;   // nt*nt (A transposed)
  const double* Bt;   // nu*nt (B transposed)
  const double* Wu;   // nu*nu
  const double* T;    // H*nu*nu
  const double* Lam;  // H*nu*nu
  const double* Mb;   // H*(nt+nu)*nu : [[B],[D_{s+1}]]
  const double* Mf;   // H*(2nu)*nu   : [[D_s^T],[-T_s]]
  const double* E;      // ns*nu
  const double* e_pinv; // nu*ns
  // node data
  const NodePtrs* np;   // device copy of the bound node state
  const double* econ;   // n*nu
  // bounds
  const double *xmin, *xmax, *xsafe, *umin, *umax, *p, *q;
  double w_x, w_s;
  // iterates
  double *Y0, *Y1, *Y2;
  double *U, *X, *Ua, *Xa;
  double *wbar, *lin;
  double* Yc;                      // collapsed extrapolated dual of the next iteration (fast path)
  const double *theta, *beta;
  int* iter;
  int* bad_nu;
  double gamma;
  const int* acct;  // subtree sharding: rows this rank accounts for in global sums (null: all)
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// numpy float semantics (NaN-propagating) — numpy/_core clip & maximum.
__device__ __forceinline__ double np_max(double a, double b) {
  return (a >= b || isnan(a)) ? a : b;
}
__device__ __forceinline__ double np_min(double a, double b) {
  return (a <= b || isnan(a)) ? a : b;
}
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
  double m = isnan(x) ? x : (x > lo ? x : lo);
  return isnan(m) ? m : (m < hi ? m : hi);
}

__device__ __forceinline__ const double* ybuf(const DevView& d, int k) {
  k %= 3;
  return k == 0 ? d.Y0 : (k == 1 ? d.Y1 : d.Y2);
}
__device__ __forceinline__ double* ybuf_w(const DevView& d, int k) {
  k %= 3;
  return k == 0 ? d.Y0 : (k == 1 ? d.Y1 : d.Y2);
}

// numpy pairwise summation (loops_utils.h pairwise_sum), serial, any n.
template <class F>
__device__ double pw_serial(const F& f, int lo, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = dadd(res, f(lo + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], f(lo + i + j));
    double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                      dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
    for (; i < n; ++i) res = dadd(res, f(lo + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return dadd(pw_serial(f, lo, n2), pw_serial(f, lo + n2, n - n2));
}

// Same sum, one warp cooperating (all 32 lanes call; result in every lane).
template <class F>
__device__ double pw_warp(const F& f, int n) {
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31;
  if (n < 8 || n > 128) {
    double res = 0.0;
    if (lane == 0) res = pw_serial(f, 0, n);
    return __shfl_sync(full, res, 0);
  }
  int nb = n - (n % 8);
  double r = 0.0;
  if (lane < 8) {
    r = f(lane);
    for (int i = 8 + lane; i < nb; i += 8) r = dadd(r, f(i));
  }
  double s = dadd(r, __shfl_down_sync(full, r, 1));
  double t = dadd(s, __shfl_down_sync(full, s, 2));
  double res = dadd(t, __shfl_down_sync(full, t, 4));
  res = __shfl_sync(full, res, 0);
  for (int i = nb; i < n; ++i) res = dadd(res, f(i));
  return res;
}

// Deterministic block reductions (fixed shuffle tree, fixed warp order).
template <int OP>  // 0 sum, 1 max
__device__ __forceinline__ double comb(double a, double b) {
  if (OP == 0) return a + b;
  return np_max(a, b);
}
template <int OP>
__device__ double block_reduce(double v, double* sh) {
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = comb<OP>(v, __shfl_down_sync(full, v, o));
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  if (wid == 0) {
    v = lane < nw ? sh[lane] : (OP == 0 ? 0.0 : -INFINITY);
    for (int o = 16; o > 0; o >>= 1) v = comb<OP>(v, __shfl_down_sync(full, v, o));
  }
  return v;  // valid in thread 0
}

}  // namespace wmpc
