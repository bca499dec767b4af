// wmpc_kernels.cuh — v1 kernels: stage-tiled dual gradient, fused prox/averaging,
// reductions, certificate and factor-step per-node part. General dimensions.
//
// Reference mapping (paths relative to /root/reference/pkg/src/watermpc):
//   k_bwd_stage   solver.py:261-274  backward cost-to-go (one launch per stage)
//   k_fwd_stage   solver.py:276-287  forward rollout, + solver.py:461-484 fused
//                 (extrapolation, w + gamma Hz, Moreau prox, ergodic average)
//   k_prox_rows   problem.py:290-327 / solver.py:546-583
//   k_node_*      solver.py:206-225  factor step per-node part
//   k_dyk_*       problem.py:221-250 Dykstra restoration
//   k_cost_*      problem.py:269-275, solver.py:390-395, problem.py:342-374
#pragma once
#include <climits>
#include <type_traits>
#include "wmpc_common.cuh"

namespace wmpc {

constexpr int TM = 8;        // nodes per CTA tile in the stage kernels
constexpr int NTHR = 128;

// ---------------------------------------------------------------------------
// Backward stage: for every node r of stage s (rows r0..r0+cnt):
//   wbar_r = Yx_r + (sum_c wbar_c) A          (children ascending)
//   lin_r  = Yu_r + R_r + [wbar_r | sum_c lin_c] [[B],[D_{s+1}]]
// Yx/Yu come from the extrapolated dual w = y + beta (y - y_prev) (APG) or
// directly from ysrc (plain mode).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_bwd_stage(DevView d, int s, int r0, int cnt,
                                                    const double* __restrict__ ysrc) {
  extern __shared__ double sm[];
  const int nt = d.nt, nu = d.nu, W = d.W;
  const int tile = blockIdx.x * TM;
  const int rows = min(TM, cnt - tile);
  const bool kids = s < d.H - 1;
  const int K = nt + (kids ? nu : 0);
  double* in = sm;                 // TM*K
  double* add = in + TM * K;       // TM*nu
  double* sw = add + TM * nu;      // TM*nt (child wbar sums when A != I)

  const double *yc, *yp = nullptr;
  double beta = 0.0;
  if (ysrc) {
    yc = ysrc;
  } else {
    int it = *d.iter;
    yc = ybuf(d, it);
    yp = ybuf(d, it + 2);
    beta = d.beta[it];
  }
  for (int idx = threadIdx.x; idx < rows * nt; idx += blockDim.x) {
    int m = idx / nt, j = idx - m * nt;
    int r = r0 + tile + m;
    const double* yr = yc + (size_t)r * W;
    double w1 = yr[j], w2 = yr[nt + j];
    if (yp) {
      const double* pr = yp + (size_t)r * W;
      w1 = dadd(w1, dmul(beta, dsub(w1, pr[j])));
      w2 = dadd(w2, dmul(beta, dsub(w2, pr[nt + j])));
    }
    double yx = dadd(w1, w2);
    double cs = 0.0;
    if (kids)
      for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) cs += d.wbar[(size_t)d.cidx[e] * d.lx + j];
    if (d.a_identity) {
      in[m * K + j] = yx + cs;
    } else {
      in[m * K + j] = yx;
      sw[m * nt + j] = cs;
    }
  }
  for (int idx = threadIdx.x; idx < rows * nu; idx += blockDim.x) {
    int m = idx / nu, j = idx - m * nu;
    int r = r0 + tile + m;
    double w3 = yc[(size_t)r * W + 2 * nt + j];
    if (yp) w3 = dadd(w3, dmul(beta, dsub(w3, yp[(size_t)r * W + 2 * nt + j])));
    double a = w3;
    if (kids) {
      a = w3 + d.np->R[(size_t)r * nu + j];
      double ls = 0.0;
      for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) ls += d.lin[(size_t)d.cidx[e] * nu + j];
      in[m * K + nt + j] = ls;
    }
    add[m * nu + j] = a;
  }
  __syncthreads();
  if (!d.a_identity && kids) {
    for (int idx = threadIdx.x; idx < rows * nt; idx += blockDim.x) {
      int m = idx / nt, j = idx - m * nt;
      double acc = 0.0;
      for (int k = 0; k < nt; ++k) acc = fma(sw[m * nt + k], d.A[k * nt + j], acc);
      in[m * K + j] += acc;
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < rows * nt; idx += blockDim.x) {
    int m = idx / nt, j = idx - m * nt;
    d.wbar[(size_t)(r0 + tile + m) * d.lx + j] = in[m * K + j];
  }
  const double* M = d.Mb + (size_t)s * (nt + nu) * nu;
  for (int c = threadIdx.x; c < nu; c += blockDim.x) {
    double acc[TM];
#pragma unroll
    for (int m = 0; m < TM; ++m) acc[m] = 0.0;
    for (int k = 0; k < K; ++k) {
      double b = __ldg(M + (size_t)k * nu + c);
#pragma unroll
      for (int m = 0; m < TM; ++m) acc[m] = fma(in[m * K + k], b, acc[m]);
    }
    for (int m = 0; m < rows; ++m)
      d.lin[(size_t)(r0 + tile + m) * nu + c] = add[m * nu + c] + acc[m];
  }
}

// Prox of the three slots for one node row held in shared memory.
// v: the row w + gamma Hz (conj=1) or the prox argument (conj=0).
// Writes the result row to out (global). Exact numpy expression order.
struct ProxParams {
  double gamma;  // conj: Moreau gamma; plain: prox gamma
  int conj;
};

__device__ __forceinline__ double prox_arg(const double v, const ProxParams& pp) {
  return pp.conj ? ddiv(v, pp.gamma) : v;
}

// step factors for slots 1 and 2 of a row (one warp).
__device__ void prox_steps(const DevView& d, const double* v, const ProxParams& pp,
                           double& st1, double& st2) {
  const int nt = d.nt;
  const double g = pp.conj ? ddiv(1.0, pp.gamma) : pp.gamma;
  auto f1 = [&](int j) {
    double V = prox_arg(v[j], pp);
    double df = dsub(V, np_clip(V, d.xmin[j], d.xmax[j]));
    return dmul(df, df);
  };
  auto f2 = [&](int j) {
    double V = prox_arg(v[nt + j], pp);
    double df = dsub(V, np_max(V, d.xsafe[j]));
    return dmul(df, df);
  };
  double dist1 = __dsqrt_rn(pw_warp(f1, nt));
  double dist2 = __dsqrt_rn(pw_warp(f2, nt));
  double thr1 = dmul(g, d.w_x), thr2 = dmul(g, d.w_s);
  st1 = dist1 > 0.0 ? np_min(1.0, ddiv(thr1, dist1)) : 0.0;
  st2 = dist2 > 0.0 ? np_min(1.0, ddiv(thr2, dist2)) : 0.0;
}

__device__ __forceinline__ double prox_elem(const DevView& d, int c, double v, double st1,
                                            double st2, const ProxParams& pp) {
  const int nt = d.nt;
  double V = prox_arg(v, pp);
  double O;
  if (c < nt) {
    double df = dsub(V, np_clip(V, d.xmin[c], d.xmax[c]));
    O = dsub(V, dmul(st1, df));
  } else if (c < 2 * nt) {
    double df = dsub(V, np_max(V, d.xsafe[c - nt]));
    O = dsub(V, dmul(st2, df));
  } else {
    O = np_clip(V, d.umin[c - 2 * nt], d.umax[c - 2 * nt]);
  }
  return pp.conj ? dsub(v, dmul(pp.gamma, O)) : O;
}

// ---------------------------------------------------------------------------
// Forward stage: u_r = e_off_r + [u_anc | lin_r/p_r] [[D_s^T],[-T_s]];
//                x_r = x_anc A^T + u_r B^T + g_r.
// mode 0: plain (store U, X). mode 1: APG — additionally y+ = prox_{gamma g*}(
// w + gamma (x, x, u)) with w re-extrapolated, non-finite flag, ergodic average.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_fwd_stage(DevView d, int s, int r0, int cnt, int mode) {
  extern __shared__ double sm[];
  const int nt = d.nt, nu = d.nu, W = d.W;
  const int tile = blockIdx.x * TM;
  const int rows = min(TM, cnt - tile);
  double* inF = sm;                // TM*2nu
  double* us = inF + TM * 2 * nu;  // TM*nu
  double* xa = us + TM * nu;       // TM*nt
  double* xs = xa + TM * nt;       // TM*nt
  double* vrow = xs + TM * nt;     // TM*W (mode 1)
  double* stp = vrow + TM * W;     // TM*2

  for (int idx = threadIdx.x; idx < rows * nu; idx += blockDim.x) {
    int m = idx / nu, j = idx - m * nu;
    int r = r0 + tile + m;
    int a = d.anc[r];
    inF[m * 2 * nu + j] = a < 0 ? d.q[j] : d.U[(size_t)a * nu + j];
    inF[m * 2 * nu + nu + j] = d.lin[(size_t)r * nu + j] / d.prob[r];
  }
  for (int idx = threadIdx.x; idx < rows * nt; idx += blockDim.x) {
    int m = idx / nt, j = idx - m * nt;
    int r = r0 + tile + m;
    int a = d.anc[r];
    xa[m * nt + j] = a < 0 ? d.p[j] : d.X[(size_t)a * d.lx + j];
  }
  __syncthreads();
  const double* M = d.Mf + (size_t)s * 2 * nu * nu;
  for (int c = threadIdx.x; c < nu; c += blockDim.x) {
    double acc[TM];
#pragma unroll
    for (int m = 0; m < TM; ++m) acc[m] = 0.0;
    for (int k = 0; k < 2 * nu; ++k) {
      double b = __ldg(M + (size_t)k * nu + c);
#pragma unroll
      for (int m = 0; m < TM; ++m) acc[m] = fma(inF[m * 2 * nu + k], b, acc[m]);
    }
    for (int m = 0; m < rows; ++m) {
      int r = r0 + tile + m;
      double u = d.np->e_off[(size_t)r * nu + c] + acc[m];
      us[m * nu + c] = u;
      d.U[(size_t)r * nu + c] = u;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nt; c += blockDim.x) {
    double acc[TM], acx[TM];
#pragma unroll
    for (int m = 0; m < TM; ++m) acc[m] = acx[m] = 0.0;
    for (int k = 0; k < nu; ++k) {
      double b = __ldg(d.Bt + (size_t)k * nt + c);
#pragma unroll
      for (int m = 0; m < TM; ++m) acc[m] = fma(us[m * nu + k], b, acc[m]);
    }
    if (!d.a_identity) {
      for (int k = 0; k < nt; ++k) {
        double b = __ldg(d.At + (size_t)k * nt + c);
#pragma unroll
        for (int m = 0; m < TM; ++m) acx[m] = fma(xa[m * nt + k], b, acx[m]);
      }
    }
    for (int m = 0; m < rows; ++m) {
      int r = r0 + tile + m;
      double xprev = d.a_identity ? xa[m * nt + c] : acx[m];
      double x = (xprev + acc[m]) + d.np->g[(size_t)r * d.lx + c];
      xs[m * nt + c] = x;
      d.X[(size_t)r * d.lx + c] = x;
    }
  }
  if (mode == 0) return;
  __syncthreads();

  const int it = *d.iter;
  const double* yc = ybuf(d, it);
  const double* yp = ybuf(d, it + 2);
  double* yn = ybuf_w(d, it + 1);
  const double beta = d.beta[it], theta = d.theta[it], gamma = d.gamma;
  for (int idx = threadIdx.x; idx < rows * W; idx += blockDim.x) {
    int m = idx / W, c = idx - m * W;
    int r = r0 + tile + m;
    double y0 = yc[(size_t)r * W + c];
    double w = dadd(y0, dmul(beta, dsub(y0, yp[(size_t)r * W + c])));
    double hz = c < nt ? xs[m * nt + c] : (c < 2 * nt ? xs[m * nt + c - nt] : us[m * nu + c - 2 * nt]);
    vrow[m * W + c] = dadd(w, dmul(gamma, hz));
  }
  __syncthreads();
  ProxParams pp{gamma, 1};
  const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int m = warp; m < rows; m += nwarp) {
    double s1, s2;
    prox_steps(d, vrow + m * W, pp, s1, s2);
    if ((threadIdx.x & 31) == 0) {
      stp[2 * m] = s1;
      stp[2 * m + 1] = s2;
    }
  }
  __syncthreads();
  bool bad = false;
  for (int idx = threadIdx.x; idx < rows * W; idx += blockDim.x) {
    int m = idx / W, c = idx - m * W;
    int r = r0 + tile + m;
    double out = prox_elem(d, c, vrow[m * W + c], stp[2 * m], stp[2 * m + 1], pp);
    yn[(size_t)r * W + c] = out;
    bad |= !isfinite(out);
  }
  if (bad) atomicMin(d.bad_nu, it);
  const double om = dsub(1.0, theta);
  for (int idx = threadIdx.x; idx < rows * nu; idx += blockDim.x) {
    int m = idx / nu, j = idx - m * nu;
    size_t o = (size_t)(r0 + tile + m) * nu + j;
    double u = us[m * nu + j];
    d.Ua[o] = it == 0 ? u : dadd(dmul(d.Ua[o], om), dmul(theta, u));
  }
  for (int idx = threadIdx.x; idx < rows * nt; idx += blockDim.x) {
    int m = idx / nt, j = idx - m * nt;
    size_t o = (size_t)(r0 + tile + m) * d.lx + j;
    double x = xs[m * nt + j];
    d.Xa[o] = it == 0 ? x : dadd(dmul(d.Xa[o], om), dmul(theta, x));
  }
}

__global__ void k_advance(int* iter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *iter += 1;
}

// ---------------------------------------------------------------------------
// Standalone prox (public prox_g / prox_g_conjugate). One warp per row.
// ---------------------------------------------------------------------------
__global__ void k_prox_rows(DevView d, const double* __restrict__ vin, double* __restrict__ out,
                            double gamma, int conj) {
  const int W = d.W;
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= d.n) return;
  const double* v = vin + (size_t)warp * W;
  ProxParams pp{gamma, conj};
  double s1, s2;
  prox_steps(d, v, pp, s1, s2);
  for (int c = lane; c < W; c += 32) out[(size_t)warp * W + c] = prox_elem(d, c, v[c], s1, s2, pp);
}

// ---------------------------------------------------------------------------
// Check-iteration reductions: per-block partials then a one-block finisher.
// part layout: [resid, scale, dchange] per block.
// ---------------------------------------------------------------------------
__global__ void k_check_partial(DevView d, const double* __restrict__ ynew,
                                const double* __restrict__ yold, double* part) {
  __shared__ double sh[32];
  double over = 0.0, scale = 0.0, dch = 0.0;
  const size_t nU = (size_t)d.n * d.nu, nX = (size_t)d.n * d.lx, nY = (size_t)d.n * d.W;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nU; i += (size_t)gridDim.x * blockDim.x) {
    int j = (int)(i % d.nu);
    double u = d.Ua[i];
    over = np_max(over, np_max(u - d.umax[j], 0.0));
    over = np_max(over, np_max(d.umin[j] - u, 0.0));
    scale = np_max(scale, fabs(u));
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nX; i += (size_t)gridDim.x * blockDim.x)
    scale = np_max(scale, fabs(d.Xa[i]));
  if (ynew)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nY; i += (size_t)gridDim.x * blockDim.x)
      dch = np_max(dch, fabs(ynew[i] - yold[i]));
  over = block_reduce<1>(over, sh);
  if (threadIdx.x == 0) part[3 * blockIdx.x] = over;
  scale = block_reduce<1>(scale, sh);
  if (threadIdx.x == 0) part[3 * blockIdx.x + 1] = scale;
  dch = block_reduce<1>(dch, sh);
  if (threadIdx.x == 0) part[3 * blockIdx.x + 2] = dch;
}

// Generic finisher: out[k] = OP over part[b*stride + k], b < nb.
template <int OP>
__global__ void k_finish(const double* part, int nb, int stride, int k0, int nk, double* out) {
  __shared__ double sh[32];
  for (int k = k0; k < k0 + nk; ++k) {
    double v = OP == 0 ? 0.0 : -INFINITY;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) v = comb<OP>(v, part[(size_t)b * stride + k]);
    v = block_reduce<OP>(v, sh);
    if (threadIdx.x == 0) out[k] = v;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Per-node cost terms (one warp per node), summed per block:
//   part[b*4+0] = sum p_r (c_r.u_r + du' W du)      smooth cost   (problem.py:269-275)
//   part[b*4+1] = sum Yx.x + Yu.u  (if y given)     <H'y, z>       (solver.py:289)
//   part[b*4+2] = sum ||x - clip(x)||               box distance   (solver.py:393)
//   part[b*4+3] = sum ||x - max(x, xs)||            safety distance(solver.py:394)
// ---------------------------------------------------------------------------
__global__ void k_cost_partial(DevView d, const double* __restrict__ Uin, const double* __restrict__ Xin,
                               const double* __restrict__ y, int want_pen, double* part) {
  __shared__ double sh[32];
  const int nt = d.nt, nu = d.nu, W = d.W;
  int lane = threadIdx.x & 31;
  int wpb = blockDim.x >> 5;
  double acc_cost = 0.0, acc_dot = 0.0, acc_box = 0.0, acc_safe = 0.0;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < d.n; r += gridDim.x * wpb) {
    if (d.acct && !d.acct[r]) continue;
    const double* u = Uin + (size_t)r * nu;
    int a = d.anc[r];
    const double* ua = a < 0 ? d.q : Uin + (size_t)a * nu;
    double lin = 0.0, quad = 0.0;
    for (int j = lane; j < nu; j += 32) {
      lin += d.econ[(size_t)r * nu + j] * u[j];
      double wd;
      if (d.w_scalar) {
        wd = d.w_c * (u[j] - ua[j]);
      } else {
        wd = 0.0;
        for (int k = 0; k < nu; ++k) wd = fma(d.Wu[(size_t)j * nu + k], u[k] - ua[k], wd);
      }
      quad += (u[j] - ua[j]) * wd;
    }
    double dot = 0.0;
    if (y) {
      const double* yr = y + (size_t)r * W;
      const double* x = Xin + (size_t)r * d.lx;
      for (int j = lane; j < nt; j += 32) dot += (yr[j] + yr[nt + j]) * x[j];
      for (int j = lane; j < nu; j += 32) dot += yr[2 * nt + j] * u[j];
    }
    double box = 0.0, safe = 0.0;
    if (want_pen) {
      const double* x = Xin + (size_t)r * d.lx;
      for (int j = lane; j < nt; j += 32) {
        double b = x[j] - np_clip(x[j], d.xmin[j], d.xmax[j]);
        double sf = x[j] - np_max(x[j], d.xsafe[j]);
        box += b * b;
        safe += sf * sf;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      lin += __shfl_down_sync(0xffffffffu, lin, o);
      quad += __shfl_down_sync(0xffffffffu, quad, o);
      dot += __shfl_down_sync(0xffffffffu, dot, o);
      box += __shfl_down_sync(0xffffffffu, box, o);
      safe += __shfl_down_sync(0xffffffffu, safe, o);
    }
    if (lane == 0) {
      acc_cost += d.prob[r] * (lin + quad);
      acc_dot += dot;
      acc_box += sqrt(box);
      acc_safe += sqrt(safe);
    }
  }
  double v;
  v = block_reduce<0>(acc_cost, sh);
  if (threadIdx.x == 0) part[4 * blockIdx.x] = v;
  v = block_reduce<0>(acc_dot, sh);
  if (threadIdx.x == 0) part[4 * blockIdx.x + 1] = v;
  v = block_reduce<0>(acc_box, sh);
  if (threadIdx.x == 0) part[4 * blockIdx.x + 2] = v;
  v = block_reduce<0>(acc_safe, sh);
  if (threadIdx.x == 0) part[4 * blockIdx.x + 3] = v;
}

// g*(y) (problem.py:342-374): part[b*2] = support sums, part[b*2+1] = domain
// violation flag (max).
__device__ __forceinline__ double box_support(double lo, double hi, double y) {
  double v = hi * (y > 0.0 ? y : 0.0) + lo * (y < 0.0 ? y : 0.0);
  return isnan(v) ? 0.0 : v;
}
__global__ void k_gconj_partial(DevView d, const double* __restrict__ y, double tol, double* part) {
  __shared__ double sh[32];
  const int nt = d.nt, nu = d.nu, W = d.W;
  int lane = threadIdx.x & 31;
  int wpb = blockDim.x >> 5;
  double acc = 0.0, viol = 0.0;
  const double slack = 1.0 + tol;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < d.n; r += gridDim.x * wpb) {
    if (d.acct && !d.acct[r]) continue;
    const double* yr = y + (size_t)r * W;
    double n1 = 0.0, n2 = 0.0, sup = 0.0, v = 0.0;
    for (int j = lane; j < nt; j += 32) {
      double a = yr[j], b = yr[nt + j];
      n1 += a * a;
      n2 += b * b;
      if (b > tol * (1.0 + fabs(d.xsafe[j]))) v = 1.0;
      sup += box_support(d.xmin[j], d.xmax[j], a) + d.xsafe[j] * (b < 0.0 ? b : 0.0);
    }
    for (int j = lane; j < nu; j += 32) sup += box_support(d.umin[j], d.umax[j], yr[2 * nt + j]);
    for (int o = 16; o > 0; o >>= 1) {
      n1 += __shfl_down_sync(0xffffffffu, n1, o);
      n2 += __shfl_down_sync(0xffffffffu, n2, o);
      sup += __shfl_down_sync(0xffffffffu, sup, o);
      v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    if (lane == 0) {
      if (sqrt(n1) > d.w_x * slack + tol) v = 1.0;
      if (sqrt(n2) > d.w_s * slack + tol) v = 1.0;
      acc += sup;
      viol = fmax(viol, v);
    }
  }
  double t = block_reduce<0>(acc, sh);
  if (threadIdx.x == 0) part[2 * blockIdx.x] = t;
  t = block_reduce<1>(viol, sh);
  if (threadIdx.x == 0) part[2 * blockIdx.x + 1] = t;
}

__global__ void k_absmax_partial(const double* __restrict__ a, size_t len, double* part) {
  __shared__ double sh[32];
  double m = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
    m = np_max(m, fabs(a[i]));
  m = block_reduce<1>(m, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ void k_dyk_tol(const double* part, int nb, double* tol) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v = np_max(v, part[b]);
  v = block_reduce<1>(v, sh);
  if (threadIdx.x == 0) *tol = 1e-13 * (1.0 + v);
}

__global__ void k_clip_inputs(DevView d, const double* __restrict__ src, double* dst) {
  size_t len = (size_t)d.n * d.nu;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
    int j = (int)(i % d.nu);
    dst[i] = np_clip(src[i], d.umin[j], d.umax[j]);
  }
}

// Rollout x_r = x_anc A^T + u_r B^T + g_r for one stage (problem.py:207-218).
__global__ void k_rollout_stage(DevView d, int r0, int cnt, const double* __restrict__ Uin, double* Xout) {
  const int nt = d.nt, nu = d.nu;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < cnt * nt; idx += gridDim.x * blockDim.x) {
    int m = idx / nt, j = idx - m * nt;
    int r = r0 + m;
    int a = d.anc[r];
    const double* xa = a < 0 ? d.p : Xout + (size_t)a * d.lx;
    double xp = 0.0;
    if (d.a_identity) {
      xp = xa[j];
    } else {
      for (int k = 0; k < nt; ++k) xp = fma(xa[k], d.A[(size_t)j * nt + k], xp);
    }
    double bu = 0.0;
    for (int k = 0; k < nu; ++k) bu = fma(Uin[(size_t)r * nu + k], d.Bt[(size_t)k * nt + j], bu);
    Xout[(size_t)r * d.lx + j] = (xp + bu) + d.np->g[(size_t)r * d.lx + j];
  }
}

// ---------------------------------------------------------------------------
// Factor step per-node part (solver.py:206-225), one warp per node.
// ---------------------------------------------------------------------------
__global__ void k_node_offsets(DevView d, const double* __restrict__ demand, const double* __restrict__ Ed,
                               double* shift, double* u_part, double* e_off, double* tmp, int* bad_row) {
  const int nu = d.nu, ns = d.ns, nd = d.nd;
  int lane = threadIdx.x & 31;
  int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= d.n) return;
  double* up = u_part + (size_t)r * nu;
  double* t = tmp + (size_t)r * nu;
  if (ns > 0) {
    for (int i = lane; i < ns; i += 32) {
      double s = 0.0;
      for (int k = 0; k < nd; ++k) s = fma(demand[(size_t)r * nd + k], Ed[(size_t)i * nd + k], s);
      shift[(size_t)r * ns + i] = s;
    }
    __syncwarp();
    for (int j = lane; j < nu; j += 32) {
      double s = 0.0;
      for (int i = 0; i < ns; ++i) s = fma(shift[(size_t)r * ns + i], d.e_pinv[(size_t)j * ns + i], s);
      up[j] = -s;
    }
    __syncwarp();
    bool bad = false;
    for (int i = lane; i < ns; i += 32) {
      double s = 0.0;
      for (int j = 0; j < nu; ++j) s = fma(up[j], d.E[(size_t)i * nu + j], s);
      double rhs = shift[(size_t)r * ns + i];
      if (fabs(s + rhs) > 1e-9 * (1.0 + fabs(rhs))) bad = true;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(bad_row, r);
  } else {
    for (int j = lane; j < nu; j += 32) up[j] = 0.0;
  }
  __syncwarp();
  const int s = d.stage_of[r];
  const double* L = d.Lam + (size_t)s * nu * nu;
  const double* T = d.T + (size_t)s * nu * nu;
  for (int j = lane; j < nu; j += 32) {
    double a = 0.0;
    for (int k = 0; k < nu; ++k) a = fma(up[k], L[(size_t)k * nu + j], a);
    t[j] = a + d.econ[(size_t)r * nu + j];
  }
  __syncwarp();
  for (int j = lane; j < nu; j += 32) {
    double a = 0.0;
    for (int k = 0; k < nu; ++k) a = fma(t[k], T[(size_t)k * nu + j], a);
    e_off[(size_t)r * nu + j] = up[j] - a;
  }
}

// Structured factor step (W = cI, every T_s = P/(2c), D_s = P, checked on the
// host): Lam_s = Pi_{s+1} + 2W = 2c(2I - P) (2cI at the last stage) and
// u_part = -E^+ shift lies in range(E^T), so e_off = u_part - (u_part Lam_s
// + econ) T_s reduces to u_part - P econ / (2c): no per-node dense 114x114
// products. P econ = econ - E^T (K econ) with K = (E E^T)^{-1} E sparse.
__global__ void k_node_offsets_proj(DevView d, const double* __restrict__ demand, const double* __restrict__ Ed,
                                    const int* __restrict__ kp, const int* __restrict__ kc,
                                    const double* __restrict__ kv, const int* __restrict__ ecp,
                                    const int* __restrict__ ecr, const double* __restrict__ ecv, double inv_2c,
                                    double* shift, double* u_part, double* e_off, int* bad_row) {
  __shared__ double st[8][32];
  const int nu = d.nu, ns = d.ns, nd = d.nd;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * 8 + warp;
  if (r >= d.n) return;
  double* up = u_part + (size_t)r * nu;
  const double* ec = d.econ + (size_t)r * nu;
  if (lane < ns) {
    double s = 0.0;
    for (int k = 0; k < nd; ++k) s = fma(demand[(size_t)r * nd + k], Ed[(size_t)lane * nd + k], s);
    shift[(size_t)r * ns + lane] = s;
    st[warp][lane] = s;
  }
  __syncwarp();
  for (int j = lane; j < nu; j += 32) {
    double s = 0.0;
    for (int i = 0; i < ns; ++i) s = fma(st[warp][i], d.e_pinv[(size_t)j * ns + i], s);
    up[j] = -s;
  }
  __syncwarp();
  bool bad = false;
  if (lane < ns) {  // feasibility of E u = -Ed d (solver.py:213)
    double s = 0.0;
    for (int j = 0; j < nu; ++j) s = fma(up[j], d.E[(size_t)lane * nu + j], s);
    const double rhs = st[warp][lane];
    bad = fabs(s + rhs) > 1e-9 * (1.0 + fabs(rhs));
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(bad_row, r);
  double t = 0.0;  // K econ
  if (lane < ns)
    for (int e = kp[lane]; e < kp[lane + 1]; ++e) t = fma(kv[e], ec[kc[e]], t);
  __syncwarp();
  if (lane < ns) st[warp][lane] = t;
  __syncwarp();
  for (int j = lane; j < nu; j += 32) {
    double c = 0.0;
    for (int e = ecp[j]; e < ecp[j + 1]; ++e) c = fma(ecv[e], st[warp][ecr[e]], c);
    e_off[(size_t)r * nu + j] = up[j] - (ec[j] - c) * inv_2c;
  }
}

// R_a = sum_c -2 p_c (e_off_c W), children ascending.
__global__ void k_node_R(DevView d, const double* __restrict__ e_off, double* Rout) {
  const int nu = d.nu;
  int lane = threadIdx.x & 31;
  int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= d.n) return;
  for (int j = lane; j < nu; j += 32) {
    double acc = 0.0;
    for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) {
      int c = d.cidx[e];
      double ew = 0.0;
      if (d.w_scalar) {
        ew = e_off[(size_t)c * nu + j] * d.w_c;
      } else {
        for (int k = 0; k < nu; ++k) ew = fma(e_off[(size_t)c * nu + k], d.Wu[(size_t)k * nu + j], ew);
      }
      acc += (-2.0 * d.prob[c]) * ew;
    }
    Rout[(size_t)r * nu + j] = acc;
  }
}

// Subtree sharding: R of a replicated row sums over children on several ranks.
// phase 0: this rank's accounted children into the exchange buffer;
// phase 1 (after the cross-rank sum): the full R back into the row.
__global__ void k_shard_R(DevView d, const double* __restrict__ e_off, const int* __restrict__ rep_gidx,
                          double* xbuf, int phase, double* Rout) {
  const int nu = d.nu;
  int lane = threadIdx.x & 31;
  int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= d.n || rep_gidx[r] < 0) return;
  double* xb = xbuf + (size_t)rep_gidx[r] * 256;
  for (int j = lane; j < nu; j += 32) {
    if (phase == 1) {
      Rout[(size_t)r * nu + j] = xb[j];
      continue;
    }
    double acc = 0.0;
    for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) {
      int c = d.cidx[e];
      if (!d.acct[c]) continue;
      double ew = 0.0;
      if (d.w_scalar) {
        ew = e_off[(size_t)c * nu + j] * d.w_c;
      } else {
        for (int k = 0; k < nu; ++k) ew = fma(e_off[(size_t)c * nu + k], d.Wu[(size_t)k * nu + j], ew);
      }
      acc += (-2.0 * d.prob[c]) * ew;
    }
    xb[j] = acc;
  }
}

// Chain-local prefix of e_off for the scan-form kernel: for the node at chain
// position t, sum_{t' < t} e_off[chain node t'] (sequential, top to leaf).
__global__ void k_chain_ebar(const int* __restrict__ chain_node, int nchain, int nst, int nu,
                             const double* __restrict__ e_off, double* ebar) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nchain * nu) return;
  const int ci = idx / nu, k = idx - ci * nu;
  double acc = 0.0;
  for (int t = 0; t < nst; ++t) {
    const size_t r = (size_t)chain_node[(size_t)t * nchain + ci];
    ebar[r * nu + k] = acc;
    acc = acc + e_off[r * nu + k];
  }
}

// Power iteration helpers (solver.py:348-366).
__global__ void k_op_rows(DevView d, const double* __restrict__ U0, const double* __restrict__ X0,
                          const double* __restrict__ Uv, const double* __restrict__ Xv,
                          const double* __restrict__ v, double* gv, double* part) {
  __shared__ double sh[32];
  const int nt = d.nt, nu = d.nu, W = d.W;
  double dot = 0.0, nn = 0.0;
  size_t len = (size_t)d.n * W;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / W;
    int c = (int)(i - r * W);
    double gval = c < 2 * nt ? X0[r * d.lx + (c < nt ? c : c - nt)] - Xv[r * d.lx + (c < nt ? c : c - nt)]
                             : U0[r * nu + c - 2 * nt] - Uv[r * nu + c - 2 * nt];
    gv[i] = gval;
    dot += v[i] * gval;
    nn += gval * gval;
  }
  dot = block_reduce<0>(dot, sh);
  if (threadIdx.x == 0) part[2 * blockIdx.x] = dot;
  nn = block_reduce<0>(nn, sh);
  if (threadIdx.x == 0) part[2 * blockIdx.x + 1] = nn;
}

__global__ void k_scale_into(const double* __restrict__ src, size_t len, const double* nrm2, double* dst) {
  double nrm = sqrt(*nrm2);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i] / nrm;
}

// u0 = sum_{stage 1} p_r U_r, clipped (solver.py:525-528).
// factor step: demand_gd rows (n x nt, contiguous as uploaded) into the padded
// node layout (n x lx, zero pad), and the infeasibility sentinel
__global__ void k_pad_rows(const double* __restrict__ src, int nt, double* dst, int lx, int n, int* sentinel) {
  const size_t tot = (size_t)n * lx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / lx;
    const int j = (int)(i - r * lx);
    dst[i] = j < nt ? src[r * nt + j] : 0.0;
  }
  if (sentinel && blockIdx.x == 0 && threadIdx.x == 0) *sentinel = INT_MAX;
}

__global__ void k_u0(DevView d, const double* __restrict__ Uin, int cnt1, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.nu; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < cnt1; ++r) s = fma(d.prob[r], Uin[(size_t)r * d.nu + j], s);
    out[j] = np_clip(s, d.umin[j], d.umax[j]);
  }
}

// join (U, X) rows into primal rows [u | x].
__global__ void k_join_primal(int n, int nu, int nt, int lx, const double* __restrict__ U,
                              const double* __restrict__ X, double* z) {
  const int P = nu + nt;
  size_t len = (size_t)n * P;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / P;
    int c = (int)(i - r * P);
    z[i] = c < nu ? U[r * nu + c] : X[r * lx + c - nu];
  }
}

}  // namespace wmpc

namespace wmpc {
// Dykstra feasibility restoration (problem.py:221-250), one warp per node,
// all sweeps in one launch. The reference stops every node at the first sweep
// whose global max movement is <= tol, so it runs twice: pass 1 runs all
// sweeps and atomically maxes each sweep's movement into mv[sweep] (a node at
// an exact fixed point stops contributing); pass 2 reruns each node for the
// global sweep count and writes the result. The affine projection is
// P(a) - E^+ shift_r with the sparse form P a = a - E^T (K a), K = (E E^T)^{-1} E.
struct DykOps {
  const int *kp, *kc, *ecp, *ecr;
  const double *kv, *ecv;
  // optional ELL copies (structured path): owners [.. | E cols at ec0 | K rows at kr0], stride ew
  const int* eidx;
  const double* eval;
  int ew, ec0, kr0;
  const int* freek;  // inputs in no coupling row (E column empty), nfree of them
  int nfree;
};
constexpr int DYK_MAXQ = 4;  // nu <= 128
// fix (optional): pass 1 stores its final state in u_out and, per node, the
// sweep count after which that state no longer changes (max_sweeps when it
// never settled); pass 2 then only recomputes the nodes whose pass-1 state is
// not already the state after the global sweep count.
// ELL: the operators come as the register ELL copy (po.eidx); slots past n_u
// then carry zero state and zero operator entries, so the sweep needs no
// per-slot branch (a zero slot never moves and is always "same").
#ifndef DYK_WPB
#define DYK_WPB 4  // nodes (warps) per CTA (measured: 4 beats 8 and 2 by 3-5 % at C3)
#endif
// pass 3: pass 1 for the local certificate, with the stop threshold already
// known (*tol): instead of the per-sweep maximum, each node votes whether
// any of its movements exceeds it (the same test as k_dyk_count's max <= tol,
// NaN counting as exceeding) into a per-sweep bit mask (mv as 32-bit words,
// one atomicOr per node and 32 sweeps).
template <bool ELL>
__global__ void __launch_bounds__(DYK_WPB * 32) k_dyk_warp(DevView d, DykOps po, const double* __restrict__ u_in,
                                                  double* __restrict__ u_out, unsigned long long* mv,
                                                  const int* sweeps_in, int max_sweeps, int pass, int* fix,
                                                  const double* tol) {
  __shared__ double sA[DYK_WPB][128];
  __shared__ double sT[DYK_WPB][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * DYK_WPB + warp;
  if (r >= d.n) return;
  const int nu = d.nu, ns = d.ns;
  const int nsw = pass != 2 ? max_sweeps : *sweeps_in;
  const double thr = pass == 3 ? *tol : 0.0;
  unsigned* bad_words = reinterpret_cast<unsigned*>(mv);
  unsigned wbits = 0u;
  if (pass == 2 && fix && nsw >= fix[r]) return;  // pass 1 already left the answer in u_out
  int settled = nsw;
  double cur[DYK_MAXQ], pc[DYK_MAXQ], qc[DYK_MAXQ], c[DYK_MAXQ], lo[DYK_MAXQ], hi[DYK_MAXQ];
  const double* sh = d.np->shift + (size_t)r * ns;
#pragma unroll
  for (int q = 0; q < DYK_MAXQ; ++q) {
    const int k = lane + 32 * q;
    const bool ok = k < nu;
    cur[q] = ok ? u_in[(size_t)r * nu + k] : 0.0;
    pc[q] = 0.0;
    qc[q] = 0.0;
    double e = 0.0;
    if (ok)
      for (int i = 0; i < ns; ++i) e = fma(d.e_pinv[(size_t)k * ns + i], sh[i], e);
    c[q] = e;
    lo[q] = ok ? d.umin[k] : 0.0;
    hi[q] = ok ? d.umax[k] : 0.0;
  }
  // operator entries in registers when the ELL copy is given (the water-network
  // variant: K rows <= 4 entries, E columns <= 1, zero-padded)
  constexpr int DWK = 4, DWE = 1;
  constexpr bool ell = ELL;
  int kix[DWK], eix[DYK_MAXQ][DWE];
  double kvv[DWK], evv[DYK_MAXQ][DWE];
  if (ell) {
#pragma unroll
    for (int e = 0; e < DWK; ++e) {
      const size_t o = (size_t)(po.kr0 + (lane < ns ? lane : 0)) * po.ew + e;
      kix[e] = po.eidx[o];
      kvv[e] = po.eval[o];
    }
#pragma unroll
    for (int q = 0; q < DYK_MAXQ; ++q) {
      const int k = lane + 32 * q;
#pragma unroll
      for (int e = 0; e < DWE; ++e) {
        const size_t o = (size_t)(po.ec0 + (k < nu ? k : 0)) * po.ew + e;
        eix[q][e] = k < nu ? po.eidx[o] : 0;
        evv[q][e] = k < nu ? po.eval[o] : 0.0;
      }
    }
  }
  // Fast path (warp-uniform): every input finite and below 1e150 in magnitude,
  // so no sweep can produce a NaN (bounds may be infinite) and the NaN-aware
  // clip / max reduce to plain compares with identical results.
  bool fin = true;
#pragma unroll
  for (int q = 0; q < DYK_MAXQ; ++q) fin &= fabs(cur[q]) <= 1e150 && fabs(c[q]) <= 1e150;
  if constexpr (ELL) {
#pragma unroll
    for (int e = 0; e < DWK; ++e) fin &= fabs(kvv[e]) <= 1e150;
#pragma unroll
    for (int q = 0; q < DYK_MAXQ; ++q)
#pragma unroll
      for (int e = 0; e < DWE; ++e) fin &= fabs(evv[q][e]) <= 1e150;
  }
  const bool fast = __all_sync(0xffffffffu, fin);
  // One sweep. CHECK: also test for an exact fixed point (done every 4th sweep:
  // a node detected a few sweeps late only recomputes identical sweeps).
  auto sweep = [&](int s, auto check_tag, auto fast_tag) -> bool {
    constexpr bool CHECK = decltype(check_tag)::value, FAST = decltype(fast_tag)::value;
#pragma unroll
    for (int q = 0; q < DYK_MAXQ; ++q) {
      const int k = lane + 32 * q;
      if (ELL || k < nu) sA[warp][k] = cur[q] + pc[q];
    }
    __syncwarp();
    if constexpr (ELL) {  // zero rows past n_s
      double t = 0.0;
#pragma unroll
      for (int e = 0; e < DWK; ++e) t = fma(kvv[e], sA[warp][kix[e]], t);
      sT[warp][lane] = t;
    } else if (lane < ns) {
      double t = 0.0;
      for (int e = po.kp[lane]; e < po.kp[lane + 1]; ++e) t = fma(po.kv[e], sA[warp][po.kc[e]], t);
      sT[warp][lane] = t;
    }
    __syncwarp();
    double moved = 0.0;
    bool same = true;
#pragma unroll
    for (int q = 0; q < DYK_MAXQ; ++q) {
      const int k = lane + 32 * q;
      if (ELL || k < nu) {
        double corr = 0.0;
        if constexpr (ELL) {
#pragma unroll
          for (int e = 0; e < DWE; ++e) corr = fma(evv[q][e], sT[warp][eix[q][e]], corr);
        } else {
          for (int e = po.ecp[k]; e < po.ecp[k + 1]; ++e) corr = fma(po.ecv[e], sT[warp][po.ecr[e]], corr);
        }
        const double A = sA[warp][k];
        const double a = A - (corr + c[q]);
        const double pn = A - a;  // cur + pc - aff
        const double v = a + qc[q];
        double nx;
        if constexpr (FAST) {
          const double m = v > lo[q] ? v : lo[q];
          nx = m < hi[q] ? m : hi[q];
        } else {
          nx = np_clip(v, lo[q], hi[q]);
        }
        const double qn = v - nx;
        if constexpr (FAST) moved = fmax(moved, fabs(nx - cur[q]));
        else moved = np_max(moved, fabs(nx - cur[q]));
        if constexpr (CHECK) same &= nx == cur[q] && pn == pc[q] && qn == qc[q];
        pc[q] = pn;
        qc[q] = qn;
        cur[q] = nx;
      }
    }
    if (pass == 3) {
      wbits |= (__any_sync(0xffffffffu, !(moved <= thr)) ? 1u : 0u) << (s & 31);
      if ((s & 31) == 31) {
        if (lane == 0 && wbits) atomicOr(bad_words + (s >> 5), wbits);
        wbits = 0u;
      }
    } else if (pass == 1) {
      // warp max of a nonnegative double (NaN largest, as np.max propagates it)
      // on its bit pattern: high words, then low words among the top holders
      const unsigned long long bits = (unsigned long long)__double_as_longlong(moved);
      const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(bits >> 32));
      const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(bits >> 32) == hi ? (unsigned)bits : 0u);
      const unsigned long long mb = ((unsigned long long)hi << 32) | lo;
      if (lane == 0 && mb != 0ull) atomicMax(mv + s, mb);
    }
    bool stop = false;
    if constexpr (CHECK) stop = __all_sync(0xffffffffu, same);  // every later sweep repeats it
    __syncwarp();
    return stop;
  };
  int s_end = nsw;
  for (int s = 0; s < nsw; ++s) {
    const bool chk = (s & 3) == 3;
    const bool stop = fast ? (chk ? sweep(s, std::true_type{}, std::true_type{})
                                  : sweep(s, std::false_type{}, std::true_type{}))
                           : (chk ? sweep(s, std::true_type{}, std::false_type{})
                                  : sweep(s, std::false_type{}, std::false_type{}));
    if (stop) {
      settled = s;
      s_end = s + 1;
      break;
    }
  }
  if (pass == 3 && lane == 0 && wbits) atomicOr(bad_words + ((s_end - 1) >> 5), wbits);
  if (pass != 2 && fix && lane == 0) fix[r] = settled;
  if (pass == 2 || (fix && u_out)) {
#pragma unroll
    for (int q = 0; q < DYK_MAXQ; ++q) {
      const int k = lane + 32 * q;
      if (k < nu) u_out[(size_t)r * nu + k] = cur[q];
    }
  }
}

// Dykstra with the structured operators (DykOps ELL copy: every E column has
// at most one entry, so E E^T is diagonal and the affine projection splits
// into independent blocks, one per coupling row j: the coordinates of K row j):
// one THREAD per (node, block) runs the sweeps of its <= 4 coordinates in
// registers, no shared-memory exchange; the inputs outside every block are
// box-only (a fixed point after the first sweep) and clipped by the node's
// block threads. Per element the same arithmetic as k_dyk_warp (the K-row sum over
// the row's entries in ELL order; k_dyk_warp also adds the zero padding
// slots, which can only change the sign of a zero sum). pass 3 votes into the
// per-sweep bit mask against *tol and stores each block's settled sweep in
// fix; pass 2 recomputes the blocks that had not settled by the global count.
// One (node r, coupling row j) block through nsw sweeps (k_dyk_block / k_dyk_redo).
template <int PASS>
__device__ __forceinline__ void dyk_block_run(const DevView& d, const DykOps& po, const double* __restrict__ u_in,
                                              double* __restrict__ u_out, unsigned* bad_words, int nsw,
                                              double thr, int* fix, int r, int j, int lane) {
  const int nu = d.nu, ns = d.ns;
  const long long fi = (long long)r * ns + j;
  constexpr int W = 4;
  int kk[W];
  double kv[W], ev[W], cur[W], pc[W], qc[W], c[W], lo[W], hi[W];
  int cnt = 0;
  const double* sh = d.np->shift + (size_t)r * ns;
  bool fin = true;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const size_t o = (size_t)(po.kr0 + j) * po.ew + e;
    const double v = po.eval[o];
    const int k = po.eidx[o];
    const bool ok = v != 0.0;  // zero-padded slots past the row's entries
    cnt += ok;
    kk[e] = ok ? k : 0;
    kv[e] = ok ? v : 0.0;
    ev[e] = ok ? po.eval[(size_t)(po.ec0 + k) * po.ew] : 0.0;
    cur[e] = ok ? u_in[(size_t)r * nu + k] : 0.0;
    pc[e] = qc[e] = 0.0;
    double cc = 0.0;
    if (ok)
      for (int i = 0; i < ns; ++i) cc = fma(d.e_pinv[(size_t)k * ns + i], sh[i], cc);
    c[e] = cc;
    lo[e] = ok ? d.umin[k] : 0.0;
    hi[e] = ok ? d.umax[k] : 0.0;
    fin &= fabs(cur[e]) <= 1e150 && fabs(c[e]) <= 1e150 && fabs(kv[e]) <= 1e150 && fabs(ev[e]) <= 1e150;
  }
  int settled = nsw, s_end = nsw;
  unsigned wbits = 0u;
  if (PASS == 3) {  // the node's inputs outside every block, shared over its ns block threads:
                    // clip = their state after any sweep count >= 1; movement counts in sweep 0
    double moved0 = 0.0;
    for (int i = j; i < po.nfree; i += ns) {
      const int k = po.freek[i];
      const double x0 = u_in[(size_t)r * nu + k];
      const double x1 = np_clip(x0, d.umin[k], d.umax[k]);
      u_out[(size_t)r * nu + k] = x1;
      moved0 = np_max(moved0, fabs(x1 - x0));
    }
    wbits = !(moved0 <= thr) ? 1u : 0u;
  }
  // one sweep; CHECK: the exact fixed-point test (every 4th sweep, as k_dyk_warp)
  auto sweep = [&](int s, auto check_tag) -> bool {
    constexpr bool CHECK = decltype(check_tag)::value;
    double A[W], t = 0.0;
#pragma unroll
    for (int e = 0; e < W; ++e) A[e] = cur[e] + pc[e];
#pragma unroll
    for (int e = 0; e < W; ++e)
      if (e < cnt) t = fma(kv[e], A[e], t);
    double moved = 0.0;
    bool same = true;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      if (e >= cnt) continue;
      const double corr = fma(ev[e], t, 0.0);
      const double a = A[e] - (corr + c[e]);
      const double pn = A[e] - a;
      const double v = a + qc[e];
      double nx;
      if (fin) {
        const double m = v > lo[e] ? v : lo[e];
        nx = m < hi[e] ? m : hi[e];
        if (PASS == 3) moved = fmax(moved, fabs(nx - cur[e]));
      } else {
        nx = np_clip(v, lo[e], hi[e]);
        if (PASS == 3) moved = np_max(moved, fabs(nx - cur[e]));
      }
      const double qn = v - nx;
      if (CHECK) same &= nx == cur[e] && pn == pc[e] && qn == qc[e];
      pc[e] = pn;
      qc[e] = qn;
      cur[e] = nx;
    }
    if (PASS == 3) {  // own votes; OR-reduced over whichever lanes arrive together (a union either way)
      wbits |= (!(moved <= thr) ? 1u : 0u) << (s & 31);
      if ((s & 31) == 31) {
        const unsigned am = __activemask();
        const unsigned wv = __reduce_or_sync(am, wbits);
        if (lane == __ffs(am) - 1 && wv) atomicOr(bad_words + (s >> 5), wv);
        wbits = 0u;
      }
    }
    return CHECK && same;  // every later sweep repeats it
  };
  for (int s = 0; s < nsw; ++s) {
    if (((s & 3) == 3 ? sweep(s, std::true_type{}) : sweep(s, std::false_type{}))) {
      settled = s;
      s_end = s + 1;
      break;
    }
  }
  if (PASS == 3) {
    const unsigned am = __activemask();  // threads leaving here together: one of them flushes
    const unsigned wv = __reduce_or_sync(am, wbits);
    if (lane == __ffs(am) - 1 && wv) atomicOr(bad_words + ((s_end - 1) >> 5), wv);
    fix[fi] = settled;
  }
#pragma unroll
  for (int e = 0; e < W; ++e)
    if (e < cnt) u_out[(size_t)r * nu + kk[e]] = cur[e];
}

#ifndef DYK_MINB
#define DYK_MINB 3  // 80 registers, 24 warps per SM (measured: C3 certificate 0.45-0.47 vs 0.47-0.55 ms at 1, C4 2.2 vs 2.4-3.3)
#endif
template <int PASS>
__global__ void __launch_bounds__(256, DYK_MINB) k_dyk_block(DevView d, DykOps po, const double* __restrict__ u_in,
                                                   double* __restrict__ u_out, unsigned* bad_words,
                                                   const int* sweeps_in, int max_sweeps, int* fix,
                                                   const double* tol) {
  const int nu = d.nu, ns = d.ns;
  // warp w takes coupling row j = w % ns of 32 consecutive nodes (warp-uniform
  // operator entries and slot counts); each block thread also clips its share
  // of the node's inputs outside every block
  const long long nb = (long long)((d.n + 31) / 32) * 32 * ns;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int nsw = PASS == 3 ? max_sweeps : *sweeps_in;
  const double thr = PASS == 3 ? *tol : 0.0;
  if (tid >= nb) return;
  const long long w = tid >> 5;
  const int j = (int)(w % ns), r = (int)((w / ns) * 32 + lane);
  if (r >= d.n) return;
  dyk_block_run<PASS>(d, po, u_in, u_out, bad_words, nsw, thr, fix, r, j, lane);
}

// Pass 2 over the compacted blocks that had not settled by the global count.
__global__ void __launch_bounds__(256) k_dyk_redo(DevView d, DykOps po, const double* __restrict__ u_in,
                                                  double* __restrict__ u_out, const int* sweeps_in,
                                                  const int* list, const int* count) {
  const int nsw = *sweeps_in, cnt = *count, ns = d.ns;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int fi = list[t];
    dyk_block_run<2>(d, po, u_in, u_out, nullptr, nsw, 0.0, nullptr, fi / ns, fi % ns, threadIdx.x & 31);
  }
}

// The blocks pass 2 must recompute: settled after the global count (or never).
__global__ void k_dyk_compact(const int* fix, long long nblk, const int* sweeps_in, int* list, int* count) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool need = i < nblk && *sweeps_in < fix[i];
  const unsigned m = __ballot_sync(0xffffffffu, need);
  int base = 0;
  const int lane = threadIdx.x & 31;
  if (lane == 0 && m) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (need) list[base + __popc(m & ((1u << lane) - 1u))] = (int)i;
}

// Global sweep count from pass 3's bit mask: first sweep no node voted for.
__global__ void k_dyk_count_bits(const unsigned* bad, int max_sweeps, int* sweeps) {
  __shared__ int smin[32];
  int best = max_sweeps;
  for (int s = threadIdx.x; s < max_sweeps; s += blockDim.x)
    if (!((bad[s >> 5] >> (s & 31)) & 1u)) best = min(best, s + 1);
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = min(best, smin[w]);
    *sweeps = best;
  }
}

// Global sweep count: first sweep whose max movement is <= tol (or all);
// one thread per sweep, min-reduced.
__global__ void k_dyk_count(const unsigned long long* mv, int max_sweeps, const double* tol, int* sweeps) {
  __shared__ int smin[32];
  int best = max_sweeps;
  const double tl = *tol;
  for (int s = threadIdx.x; s < max_sweeps; s += blockDim.x)
    if (__longlong_as_double((long long)mv[s]) <= tl) best = min(best, s + 1);
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = min(best, smin[w]);
    *sweeps = best;
  }
}
}  // namespace wmpc
