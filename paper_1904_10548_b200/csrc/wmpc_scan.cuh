// wmpc_scan.cuh — scan-form APG iteration as a CUDA graph of small kernels
// (structured case: A = I, W_u = c I, every stage factor = the null(E)
// projector P; see wmpc_fast.cuh for the derivation).
//
// The Riccati-type recursion over the tree collapses to scans because P is
// idempotent (P(a + P b) = P(a + b)):
//   wbar_r = sum_{sub(r)} Yx,     a_r = (Yu_r + wbar_r B) + R_r,
//   lin_r  = a_r + P sum_{desc(r)} a,           L_r = lin_r / (2c p_r),
//   u_r    = e_off_r + P(q + Ebar_r - sum_{path(r)} L),
//   x_r    = (x_anc + u_r B^T) + g_r.
// One APG iteration (solver.py:460-506) is six graph nodes:
//   k_chain_up    one CTA per chain: suffix scans, projector   -> L, chain totals
//   k_branch_up   one CTA per branching node: depth-weighted sums over its
//                 subtree (chain totals stand in for whole chains) -> L
//   k_branch_u    one CTA per branching node: walk-up sum of L, projector -> U, B u + g
//   k_chain_down  one CTA per chain: prefix scans, projector   -> U, X
//   k_prox_nodes  node-parallel Moreau prox, averages, next collapsed dual
//   k_advance     iteration counter
// Graph edges replace grid barriers (measured 0.7 us per dependent kernel
// vs 1.25 us per cooperative grid.sync on B200).
#pragma once
#include "wmpc_fast.cuh"

namespace wmpc {

constexpr int SC_THREADS = 256;
constexpr int SC_NPB = 4;  // nodes per CTA in k_prox_nodes

// E^+ (transposed), E rows, B both ways, into shared memory; returns the Ops view.
__device__ Ops load_ops(const FastView& f, double* sp) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, ns = d.ns, bnnz = f.b_nnz;
  double* s_bnd = sp;             sp += 3 * nt + 2 * nu;
  double* s_ept = sp;             sp += nu * ns;
  double* s_ev = sp;              sp += f.e_nnz;
  double* s_bcv = sp;             sp += bnnz;
  double* s_brv = sp;             sp += bnnz;
  int* ip = reinterpret_cast<int*>(sp);
  int* s_eptr = ip;               ip += ns + 1;
  int* s_ecol = ip;               ip += f.e_nnz;
  int* s_bcp = ip;                ip += nu + 1;
  int* s_bcr = ip;                ip += bnnz;
  int* s_brp = ip;                ip += nt + 1;
  int* s_brc = ip;
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    s_bnd[i] = d.xmin[i];
    s_bnd[nt + i] = d.xmax[i];
    s_bnd[2 * nt + i] = d.xsafe[i];
  }
  for (int i = threadIdx.x; i < nu; i += blockDim.x) {
    s_bnd[3 * nt + i] = d.umin[i];
    s_bnd[3 * nt + nu + i] = d.umax[i];
  }
  for (int i = threadIdx.x; i < nu * ns; i += blockDim.x) {
    int j = i / ns, k = i - j * ns;
    s_ept[k * nu + j] = d.e_pinv[i];
  }
  for (int i = threadIdx.x; i < f.e_nnz; i += blockDim.x) {
    s_ev[i] = f.e_val[i];
    s_ecol[i] = f.e_col[i];
  }
  for (int i = threadIdx.x; i <= ns; i += blockDim.x) s_eptr[i] = f.e_ptr[i];
  for (int i = threadIdx.x; i < bnnz; i += blockDim.x) {
    s_bcv[i] = f.bc_val[i];
    s_bcr[i] = f.bc_row[i];
    s_brv[i] = f.br_val[i];
    s_brc[i] = f.br_col[i];
  }
  for (int i = threadIdx.x; i <= nu; i += blockDim.x) s_bcp[i] = f.bc_ptr[i];
  for (int i = threadIdx.x; i <= nt; i += blockDim.x) s_brp[i] = f.br_ptr[i];
  return Ops{s_ept, s_eptr, s_ecol, s_ev, s_bcp, s_bcr, s_bcv, s_brp, s_brc, s_brv,
             s_bnd, s_bnd + nt, s_bnd + 2 * nt, s_bnd + 3 * nt, s_bnd + 3 * nt + nu};
}
__host__ __device__ inline size_t ops_bytes(int nt, int nu, int ns, int enz, int bnz) {
  return sizeof(double) * ((size_t)3 * nt + 2 * nu + (size_t)nu * ns + enz + 2 * (size_t)bnz) +
         sizeof(int) * ((size_t)ns + 1 + enz + nu + 1 + bnz + nt + 1 + bnz) + 16;
}

// out[m] = P in[m] for m < rows (stride nu); T scratch rows x FAST_MAXNS. 2 barriers.
__device__ __forceinline__ void proj_rows(const DevView& d, const Ops& op, const double* in, double* out,
                                          double* T, int rows) {
  const int nu = d.nu, ns = d.ns;
  FOR_RC(rows, 5, ns, m, i) {
    double v = 0.0;
    for (int e = op.eptr[i]; e < op.eptr[i + 1]; ++e) v = fma(op.eval[e], in[m * nu + op.ecol[e]], v);
    T[m * FAST_MAXNS + i] = v;
  }
  __syncthreads();
  FOR_NU(rows, m, k) {
    const double* tm = T + m * FAST_MAXNS;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
    for (; i + 3 < ns; i += 4) {
      a0 = fma(op.ep[i * nu + k], tm[i], a0);
      a1 = fma(op.ep[(i + 1) * nu + k], tm[i + 1], a1);
      a2 = fma(op.ep[(i + 2) * nu + k], tm[i + 2], a2);
      a3 = fma(op.ep[(i + 3) * nu + k], tm[i + 3], a3);
    }
    for (; i < ns; ++i) a0 = fma(op.ep[i * nu + k], tm[i], a0);
    out[m * nu + k] = in[m * nu + k] - ((a0 + a1) + (a2 + a3));
  }
  __syncthreads();
}

// ---------------------------------------------------------------- k_chain_up
__global__ void __launch_bounds__(SC_THREADS) k_chain_up(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly;
  const int nst = d.H - f.kstar, ci = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int ra = ly + nu;                                   // [Yx | Yu | R]
  double* rec = reinterpret_cast<double*>(smem_raw);        // nst * ra
  double* WB = rec + (size_t)nst * ra;                      // nst * lx
  double* S = WB + (size_t)nst * lx;                        // nst * nu (projected in place)
  double* T = S + (size_t)nst * nu;                         // nst * FAST_MAXNS
  int* rows = reinterpret_cast<int*>(T + (size_t)nst * FAST_MAXNS);
  double* opsp = reinterpret_cast<double*>(rows + ((nst + 3) & ~3));
  const NodePtrs np = *d.np;
  if (threadIdx.x < nst) rows[threadIdx.x] = f.chain_node[(size_t)threadIdx.x * f.nchain + ci];
  __syncthreads();
  FOR_RC(nst, 7, (ly >> 1), t, k) cp16(rec + (size_t)t * ra + 2 * k, d.Yc + (size_t)rows[t] * ly + 2 * k);
  FOR_RC(nst - 1, 6, (nu >> 1), t, k) cp16(rec + (size_t)t * ra + ly + 2 * k, np.R + (size_t)rows[t] * nu + 2 * k);
  cp_commit();
  const Ops op = load_ops(f, opsp);
  cp_wait<0>();
  __syncthreads();
  if (threadIdx.x < nt) {  // wbar suffix scan: wbar_t = Yx_t + wbar_{t+1}
    const int j = threadIdx.x;
    double acc = 0.0;
    for (int t = nst - 1; t >= 0; --t) {
      const double yx = rec[(size_t)t * ra + j];
      acc = t == nst - 1 ? yx : yx + acc;
      WB[t * lx + j] = acc;
    }
    d.wbar[(size_t)rows[0] * lx + j] = acc;
  }
  __syncthreads();
  FOR_NU(nst, t, k) {  // a = (Yu + wbar B) + R over Yu
    double* R = rec + (size_t)t * ra;
    double bw = 0.0;
    for (int e = op.bcp[k]; e < op.bcp[k + 1]; ++e) bw = fma(WB[t * lx + op.bcr[e]], op.bcv[e], bw);
    double a = R[lx + k] + bw;
    if (t < nst - 1) a = a + R[ly + k];
    R[lx + k] = a;
  }
  __syncthreads();
  if (threadIdx.x < nu) {  // S_t = A_{t+1}, A_t = a_t + S_t
    const int k = threadIdx.x;
    double acc = 0.0;
    for (int t = nst - 1; t >= 0; --t) {
      S[t * nu + k] = acc;
      const double a = rec[(size_t)t * ra + lx + k];
      acc = t == nst - 1 ? a : a + acc;
    }
    f.Atop[(size_t)ci * nu + k] = acc;
  }
  __syncthreads();
  proj_rows(d, op, S, S, T, nst - 1);
  FOR_NU(nst, t, k) {
    const double a = rec[(size_t)t * ra + lx + k];
    const double l = t < nst - 1 ? a + S[t * nu + k] : a;
    f.Lb[(size_t)rows[t] * nu + k] = l * f.aux[(size_t)rows[t] * 2];
  }
}

// ---------------------------------------------------------------- k_branch_up
// One CTA per branching node r: depth-weighted sums over its subtree.
//   W1 = wbar_r = Yx_r + sum_{e in desc_B} Yx_e + sum_{tops} wbar_t
//   W2 = sum_{d in desc_B(r)} wbar_d = sum_e w_e Yx_e + sum_t w_t wbar_t
//   Su = sum_e (Yu_e + R_e) + sum_t Atop_t
//   a_r = (Yu_r + W1 B) + R_r,  S_r = Su + W2 B,  lin_r = a_r + P S_r.
__global__ void __launch_bounds__(SC_THREADS) k_branch_up(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly;
  const int r = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* part = reinterpret_cast<double*>(smem_raw);  // 4 * (2 lx + nu) partials
  const int pw = 2 * lx + nu;
  double* W1 = part + 4 * pw;   // lx
  double* W2 = W1 + lx;         // lx
  double* Sv = W2 + lx;         // nu
  double* av = Sv + nu;         // nu
  double* PS = av + nu;         // nu
  double* T = PS + nu;          // FAST_MAXNS
  double* opsp = T + FAST_MAXNS;
  const NodePtrs np = *d.np;
  const Ops op = load_ops(f, opsp);
  const int grp = threadIdx.x >> 6, c = threadIdx.x & 63;  // 4 groups x 64 lanes
  const int e0 = f.bd_ptr[r], e1 = f.bd_ptr[r + 1], t0 = f.bt_ptr[r], t1 = f.bt_ptr[r + 1];
  // Yx part (c < nt)
  if (c < nt) {
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
    for (int e = e0 + grp; e < e1; e += 4) {
      const double v = d.Yc[(size_t)f.bd_idx[e] * ly + c];
      s1 += v;
      s2 = fma((double)f.bd_w[e], v, s2);
    }
    for (int e = t0 + grp; e < t1; e += 4) {
      const int tr = f.chain_node[f.bt_idx[e]];  // chain top row (stage kstar, t = 0)
      const double v = d.wbar[(size_t)tr * lx + c];
      s1 += v;
      s2 = fma((double)f.bt_w[e], v, s2);
    }
    part[grp * pw + c] = s1;
    part[grp * pw + lx + c] = s2;
  }
  // Yu + R part (two passes of 64 lanes over nu <= 128)
  for (int k = c; k < nu; k += 64) {
    double s = 0.0;
    for (int e = e0 + grp; e < e1; e += 4) {
      const size_t er = (size_t)f.bd_idx[e];
      s += d.Yc[er * ly + lx + k] + np.R[er * nu + k];
    }
    for (int e = t0 + grp; e < t1; e += 4) s += f.Atop[(size_t)f.bt_idx[e] * nu + k];
    part[grp * pw + 2 * lx + k] = s;
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    const int j = threadIdx.x;
    const double* yc = d.Yc + (size_t)r * ly;
    W1[j] = yc[j] + (((part[j] + part[pw + j]) + part[2 * pw + j]) + part[3 * pw + j]);
    W2[j] = ((part[lx + j] + part[pw + lx + j]) + part[2 * pw + lx + j]) + part[3 * pw + lx + j];
  }
  __syncthreads();
  if (threadIdx.x < nu) {
    const int k = threadIdx.x;
    const double su = ((part[2 * lx + k] + part[pw + 2 * lx + k]) + part[2 * pw + 2 * lx + k]) +
                      part[3 * pw + 2 * lx + k];
    double b1 = 0.0, b2 = 0.0;
    for (int e = op.bcp[k]; e < op.bcp[k + 1]; ++e) {
      b1 = fma(W1[op.bcr[e]], op.bcv[e], b1);
      b2 = fma(W2[op.bcr[e]], op.bcv[e], b2);
    }
    av[k] = (d.Yc[(size_t)r * ly + lx + k] + b1) + np.R[(size_t)r * nu + k];
    Sv[k] = su + b2;
  }
  __syncthreads();
  proj_rows(d, op, Sv, PS, T, 1);
  if (threadIdx.x < nu) {
    const int k = threadIdx.x;
    f.Lb[(size_t)r * nu + k] = (av[k] + PS[k]) * f.aux[(size_t)r * 2];
  }
}

// ---------------------------------------------------------------- k_branch_u
// One CTA per branching node: u_r = e_off_r + P(q + Ebar_r - sum_{path} L), delta = B u + g.
__global__ void __launch_bounds__(SC_THREADS) k_branch_u(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx;
  const int r = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* z = reinterpret_cast<double*>(smem_raw);  // nu
  double* pz = z + nu;                               // nu
  double* T = pz + nu;                               // FAST_MAXNS
  double* opsp = T + FAST_MAXNS;
  const NodePtrs np = *d.np;
  const Ops op = load_ops(f, opsp);
  if (threadIdx.x < nu) {
    const int k = threadIdx.x;
    double ls = 0.0;  // sum over the path, root side first
    int path[32];
    int depth = 0;
    for (int a = r; a >= 0 && depth < 32; a = d.anc[a]) path[depth++] = a;
    for (int i = depth - 1; i >= 0; --i) ls = ls + f.Lb[(size_t)path[i] * nu + k];
    z[k] = (d.q[k] + np.ebar[(size_t)r * nu + k]) - ls;
  }
  __syncthreads();
  proj_rows(d, op, z, pz, T, 1);
  if (threadIdx.x < nu) {
    const int k = threadIdx.x;
    const double u = np.e_off[(size_t)r * nu + k] + pz[k];
    pz[k] = u;
    d.U[(size_t)r * nu + k] = u;
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    const int j = threadIdx.x;
    double bu = 0.0;
    for (int e = op.brp[j]; e < op.brp[j + 1]; ++e) bu = fma(pz[op.brc[e]], op.brv[e], bu);
    f.delta[(size_t)r * lx + j] = bu;  // B u; g added by the x walk-up
  }
}

// x of a branching row by the walk-up sum x = (x_anc + B u) + g (reference association).
__device__ __forceinline__ double branch_x(const FastView& f, const NodePtrs& np, int r, int j) {
  const DevView& d = f.d;
  int path[32];
  int depth = 0;
  for (int a = r; a >= 0 && depth < 32; a = d.anc[a]) path[depth++] = a;
  double x = d.p[j];
  for (int i = depth - 1; i >= 0; --i) x = (x + f.delta[(size_t)path[i] * d.lx + j]) + np.g[(size_t)path[i] * d.lx + j];
  return x;
}

// ---------------------------------------------------------------- k_chain_down
__global__ void __launch_bounds__(SC_THREADS) k_chain_down(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx;
  const int nst = d.H - f.kstar, ci = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rd = 3 * nu + lx + 2;                           // [L | e_off | ebar | g | aux]
  double* rec = reinterpret_cast<double*>(smem_raw);        // nst * rd
  double* Z = rec + (size_t)nst * rd;                       // nst * nu: z, then u
  double* T = Z + (size_t)nst * nu;                         // nst * FAST_MAXNS
  double* ua = T + (size_t)nst * FAST_MAXNS;                // nu
  double* xa = ua + nu;                                     // lx
  int* rows = reinterpret_cast<int*>(xa + lx);
  double* opsp = reinterpret_cast<double*>(rows + ((nst + 3) & ~3));
  const NodePtrs np = *d.np;
  if (threadIdx.x < nst) rows[threadIdx.x] = f.chain_node[(size_t)threadIdx.x * f.nchain + ci];
  __syncthreads();
  FOR_RC(nst, 6, (nu >> 1), t, k) cp16(rec + (size_t)t * rd + 2 * k, f.Lb + (size_t)rows[t] * nu + 2 * k);
  FOR_RC(nst, 6, (nu >> 1), t, k) cp16(rec + (size_t)t * rd + nu + 2 * k, np.e_off + (size_t)rows[t] * nu + 2 * k);
  FOR_RC(nst, 6, (nu >> 1), t, k) cp16(rec + (size_t)t * rd + 2 * nu + 2 * k, np.ebar + (size_t)rows[t] * nu + 2 * k);
  FOR_RC(nst, 5, (lx >> 1), t, k) cp16(rec + (size_t)t * rd + 3 * nu + 2 * k, np.g + (size_t)rows[t] * lx + 2 * k);
  cp_commit();
  const Ops op = load_ops(f, opsp);
  {
    const int a = d.anc[rows[0]];
    for (int k = threadIdx.x; k < nu; k += blockDim.x) ua[k] = a < 0 ? d.q[k] : d.U[(size_t)a * nu + k];
    for (int j = threadIdx.x; j < nt; j += blockDim.x) xa[j] = a < 0 ? d.p[j] : branch_x(f, np, a, j);
  }
  cp_wait<0>();
  __syncthreads();
  if (threadIdx.x < nu) {  // z_t = (u_anc + Ebar_t) - sum_{t' <= t} L_t'
    const int k = threadIdx.x;
    const double u0 = ua[k];
    double acc = 0.0;
    for (int t = 0; t < nst; ++t) {
      const double* R = rec + (size_t)t * rd;
      acc = acc + R[k];
      Z[t * nu + k] = (u0 + R[2 * nu + k]) - acc;
    }
  }
  __syncthreads();
  proj_rows(d, op, Z, Z, T, nst);
  FOR_NU(nst, t, k) {
    const double u = rec[(size_t)t * rd + nu + k] + Z[t * nu + k];
    Z[t * nu + k] = u;
    d.U[(size_t)rows[t] * nu + k] = u;
  }
  __syncthreads();
  FOR_NT(nst, t, j) {  // u B^T into the dead L slot
    double bu = 0.0;
    for (int e = op.brp[j]; e < op.brp[j + 1]; ++e) bu = fma(Z[t * nu + op.brc[e]], op.brv[e], bu);
    rec[(size_t)t * rd + j] = bu;
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    const int j = threadIdx.x;
    double x = xa[j];
    for (int t = 0; t < nst; ++t) {
      x = (x + rec[(size_t)t * rd + j]) + rec[(size_t)t * rd + 3 * nu + j];
      d.X[(size_t)rows[t] * lx + j] = x;
    }
  }
}

// ---------------------------------------------------------------- k_prox_nodes
// Node-parallel Moreau prox (bit-exact), ergodic averages, next collapsed dual.
__global__ void __launch_bounds__(SC_THREADS) k_prox_nodes(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, W = d.W, lx = d.lx;
  const RecOff o = rec_off(d);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* rec = reinterpret_cast<double*>(smem_raw);  // SC_NPB * f.rec
  double* U = rec + (size_t)SC_NPB * f.rec;           // SC_NPB * nu
  double* X = U + SC_NPB * nu;                        // SC_NPB * lx
  double* stp = X + SC_NPB * lx;                      // 2 * SC_NPB
  double* s_bnd = stp + 2 * SC_NPB;                   // bounds
  int* rows = reinterpret_cast<int*>(s_bnd + 3 * nt + 2 * nu);
  const int r0 = blockIdx.x * SC_NPB;
  const int nrow = min(SC_NPB, d.n - r0);
  const int it = *d.iter;
  if (threadIdx.x < nrow) rows[threadIdx.x] = r0 + threadIdx.x;
  __syncthreads();
  FOR_RC(nrow, 7, (W >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.y + 2 * k, ybuf(d, it) + (size_t)rows[m] * W + 2 * k);
  FOR_RC(nrow, 7, (W >> 1), m, k)
    cp16(rec + (size_t)m * f.rec + o.ym + 2 * k, ybuf(d, it + 2) + (size_t)rows[m] * W + 2 * k);
  FOR_RC(nrow, 6, (nu >> 1), m, k) cp16(U + m * nu + 2 * k, d.U + (size_t)rows[m] * nu + 2 * k);
  if (it > 0) {
    FOR_RC(nrow, 6, (nu >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.ua + 2 * k, d.Ua + (size_t)rows[m] * nu + 2 * k);
    FOR_RC(nrow, 5, (lx >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.xa + 2 * k, d.Xa + (size_t)rows[m] * lx + 2 * k);
  }
  FOR_RC(nrow, 5, (lx >> 1), m, k) {
    if (rows[m] >= f.n_branch) cp16(X + m * lx + 2 * k, d.X + (size_t)rows[m] * lx + 2 * k);
  }
  cp_commit();
  for (int i = threadIdx.x; i < nt; i += blockDim.x) {
    s_bnd[i] = d.xmin[i];
    s_bnd[nt + i] = d.xmax[i];
    s_bnd[2 * nt + i] = d.xsafe[i];
  }
  for (int i = threadIdx.x; i < nu; i += blockDim.x) {
    s_bnd[3 * nt + i] = d.umin[i];
    s_bnd[3 * nt + nu + i] = d.umax[i];
  }
  const NodePtrs np = *d.np;
  FOR_NT(nrow, m, j) {  // branching rows: x by walk-up; store X
    if (rows[m] < f.n_branch) {
      const double x = branch_x(f, np, rows[m], j);
      X[m * lx + j] = x;
      d.X[(size_t)rows[m] * lx + j] = x;
    }
  }
  cp_wait<0>();
  __syncthreads();
  Ops op{};
  op.xmin = s_bnd;
  op.xmax = s_bnd + nt;
  op.xsafe = s_bnd + 2 * nt;
  op.umin = s_bnd + 3 * nt;
  op.umax = s_bnd + 3 * nt + nu;
  const bool has_next = it + 1 < f.max_iter;
  prox_rows(f, op, rows, nrow, U, nu, X, lx, rec, f.rec, rec + o.lin, f.rec, stp, it, d.beta[it], d.theta[it],
            has_next ? d.beta[it + 1] : 0.0, has_next);
}

}  // namespace wmpc

namespace wmpc {
// Ebar of branching rows: sum of e_off over the strict ancestors, root first.
__global__ void k_branch_ebar(const int* __restrict__ anc, int nb, int nu, const double* __restrict__ e_off,
                              double* ebar) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nb * nu) return;
  const int r = idx / nu, k = idx - r * nu;
  int path[32];
  int depth = 0;
  for (int a = anc[r]; a >= 0 && depth < 32; a = anc[a]) path[depth++] = a;
  double acc = 0.0;
  for (int i = depth - 1; i >= 0; --i) acc = acc + e_off[(size_t)path[i] * nu + k];
  ebar[(size_t)r * nu + k] = acc;
}
}  // namespace wmpc
