// wmpc_scan.cuh — scan-form APG iteration as a CUDA graph of small kernels
// (structured case: A = I, W_u = c I, every stage factor = the null(E)
// projector P; see wmpc_fast.cuh for the derivation).
//
// The Riccati-type recursion over the tree collapses to scans because P is
// idempotent (P(a + P b) = P(a + b)):
//   wbar_r = sum_{sub(r)} Yx,     a_r = (Yu_r + wbar_r B) + R_r,
//   lin_r  = a_r + P sum_{desc(r)} a,           L_r = lin_r / (2c p_r),
//   u_r    = e_off_r + P(q + sum_{anc(r)} e_off - sum_{path(r)} L),
//   x_r    = (x_anc + u_r B^T) + g_r.
// R-free iteration (f.rfree): L is linear in Yc plus a constant part from R,
// so u = ut - P(sum_{path} L_Y) with ut = u at Yc = 0 computed once per solve
// (wmpc_apg_begin) and L_Y the Yc part: the per-iteration passes never read R,
// and the down pass needs neither q nor the e_off prefix sums.
// Rows at stages >= kstar form nchain chains laid out stage-major
// (row = n_branch + t*nchain + chain). One APG iteration (solver.py:460-506)
// is the graph
//   k_chain_up       one CTA per chain: suffix scans + projector -> L, subtree totals
//   k_branch_grp x G one CTA per branching row of a stage group: depth-weighted
//                    sums over the group's rows and the frontier totals below -> L
//   k_chain_down     one CTA per chain: the whole root path (ancestors + chain):
//                    prefix scans + projector -> U, X
//   k_prox_nodes     node-parallel Moreau prox, ergodic averages, next collapsed dual
// Graph edges replace grid barriers (measured 0.7 us per dependent kernel vs
// 1.25 us per cooperative grid.sync on B200). The iteration counter is bumped
// by k_chain_up; k_prox_nodes uses it - 1.
#pragma once
#include "wmpc_fast.cuh"

namespace wmpc {

constexpr int SC_THREADS = 256;
#ifndef GRP_THREADS_N
#define GRP_THREADS_N 256
#endif
constexpr int GRP_THREADS = GRP_THREADS_N;  // k_branch_grp CTA (>= 128: one thread per u element)
constexpr int SC_NPB = 4;    // nodes per CTA in k_prox_nodes
constexpr int SC_MAXK = 30;  // max branching depth (bits of cown)

// ---------------------------------------------------------------- operators
// The projector onto null(E) is applied as P z = z - E^T (K z) with
// K = (E E^T)^{-1} E = (E^+)^T stored sparse (for the Barcelona network E E^T
// is diagonal, so K has the 56 nonzeros of E: ~130 flops per row instead of
// the ~2,000 of a dense E^+ pass).
// Blob layout (doubles, then ints): [K vals | E CSC vals | B CSC vals | B CSR vals
// | pad | K ptr | K cols | E CSC ptr | E CSC rows | B CSC ptr | B CSC rows | B CSR ptr | B CSR cols]
struct BlobLayout {
  int kv, ecv, bcv, brv, dbl_end, kptr, kcol, ecp, ecr, bcp, bcr, brp, brc, bytes;
};
__host__ __device__ inline BlobLayout blob_layout(int nt, int nu, int ns, int knz, int enz, int bnz) {
  BlobLayout b;
  b.kv = 0;
  b.ecv = b.kv + knz;
  b.bcv = b.ecv + enz;
  b.brv = b.bcv + bnz;
  b.dbl_end = b.brv + bnz;
  b.dbl_end += b.dbl_end & 1;
  b.kptr = 2 * b.dbl_end;  // int offsets
  b.kcol = b.kptr + ns + 1;
  b.ecp = b.kcol + knz;
  b.ecr = b.ecp + nu + 1;
  b.bcp = b.ecr + enz;
  b.bcr = b.bcp + nu + 1;
  b.brp = b.bcr + bnz;
  b.brc = b.brp + nt + 1;
  const int iend = b.brc + bnz;
  b.bytes = ((iend * 4 + 15) / 16) * 16;
  return b;
}

__device__ __forceinline__ void issue_blob(const FastView& f, void* dst) {
  const int4* src = reinterpret_cast<const int4*>(f.blob);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = threadIdx.x; i < f.blob16; i += blockDim.x) cp16(d + i, src + i);
}
__device__ __forceinline__ Ops blob_ops(const FastView& f, const void* sp) {
  const DevView& d = f.d;
  const BlobLayout b = blob_layout(d.nt, d.nu, d.ns, f.k_nnz, f.e_nnz, f.b_nnz);
  const double* dp = reinterpret_cast<const double*>(sp);
  const int* ip = reinterpret_cast<const int*>(sp);
  Ops op{};
  op.kval = dp + b.kv;
  op.ecv = dp + b.ecv;
  op.bcv = dp + b.bcv;
  op.brv = dp + b.brv;
  op.kptr = ip + b.kptr;
  op.kcol = ip + b.kcol;
  op.ecp = ip + b.ecp;
  op.ecr = ip + b.ecr;
  op.bcp = ip + b.bcp;
  op.bcr = ip + b.bcr;
  op.brp = ip + b.brp;
  op.brc = ip + b.brc;
  return op;
}

// out[m*so + k] = (P in[m])_k for m < rows (rows of stride si; in place
// allowed). T scratch rows x FAST_MAXNS. 2 barriers.
__device__ __forceinline__ void proj_rows_s(const DevView& d, const Ops& op, const double* in, int si, double* out,
                                            int so, double* T, int rows) {
  const int nu = d.nu, ns = d.ns;
  FOR_RC(rows, 5, ns, m, i) {
    const double* z = in + (size_t)m * si;
    double v = 0.0;
    for (int e = op.kptr[i]; e < op.kptr[i + 1]; ++e) v = fma(op.kval[e], z[op.kcol[e]], v);
    T[m * FAST_MAXNS + i] = v;
  }
  __syncthreads();
  FOR_NU(rows, m, k) {
    const double* tm = T + m * FAST_MAXNS;
    double c = 0.0;
    for (int e = op.ecp[k]; e < op.ecp[k + 1]; ++e) c = fma(op.ecv[e], tm[op.ecr[e]], c);
    out[(size_t)m * so + k] = in[(size_t)m * si + k] - c;
  }
  __syncthreads();
}
__device__ __forceinline__ void proj_rows(const DevView& d, const Ops& op, const double* in, double* out,
                                          double* T, int rows) {
  proj_rows_s(d, op, in, d.nu, out, d.nu, T, rows);
}

__device__ __forceinline__ int chain_row(const FastView& f, int t, int ci) { return f.n_branch + t * f.nchain + ci; }

// Programmatic dependent launch (the graph kernels are launched with
// programmatic stream serialization): a kernel issues the loads that do not
// depend on its predecessor (node data, operators, older iterates), then
// waits for the predecessor grid, then lets its own successor launch.
// Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Register-resident sparse operators (ELL, width WE): a thread owns one column
// (or row) for a whole phase and loops over tree rows, so the operator entries
// are loaded once (from L1) instead of walked through shared memory per row.
enum { ELL_BC = 0 };  // owner offsets: B by column [0,nu), B by row [nu,nu+nt), E by column, K by row
// Gradient-side arrays (Yc, L, subtree totals, U, X, node data, operators) in
// the precision TG of the dual-gradient kernels: double (default) or float
// (fp32 mode, SolverConfig.precision == "fp32"); y, the averages and every
// prox/certificate computation stay fp64.
template <typename TG>
struct GA {
  TG *Yc, *Lb, *Asub, *wbar, *U, *X;
  const TG *e_off, *R, *g, *aux, *ell_val;
};
template <typename TG>
__device__ __forceinline__ GA<TG> ga(const FastView& f);
template <>
__device__ __forceinline__ GA<double> ga<double>(const FastView& f) {
  const NodePtrs np = *f.d.np;
  return GA<double>{f.d.Yc, f.Lb, f.Asub, f.d.wbar, f.d.U, f.d.X, np.e_off, np.R, np.g, f.aux, f.ell_val};
}
template <>
__device__ __forceinline__ GA<float> ga<float>(const FastView& f) {
  return GA<float>{f.g32.Yc, f.g32.Lb, f.g32.Asub, f.g32.wbar, f.g32.U, f.g32.X, f.g32.e_off, f.g32.R, f.g32.g,
                   f.g32.aux, f.g32.ell_val};
}
// async copy of two elements (16 B for double, 8 B for float)
__device__ __forceinline__ void cpair(double* dst, const double* src) { cp16(dst, src); }
__device__ __forceinline__ void cpair(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int WE, typename TG = double>
struct Ell {
  int idx[WE];
  TG val[WE];
};
// Entries past an owner's count are stored as (0, 0.0): no predication, and a
// zero weight times a finite operand adds nothing (a dense product would
// propagate a non-finite operand the same way).
// Owners are stored with stride ell_w (4 or 8, >= WE): one owner's entries
// are read with 16-byte vector loads (idx as int4, values as double2/float4).
template <int WE, typename TG = double>
__device__ __forceinline__ Ell<WE, TG> ell_load(const FastView& f, int owner) {
  Ell<WE, TG> o;
  const int* ip = f.ell_idx + (size_t)owner * f.ell_w;
  const TG* vp = ga<TG>(f).ell_val + (size_t)owner * f.ell_w;
  constexpr int NI = (WE + 3) / 4;
  int ib[4 * NI];
#pragma unroll
  for (int q = 0; q < NI; ++q) {
    const int4 v = reinterpret_cast<const int4*>(ip)[q];
    ib[4 * q] = v.x; ib[4 * q + 1] = v.y; ib[4 * q + 2] = v.z; ib[4 * q + 3] = v.w;
  }
#pragma unroll
  for (int e = 0; e < WE; ++e) o.idx[e] = ib[e];
  if constexpr (sizeof(TG) == 8) {
    constexpr int NV = (WE + 1) / 2;
    double vb[2 * NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const double2 v = reinterpret_cast<const double2*>(vp)[q];
      vb[2 * q] = v.x; vb[2 * q + 1] = v.y;
    }
#pragma unroll
    for (int e = 0; e < WE; ++e) o.val[e] = (TG)vb[e];
  } else {
    constexpr int NV = (WE + 3) / 4;
    float vb[4 * NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const float4 v = reinterpret_cast<const float4*>(vp)[q];
      vb[4 * q] = v.x; vb[4 * q + 1] = v.y; vb[4 * q + 2] = v.z; vb[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int e = 0; e < WE; ++e) o.val[e] = (TG)vb[e];
  }
  return o;
}
template <int WE, typename TG>
__device__ __forceinline__ TG ell_dot(const Ell<WE, TG>& o, const TG* x) {
  TG s = 0;
#pragma unroll
  for (int e = 0; e < WE; ++e) s = fma(o.val[e], x[o.idx[e]], s);
  return s;
}
// Per-operator widths of a variant: V = 4 is the water-network shape (a flow
// touches <= 2 tanks and <= 1 mixing node, a tank has <= 3 flows, a mixing
// row of K <= 4 flows); V = 8 is the generic fallback.
template <int V>
struct EllW {
  static constexpr int BC = V == 4 ? 2 : 8, BR = V == 4 ? 3 : 8, EC = V == 4 ? 1 : 8, KR = V == 4 ? 4 : 8;
};
__device__ __forceinline__ int own_bc(const DevView& d, int k) { return k; }
__device__ __forceinline__ int own_br(const DevView& d, int j) { return d.nu + j; }
__device__ __forceinline__ int own_ec(const DevView& d, int k) { return d.nu + d.nt + k; }
__device__ __forceinline__ int own_kr(const DevView& d, int i) { return 2 * d.nu + d.nt + i; }

// ---------------------------------------------------------------- k_chain_up
// Shared: rec nst x (ly + nu + 2) [Yx->wbar | Yu->a | R->S->PS | aux],
// T nst x FAST_MAXNS (in-place phases keep 4 CTAs per SM at H = 24).
// OCC: many chains (several waves) -> cap registers for 3 CTAs per SM; few
// chains (one wave, latency-bound) -> let the compiler keep more in registers.
template <int WE, typename TG, bool OCC>
__global__ void __launch_bounds__(512, OCC ? 3 : 1) k_chain_up(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly, ns = d.ns;
  const int nst = d.H - f.kstar, ci = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int ra = ly + nu + 2;
  TG* rec = reinterpret_cast<TG*>(smem_raw);
  TG* T = rec + (size_t)nst * ra;
  const GA<TG> G = ga<TG>(f);
  const bool withR = !f.rfree;
  if (withR)
    FOR_RC(nst - 1, 6, (nu >> 1), t, k)
      cpair(rec + (size_t)t * ra + ly + 2 * k, G.R + (size_t)chain_row(f, t, ci) * nu + 2 * k);
  if (threadIdx.x < nst) cpair(rec + (size_t)threadIdx.x * ra + ly + nu, G.aux + (size_t)chain_row(f, threadIdx.x, ci) * 2);
  const int k = threadIdx.x & 127, tk = threadIdx.x >> 7, sk = blockDim.x >> 7;
  const int i = threadIdx.x & 31, ti = threadIdx.x >> 5, si = blockDim.x >> 5;
  const Ell<EllW<WE>::BC, TG> bc = ell_load<EllW<WE>::BC, TG>(f, own_bc(d, k < nu ? k : 0));
  const Ell<EllW<WE>::KR, TG> kr = ell_load<EllW<WE>::KR, TG>(f, own_kr(d, i < ns ? i : 0));
  const Ell<EllW<WE>::EC, TG> ec = ell_load<EllW<WE>::EC, TG>(f, own_ec(d, k < nu ? k : 0));
  pdl_wait();  // Yc comes from the prox of the previous iteration
  pdl_trigger();
  FOR_RC(nst, 7, (ly >> 1), t, k) cpair(rec + (size_t)t * ra + 2 * k, G.Yc + (size_t)chain_row(f, t, ci) * ly + 2 * k);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  if (threadIdx.x < nt) {  // wbar suffix scan in place: wbar_t = Yx_t + wbar_{t+1}
    const int j = threadIdx.x;
    TG acc = 0;
    for (int t = nst - 1; t >= 0; --t) {
      const TG yx = rec[(size_t)t * ra + j];
      acc = t == nst - 1 ? yx : yx + acc;
      rec[(size_t)t * ra + j] = acc;
    }
    G.wbar[(size_t)chain_row(f, 0, ci) * lx + j] = acc;
  }
  __syncthreads();
  if (k < nu)
    for (int t = tk; t < nst; t += sk) {  // a = (Yu + wbar B) + R, over Yu
      TG* R = rec + (size_t)t * ra;
      TG a = R[lx + k] + ell_dot(bc, R);
      if (withR && t < nst - 1) a = a + R[ly + k];
      R[lx + k] = a;
    }
  __syncthreads();
  if (threadIdx.x < nu) {  // S_t = A_{t+1} over R, A_t = a_t + S_t
    TG acc = 0;
    for (int t = nst - 1; t >= 0; --t) {
      TG* R = rec + (size_t)t * ra;
      R[ly + threadIdx.x] = acc;
      const TG a = R[lx + threadIdx.x];
      acc = t == nst - 1 ? a : a + acc;
    }
    G.Asub[(size_t)chain_row(f, 0, ci) * nu + threadIdx.x] = acc;
  }
  __syncthreads();
  if (i < ns) {  // T = K S
    for (int t = ti; t < nst - 1; t += si) T[t * FAST_MAXNS + i] = ell_dot(kr, rec + (size_t)t * ra + ly);
  }
  __syncthreads();
  if (k < nu) {  // L = (a + (S - E^T T)) / (2c p)
    for (int t = tk; t < nst; t += sk) {
      const TG* R = rec + (size_t)t * ra;
      const TG a = R[lx + k];
      const TG l = t < nst - 1 ? a + (R[ly + k] - ell_dot(ec, T + t * FAST_MAXNS)) : a;
      G.Lb[(size_t)chain_row(f, t, ci) * nu + k] = l * R[ly + nu];
    }
  }
}

// ---------------------------------------------------------------- k_branch_grp
// One CTA per branching row r of a stage group. Items: the group's rows below
// r (kind 0, weight depth(e)-depth(r)) and the frontier rows right below the
// group (kind 1, weight depth(f)-depth(r)-1; chain tops or the top rows of the
// group below, whose wbar / subtree totals are already final):
//   W1 = wbar_r = Yx_r + sum_0 Yx_e + sum_1 wbar_f
//   W2 = sum_{d in desc_B(r)} wbar_d = sum_0 w Yx_e + sum_1 w wbar_f
//   Su = sum_0 (Yu_e + R_e) + sum_1 Asub_f
//   a_r = (Yu_r + W1 B) + R_r,  S_r = Su + W2 B,  lin_r = a_r + P S_r.
//
// Subtree sharding (shard.py): a row replicated on several ranks runs twice.
// mode GRP_PARTIAL writes the item sums (without the row's own Yx) into the
// exchange buffer at the row's global replicated index; after the host-level
// all-reduce over ranks, mode GRP_FINISH reads them back and finishes the row
// identically on every rank. bump: first kernel of an APG iteration.
// GRP_LATE (or-ed into mode): this row group's own rows got their Yc from the
// immediate predecessor (k_chain_dp runs the branching rows' prox), so every
// Yc load waits for it.
enum { GRP_FULL = 0, GRP_PARTIAL = 1, GRP_FINISH = 2, GRP_LATE = 4 };
// GT: threads per CTA (>= 128, one per u element); 128 on the k_chain_dp paths (measured: C3 41.6 -> 40.3 us),
// 256 on the graph path (C2 19.4 vs 20.4 with 128)
template <int WE, typename TG, int GT = GRP_THREADS>
__global__ void __launch_bounds__(GT) k_branch_grp(FastView f, int r0, int bump, int mode) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly;
  const int r = r0 + blockIdx.x;
  constexpr int NW = GT / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TG* part = reinterpret_cast<TG*>(smem_raw);  // NW x 256: [s1 64 | s2 64 | su 128]
  TG* W1 = part + NW * 256;  // lx
  TG* W2 = W1 + lx;          // lx
  TG* av = W2 + lx;          // nu
  TG* Sv = av + nu;          // nu
  TG* T = Sv + nu;           // FAST_MAXNS
  const GA<TG> G = ga<TG>(f);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---- before the predecessor finishes: everything that does not come from it
  // (item lists, operators, this row's own data, in-group rows' Yc and R: the
  // previous iteration's prox finished before the predecessor started)
  const int k = threadIdx.x;
  const Ell<EllW<WE>::BC, TG> bc = ell_load<EllW<WE>::BC, TG>(f, own_bc(d, k < nu ? k : 0));
  const Ell<EllW<WE>::KR, TG> kr = ell_load<EllW<WE>::KR, TG>(f, own_kr(d, k < d.ns ? k : 0));
  const Ell<EllW<WE>::EC, TG> ec = ell_load<EllW<WE>::EC, TG>(f, own_ec(d, k < nu ? k : 0));
  if (mode & GRP_LATE) pdl_wait();
  mode &= 3;
  const TG own_yx = k < nt ? G.Yc[(size_t)r * ly + k] : TG(0);
  const TG own_yu = k < nu ? G.Yc[(size_t)r * ly + lx + k] : TG(0);
  const bool withR = !f.rfree;
  const TG own_R = withR && k < nu ? G.R[(size_t)r * nu + k] : TG(0);
  const TG own_aux = G.aux[(size_t)r * 2];
  const int e0 = mode == GRP_FINISH ? 0 : f.gi_ptr[r], e1 = mode == GRP_FINISH ? 0 : f.gi_ptr[r + 1];
  constexpr int MQ = 2;  // items per warp prefetched ahead of the wait
  int itm[MQ];
  TG wq[MQ], vx[MQ][2], vu[MQ][4];
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    const int e = e0 + warp + NW * q;
    itm[q] = e < e1 ? f.gi_item[e] : -1;
    wq[q] = e < e1 ? (TG)f.gi_w[e] : TG(0);
    const bool in_group = itm[q] >= 0 && !(itm[q] & 1);
    const size_t row = in_group ? (size_t)(itm[q] >> 1) : 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = lane + 32 * i;
      vx[q][i] = in_group && c < nt ? G.Yc[row * ly + c] : TG(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = lane + 32 * i;
      vu[q][i] = in_group && c < nu ? (withR ? G.Yc[row * ly + lx + c] + G.R[row * nu + c]
                                             : G.Yc[row * ly + lx + c]) : TG(0);
    }
  }
  pdl_wait();  // chain totals / lower groups of this iteration
  pdl_trigger();
  if (bump && blockIdx.x == 0 && threadIdx.x == 0) *d.iter += 1;
  TG s1[2] = {0, 0}, s2[2] = {0, 0}, su[4] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    if (itm[q] >= 0 && (itm[q] & 1)) {  // frontier rows: totals of the predecessor
      const size_t row = (size_t)(itm[q] >> 1);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = lane + 32 * i;
        vx[q][i] = c < nt ? G.wbar[row * lx + c] : TG(0);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = lane + 32 * i;
        vu[q][i] = c < nu ? G.Asub[row * nu + c] : TG(0);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    if (itm[q] < 0) break;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      s1[i] += vx[q][i];
      s2[i] = fma(wq[q], vx[q][i], s2[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) su[i] += vu[q][i];
  }
  for (int e = e0 + warp + NW * MQ; e < e1; e += NW) {  // rows with more than MQ items per warp
    const int item = f.gi_item[e];
    const size_t row = (size_t)(item >> 1);
    const bool fr = item & 1;
    const TG w = (TG)f.gi_w[e];
    const TG* px = fr ? G.wbar + row * lx : G.Yc + row * ly;
    TG x2[2], u4[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = lane + 32 * i;
      x2[i] = c < nt ? px[c] : TG(0);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = lane + 32 * i;
      u4[i] = c < nu ? (fr ? G.Asub[row * nu + c]
                           : (withR ? G.Yc[row * ly + lx + c] + G.R[row * nu + c] : G.Yc[row * ly + lx + c]))
                     : TG(0);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      s1[i] += x2[i];
      s2[i] = fma(w, x2[i], s2[i]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) su[i] += u4[i];
  }
  TG* pw = part + warp * 256;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    pw[lane + 32 * i] = s1[i];
    pw[64 + lane + 32 * i] = s2[i];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) pw[128 + lane + 32 * i] = su[i];
  __syncthreads();
  double* xb = mode == GRP_FULL ? nullptr : f.xbuf + (size_t)f.rep_gidx[r] * 256;  // fp64 (sharding: TG = double)
  if (mode == GRP_PARTIAL) {  // item sums to the exchange buffer
    for (int c = threadIdx.x; c < 256; c += blockDim.x) {
      TG a = part[c];
      for (int w = 1; w < NW; ++w) a += part[w * 256 + c];
      xb[c] = a;
    }
    return;
  }
  if (k < nt) {
    TG a1, a2;
    if (xb) {
      a1 = xb[k];
      a2 = xb[64 + k];
    } else {
      a1 = part[k];
      a2 = part[64 + k];
      for (int w = 1; w < NW; ++w) {
        a1 += part[w * 256 + k];
        a2 += part[w * 256 + 64 + k];
      }
    }
    W1[k] = own_yx + a1;
    W2[k] = a2;
  }
  __syncthreads();
  if (k < nu) {
    TG s;
    if (xb) {
      s = xb[128 + k];
    } else {
      s = part[128 + k];
      for (int w = 1; w < NW; ++w) s += part[w * 256 + 128 + k];
    }
    av[k] = (own_yu + ell_dot(bc, W1)) + own_R;
    Sv[k] = s + ell_dot(bc, W2);
  }
  if (k < nt) G.wbar[(size_t)r * lx + k] = W1[k];
  __syncthreads();
  if (k < nu) G.Asub[(size_t)r * nu + k] = av[k] + Sv[k];
  if (k < d.ns) T[k] = ell_dot(kr, Sv);
  __syncthreads();
  if (k < nu) G.Lb[(size_t)r * nu + k] = (av[k] + (Sv[k] - ell_dot(ec, T))) * own_aux;
}

// ---------------------------------------------------------------- k_chain_down
// One CTA per chain over its whole root path: the kstar ancestors (root
// first) then the nst chain rows, H rows in all.
//   z_m = (q + sum_{m' < m} e_off_m') - sum_{m' <= m} L_m',  u_m = e_off_m + P z_m,
//   x_m = (x_{m-1} + u_m B^T) + g_m,  x_{-1} = p.
// Ancestor rows are written by the chain that owns them (cown).
// Shared: rec H x (2nu + lx) [L->z->u | e_off->Bu | g], T H x FAST_MAXNS, rows H.
template <int WE, typename TG, bool OCC>
__global__ void __launch_bounds__(512, OCC ? 3 : 1) k_chain_down(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ns = d.ns;
  const int kb = f.kstar, nr = d.H, ci = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rd = 2 * nu + lx;
  TG* rec = reinterpret_cast<TG*>(smem_raw);
  TG* T = rec + (size_t)nr * rd;
  int* rows = reinterpret_cast<int*>(T + (size_t)nr * FAST_MAXNS);
  const GA<TG> G = ga<TG>(f);
  // global row of path position m: chain rows by arithmetic, ancestors from
  // cpath (read per use: no CTA-wide wait for a row table before the copies)
  auto grow = [&](int m) { return m < kb ? f.cpath[(size_t)ci * kb + m] : chain_row(f, m - kb, ci); };
  if (threadIdx.x < nr) rows[threadIdx.x] = grow(threadIdx.x);  // for the stores (read after a barrier)
  const TG* base = f.rfree ? (sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32) : G.e_off;
  FOR_RC(nr, 6, (nu >> 1), m, k) cpair(rec + (size_t)m * rd + nu + 2 * k, base + (size_t)grow(m) * nu + 2 * k);
  FOR_RC(nr, 5, (lx >> 1), m, k) cpair(rec + (size_t)m * rd + 2 * nu + 2 * k, G.g + (size_t)grow(m) * lx + 2 * k);
  // the chain rows' L were written by k_chain_up, which finished before the
  // group kernels (our predecessor) started: fetch them before the wait
  const int m_pre = f.lb_prewait ? kb : nr;
  FOR_RC(nr - m_pre, 6, (nu >> 1), m, k)
    cpair(rec + (size_t)(m_pre + m) * rd + 2 * k, G.Lb + (size_t)grow(m_pre + m) * nu + 2 * k);
  const int k = threadIdx.x & 127, tk = threadIdx.x >> 7, sk = blockDim.x >> 7;
  const int i = threadIdx.x & 31, ti = threadIdx.x >> 5, si = blockDim.x >> 5;
  const int j = threadIdx.x & 63, tj = threadIdx.x >> 6, sj = blockDim.x >> 6;
  const Ell<EllW<WE>::KR, TG> kr = ell_load<EllW<WE>::KR, TG>(f, own_kr(d, i < ns ? i : 0));
  const Ell<EllW<WE>::EC, TG> ec = ell_load<EllW<WE>::EC, TG>(f, own_ec(d, k < nu ? k : 0));
  const Ell<EllW<WE>::BR, TG> br = ell_load<EllW<WE>::BR, TG>(f, own_br(d, j < nt ? j : 0));
  pdl_wait();  // L of the branching rows comes from the last group kernel
  pdl_trigger();
  FOR_RC(m_pre, 6, (nu >> 1), m, k) cpair(rec + (size_t)m * rd + 2 * k, G.Lb + (size_t)grow(m) * nu + 2 * k);
  cp_commit();
  const unsigned own = kb > 0 ? f.cown[ci] : 0u;
  const TG qk = k < nu && !f.rfree ? (TG)d.q[k] : TG(0);
  cp_wait<0>();
  __syncthreads();
  if (threadIdx.x < nu) {
    TG ls = 0, es = qk;
    const bool rfree = f.rfree;
    for (int m = 0; m < nr; ++m) {
      TG* R = rec + (size_t)m * rd;
      ls = m == 0 ? R[k] : ls + R[k];
      R[k] = es - ls;  // z over L
      if (!rfree) es = es + R[nu + k];
    }
  }
  __syncthreads();
  if (i < ns) {  // T = K z
    for (int m = ti; m < nr; m += si) T[m * FAST_MAXNS + i] = ell_dot(kr, rec + (size_t)m * rd);
  }
  __syncthreads();
  if (k < nu) {  // u = e_off + (z - E^T T), in the z slot
    for (int m = tk; m < nr; m += sk) {
      TG* R = rec + (size_t)m * rd;
      const TG u = R[nu + k] + (R[k] - ell_dot(ec, T + m * FAST_MAXNS));
      R[k] = u;
      if (m >= kb || ((own >> m) & 1u)) G.U[(size_t)rows[m] * nu + k] = u;
    }
  }
  __syncthreads();
  if (j < nt) {  // u B^T into the dead e_off slot
    for (int m = tj; m < nr; m += sj) {
      TG* R = rec + (size_t)m * rd;
      R[nu + j] = ell_dot(br, R);
    }
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    TG x = (TG)d.p[threadIdx.x];
    for (int m = 0; m < nr; ++m) {
      const TG* R = rec + (size_t)m * rd;
      x = (x + R[nu + threadIdx.x]) + R[2 * nu + threadIdx.x];
      if (m >= kb || ((own >> m) & 1u)) G.X[(size_t)rows[m] * lx + threadIdx.x] = x;
    }
  }
}

// ---------------------------------------------------------------- k_chain_rollout
// Certificate rollout (problem.py:207-218) x = (x_anc + u B^T) + g over every
// root path in one launch (one CTA per chain, ancestors included), instead of
// one launch per stage. Shared: rec H x (nu + lx) [u -> Bu | g].
template <int WE>
__global__ void __launch_bounds__(256) k_chain_rollout(FastView f, const double* __restrict__ Uin, double* Xout) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx;
  const int kb = f.kstar, nr = d.H, ci = blockIdx.x;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rd = nu + lx;
  double* rec = reinterpret_cast<double*>(smem_raw);
  int* rows = reinterpret_cast<int*>(rec + (size_t)nr * rd);
  const NodePtrs np = *d.np;
  if (threadIdx.x < nr) {
    const int m = threadIdx.x;
    rows[m] = m < kb ? f.cpath[(size_t)ci * kb + m] : chain_row(f, m - kb, ci);
  }
  __syncthreads();
  FOR_RC(nr, 6, (nu >> 1), m, k) cp16(rec + (size_t)m * rd + 2 * k, Uin + (size_t)rows[m] * nu + 2 * k);
  FOR_RC(nr, 5, (lx >> 1), m, k) cp16(rec + (size_t)m * rd + nu + 2 * k, np.g + (size_t)rows[m] * lx + 2 * k);
  cp_commit();
  const int j = threadIdx.x & 63, tj = threadIdx.x >> 6, sj = blockDim.x >> 6;
  const Ell<EllW<WE>::BR, double> br = ell_load<EllW<WE>::BR, double>(f, own_br(d, j < nt ? j : 0));
  const unsigned own = kb > 0 ? f.cown[ci] : 0u;
  cp_wait<0>();
  __syncthreads();
  double bu[8];  // u B^T of this thread's rows (column j), before the u slots are reused
  int nb = 0;
  if (j < nt)
    for (int m = tj; m < nr && nb < 8; m += sj) bu[nb++] = ell_dot(br, rec + (size_t)m * rd);
  __syncthreads();
  if (j < nt) {
    nb = 0;
    for (int m = tj; m < nr && nb < 8; m += sj) rec[(size_t)m * rd + j] = bu[nb++];
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    double x = d.p[threadIdx.x];
    for (int m = 0; m < nr; ++m) {
      const double* R = rec + (size_t)m * rd;
      x = (x + R[threadIdx.x]) + R[nu + threadIdx.x];
      if (m >= kb || ((own >> m) & 1u)) Xout[(size_t)rows[m] * lx + threadIdx.x] = x;
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
  const int it = *d.iter - 1;
  if (threadIdx.x < nrow) rows[threadIdx.x] = r0 + threadIdx.x;
  FOR_RC(nrow, 7, (W >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.y + 2 * k, ybuf(d, it) + (size_t)(r0 + m) * W + 2 * k);
  FOR_RC(nrow, 7, (W >> 1), m, k)
    cp16(rec + (size_t)m * f.rec + o.ym + 2 * k, ybuf(d, it + 2) + (size_t)(r0 + m) * W + 2 * k);
  FOR_RC(nrow, 6, (nu >> 1), m, k) cp16(U + m * nu + 2 * k, d.U + (size_t)(r0 + m) * nu + 2 * k);
  FOR_RC(nrow, 5, (lx >> 1), m, k) cp16(X + m * lx + 2 * k, d.X + (size_t)(r0 + m) * lx + 2 * k);
  if (it > 0) {
    FOR_RC(nrow, 6, (nu >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.ua + 2 * k, d.Ua + (size_t)(r0 + m) * nu + 2 * k);
    FOR_RC(nrow, 5, (lx >> 1), m, k) cp16(rec + (size_t)m * f.rec + o.xa + 2 * k, d.Xa + (size_t)(r0 + m) * lx + 2 * k);
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
            has_next ? d.beta[it + 1] : 0.0, has_next, o);
}


// ---------------------------------------------------------------- k_prox_warp
// Node-parallel Moreau prox without CTA barriers: two warps per node, operands
// straight from memory into registers (every load issued up front).
//   x warp : the tank part, lanes own columns j and j+32 of both tank slots;
//            the two slot norms use numpy's pairwise order through an 8-lane
//            group each (pw_group8) on a per-warp shared array sd2 (2 x 64)
//   u warp : the input part (plain box projection), columns k + 32q
// Same expression order as prox_rows (bit-exact with numpy), V kept in registers.
struct ProxIt {
  int it;
  bool next;
  double gamma, ig, beta, theta, beta1, om;
};
__device__ __forceinline__ ProxIt prox_it(const FastView& f) {
  const DevView& d = f.d;
  ProxIt p;
  p.it = *d.iter - 1;
  p.next = p.it + 1 < f.max_iter;
  p.gamma = d.gamma;
  p.ig = f.inv_gamma;
  p.beta = d.beta[p.it];
  p.theta = d.theta[p.it];
  p.beta1 = p.next ? d.beta[p.it + 1] : 0.0;
  p.om = dsub(1.0, p.theta);
  return p;
}
// x: the node's state row (lx stride not needed: x[j]), returns bad.
template <typename TG>
__device__ __forceinline__ bool prox_x_warp(const FastView& f, const ProxIt& P, int r, const TG* x_row,
                                            double* sd2, TG* yc_row, bool pdl = false) {
  const DevView& d = f.d;
  const int nt = d.nt, W = d.W, lx = d.lx, ly = d.ly, lane = threadIdx.x & 31;
  const size_t rw = (size_t)r * W;
  const double* y = ybuf(d, P.it) + rw;
  const double* ym = ybuf(d, P.it + 2) + rw;
  double* yn = ybuf_w(d, P.it + 1) + rw;
  const double gamma = P.gamma, ig = P.ig;
  double xv[2], xa[2], y1[2], y2[2], m1[2], m2[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    const bool ok = j < nt;
    xa[q] = ok && P.it > 0 ? d.Xa[(size_t)r * lx + j] : 0.0;
    y1[q] = ok ? y[j] : 0.0;
    y2[q] = ok ? y[nt + j] : 0.0;
    m1[q] = ok ? ym[j] : 0.0;
    m2[q] = ok ? ym[nt + j] : 0.0;
  }
  if (pdl) pdl_wait();  // x comes from the down pass (the predecessor)
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    xv[q] = j < nt ? (double)x_row[j] : 0.0;
  }
  double v1[2], v2[2], V1[2], V2[2], c1[2], c2[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    const bool ok = j < nt;
    const double x = xv[q];
    if (ok) d.Xa[(size_t)r * lx + j] = P.it == 0 ? x : dadd(dmul(xa[q], P.om), dmul(P.theta, x));
    const double gx = dmul(gamma, x);
    v1[q] = dadd(dadd(y1[q], dmul(P.beta, dsub(y1[q], m1[q]))), gx);
    v2[q] = dadd(dadd(y2[q], dmul(P.beta, dsub(y2[q], m2[q]))), gx);
    V1[q] = div_by(v1[q], gamma, ig);
    V2[q] = div_by(v2[q], gamma, ig);
    c1[q] = ok ? np_clip(V1[q], d.xmin[j], d.xmax[j]) : 0.0;
    c2[q] = ok ? np_max(V2[q], d.xsafe[j]) : 0.0;
    if (ok) {
      const double df1 = dsub(V1[q], c1[q]), df2 = dsub(V2[q], c2[q]);
      sd2[j] = dmul(df1, df1);
      sd2[64 + j] = dmul(df2, df2);
    }
  }
  __syncwarp();
  double st = 0.0;
  if (lane < 16) {
    const int slot = lane >> 3;
    const double ssum = pw_group8(sd2 + 64 * slot, nt, lane & 7, 0xffu << (lane & 8));
    if ((lane & 7) == 0) {
      const double dist = __dsqrt_rn(ssum);
      const double thr = dmul(ig, slot ? d.w_s : d.w_x);  // prox parameter RN(1/gamma) (solver.py:571)
      st = dist > 0.0 ? np_min(1.0, div_exact(thr, dist)) : 0.0;
    }
  }
  const double st1 = __shfl_sync(0xffffffffu, st, 0), st2 = __shfl_sync(0xffffffffu, st, 8);
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (j < nt) {
      const double O1 = dsub(V1[q], dmul(st1, dsub(V1[q], c1[q])));
      const double O2 = dsub(V2[q], dmul(st2, dsub(V2[q], c2[q])));
      const double p1 = dsub(v1[q], dmul(gamma, O1)), p2 = dsub(v2[q], dmul(gamma, O2));
      yn[j] = p1;
      yn[nt + j] = p2;
      bad |= !isfinite(p1) || !isfinite(p2);
      if (P.next) {
        const double w1 = dadd(p1, dmul(P.beta1, dsub(p1, y1[q])));
        const double w2 = dadd(p2, dmul(P.beta1, dsub(p2, y2[q])));
        yc_row[j] = (TG)dadd(w1, w2);
      }
    }
  }
  __syncwarp();
  return bad;
}
template <typename TG>
__device__ __forceinline__ bool prox_u_warp(const FastView& f, const ProxIt& P, int r, const TG* u_row,
                                            TG* yc_row, bool pdl = false) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, W = d.W, lx = d.lx, ly = d.ly, lane = threadIdx.x & 31;
  const size_t rw = (size_t)r * W;
  const double* y = ybuf(d, P.it) + rw + 2 * nt;
  const double* ym = ybuf(d, P.it + 2) + rw + 2 * nt;
  double* yn = ybuf_w(d, P.it + 1) + rw + 2 * nt;
  constexpr int Q = 4;  // nu <= 128
  double uv[Q], ua[Q], y3[Q], m3[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k = lane + 32 * q;
    const bool ok = k < nu;
    ua[q] = ok && P.it > 0 ? d.Ua[(size_t)r * nu + k] : 0.0;
    y3[q] = ok ? y[k] : 0.0;
    m3[q] = ok ? ym[k] : 0.0;
  }
  if (pdl) pdl_wait();  // u comes from the down pass (the predecessor)
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k = lane + 32 * q;
    uv[q] = k < nu ? (double)u_row[k] : 0.0;
  }
  bool bad = false;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int k = lane + 32 * q;
    if (k < nu) {
      const double u = uv[q];
      d.Ua[(size_t)r * nu + k] = P.it == 0 ? u : dadd(dmul(ua[q], P.om), dmul(P.theta, u));
      const double v3 = dadd(dadd(y3[q], dmul(P.beta, dsub(y3[q], m3[q]))), dmul(P.gamma, u));
      const double V3 = div_by(v3, P.gamma, P.ig);
      const double p3 = dsub(v3, dmul(P.gamma, np_clip(V3, d.umin[k], d.umax[k])));
      yn[k] = p3;
      bad |= !isfinite(p3);
      if (P.next) yc_row[lx + k] = (TG)dadd(p3, dmul(P.beta1, dsub(p3, y3[q])));
    }
  }
  return bad;
}

#ifndef PW_ROWS_N
#define PW_ROWS_N 2  // measured: 2 nodes per 128-thread CTA beats 4 per 256 (C4 267.4 -> 260.8 us)
#endif
constexpr int PW_ROWS = PW_ROWS_N;  // nodes per CTA (2 warps each)
#ifndef PW_MINB
#define PW_MINB (16 / PW_ROWS_N)
#endif
template <typename TG>
__global__ void __launch_bounds__(64 * PW_ROWS, PW_MINB) k_prox_warp(FastView f) {
  const DevView& d = f.d;
  __shared__ double sd2[PW_ROWS][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = warp >> 1;
  const int r = blockIdx.x * PW_ROWS + m;
  if (r >= d.n) return;
  const ProxIt P = prox_it(f);
  const GA<TG> G = ga<TG>(f);
  TG* yc = G.Yc + (size_t)r * d.ly;
  const bool bad = (warp & 1) == 0 ? prox_x_warp<TG>(f, P, r, G.X + (size_t)r * d.lx, sd2[m], yc, true)
                                   : prox_u_warp<TG>(f, P, r, G.U + (size_t)r * d.nu, yc, true);
  pdl_trigger();
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(d.bad_nu, P.it);
}

// fp64 -> fp32 copy (fp32 mode node data) and back (fp32 iterates for results).
template <typename A, typename B>
__global__ void k_convert(const A* __restrict__ src, B* dst, size_t len) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = (B)src[i];
}

// Collapsed dual of a given y (no extrapolation): Yc = [y1 + y2 | y3], for
// evaluating the dual function with the chain/branch kernels (certificate).
__global__ void k_collapse(DevView d, const double* __restrict__ y, double* Yc) {
  const int nt = d.nt, nu = d.nu, W = d.W, lx = d.lx, ly = d.ly;
  const size_t len = (size_t)d.n * ly;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / ly;
    const int c = (int)(i - r * ly);
    const double* yr = y + r * W;
    Yc[i] = c < nt ? yr[c] + yr[nt + c] : (c < lx ? 0.0 : (c - lx < nu ? yr[2 * nt + c - lx] : 0.0));
  }
}

}  // namespace wmpc
