// wmpc_warp.cuh — warp-per-chain persistent APG kernel (structured case).
//
// Same math and bit-exact prox as k_apg_fast (wmpc_fast.cuh: projector form
// P = I - E^+ E of every stage factor, collapsed next-iteration dual), but the
// unit of work is one WARP per node: every warp owns whole chains and runs
// them independently, with only __syncwarp between the sub-steps of a node.
// A CTA of FW_WARPS warps therefore interleaves FW_WARPS independent
// dependency chains on its SM instead of stalling all warps on one node's
// ~12 block barriers (the v4 bottleneck).
//
// Lane layout (no integer division): element c of a row lives on lane
// c & 31, register slot c >> 5 (nt <= 64, nu <= 128, W <= 256).
// Each warp streams its nodes' rows into a private NR-slot shared-memory ring
// with 16-byte cp.async.cg, NR-1 node-steps ahead.
//
// Phases per iteration (solver.py:460-506):
//   A chain backward (warp per chain), grid sync,
//   B branching backward, one node per warp, grid sync per stage,
//   C branching forward + prox, one node per warp, grid sync per stage,
//   D chain forward + prox (warp per chain).
#pragma once
#include <cooperative_groups.h>

#include "wmpc_fast.cuh"

namespace wmpc {

constexpr int FW_WARPS = 8;
constexpr int FW_THREADS = 32 * FW_WARPS;
constexpr int FW_SCR = 128 + 128 + 128 + 64 + 64 + 256 + 128 + 32 + 8;  // per-warp scratch doubles

// per-warp scratch layout
struct WScr {
  double* L;    // 128: lin carry / projector input
  double* PZ;   // 128: projector output
  double* U;    // 128: u carry
  double* X;    // 64:  x carry
  double* WB;   // 64:  wbar carry
  double* V;    // 256: v, then y+
  double* D2;   // 128: squared distances (slot 1 | slot 2)
  double* T;    // 32:  E v
  double* S;    // 8:   step factors
};
__device__ __forceinline__ WScr wscr(double* base) {
  WScr s;
  s.L = base;
  s.PZ = s.L + 128;
  s.U = s.PZ + 128;
  s.X = s.U + 128;
  s.WB = s.X + 64;
  s.V = s.WB + 64;
  s.D2 = s.V + 256;
  s.T = s.D2 + 128;
  s.S = s.T + 32;
  return s;
}

struct WOps {
  const double* ept;  // E^+ transposed (ns x nu)
  const int* eptr;
  const int* ecol;
  const double* eval;
  const int* bcp;
  const int* bcr;
  const double* bcv;
  const int* brp;
  const int* brc;
  const double* brv;
  const double *xmin, *xmax, *xsafe, *umin, *umax;
};

// out = P in (nu-vectors in shared memory), one warp.
__device__ __forceinline__ void w_proj(const DevView& d, const WOps& op, const double* in, double* out,
                                       double* T, int lane) {
  const int nu = d.nu, ns = d.ns;
  if (lane < ns) {
    double t = 0.0;
    for (int e = op.eptr[lane]; e < op.eptr[lane + 1]; ++e) t = fma(op.eval[e], in[op.ecol[e]], t);
    T[lane] = t;
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = lane + 32 * k;
    if (j < nu) {
      double a0 = 0.0, a1 = 0.0;
      int i = 0;
      for (; i + 1 < ns; i += 2) {
        a0 = fma(op.ept[i * nu + j], T[i], a0);
        a1 = fma(op.ept[(i + 1) * nu + j], T[i + 1], a1);
      }
      if (i < ns) a0 = fma(op.ept[i * nu + j], T[i], a0);
      out[j] = in[j] - (a0 + a1);
    }
  }
  __syncwarp();
}

// copy `len` doubles (even) of row r (stride) into dst with 16-byte cp.async, one warp
__device__ __forceinline__ void w_cp(double* dst, const double* src, int len, int lane) {
  for (int k = lane; k < (len >> 1); k += 32) cp16(dst + 2 * k, src + 2 * k);
}
__device__ __forceinline__ void w_issue_bwd(const FastView& f, double* slot, int r, bool kid, int lane) {
  const DevView& d = f.d;
  w_cp(slot, d.Yc + (size_t)r * d.ly, d.ly, lane);
  if (kid) w_cp(slot + d.ly, d.np->R + (size_t)r * d.nu, d.nu, lane);
}
__device__ __forceinline__ void w_issue_fwd(const FastView& f, double* slot, int r, int it, int lane) {
  const DevView& d = f.d;
  const RecOff o = rec_off(d);
  w_cp(slot + o.y, ybuf(d, it) + (size_t)r * d.W, d.W, lane);
  w_cp(slot + o.ym, ybuf(d, it + 2) + (size_t)r * d.W, d.W, lane);
  w_cp(slot + o.lin, d.lin + (size_t)r * d.nu, d.nu, lane);
  w_cp(slot + o.eoff, d.np->e_off + (size_t)r * d.nu, d.nu, lane);
  w_cp(slot + o.g, d.np->g + (size_t)r * d.lx, d.lx, lane);
  w_cp(slot + o.aux, f.aux + (size_t)r * 2, 2, lane);
  if (it > 0) {
    w_cp(slot + o.ua, d.Ua + (size_t)r * d.nu, d.nu, lane);
    w_cp(slot + o.xa, d.Xa + (size_t)r * d.lx, d.lx, lane);
  }
}

// Backward node update. rec = [Yc | R]; sc.L holds the child's lin (if kid);
// sc.WB the child's wbar. Leaves this node's lin in sc.L and wbar in sc.WB.
__device__ __forceinline__ void w_bwd(const FastView& f, const WOps& op, const WScr& sc, const double* rec,
                                      int r, bool kid, bool store_w, int lane) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly;
  if (kid) w_proj(d, op, sc.L, sc.PZ, sc.T, lane);  // PZ = P lin_child
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int j = lane + 32 * k;
    if (j < nt) {
      double wb = kid ? rec[j] + sc.WB[j] : rec[j];
      sc.WB[j] = wb;
      if (store_w) d.wbar[(size_t)r * lx + j] = wb;
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = lane + 32 * k;
    if (j < nu) {
      double bw = 0.0;
      for (int e = op.bcp[j]; e < op.bcp[j + 1]; ++e) bw = fma(sc.WB[op.bcr[e]], op.bcv[e], bw);
      double l = rec[lx + j] + bw;
      if (kid) l = l + (rec[ly + j] + sc.PZ[j]);
      d.lin[(size_t)r * nu + j] = l;
      sc.L[j] = l;
    }
  }
  __syncwarp();
}

// Forward node update + prox. rec = forward record; sc.U / sc.X hold u_anc /
// x_anc on entry and this node's u / x on exit.
__device__ void w_fwd(const FastView& f, const WOps& op, const WScr& sc, double* rec, int r, int it,
                      double beta, double theta, double beta1, bool next, bool store_uv, int lane) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, W = d.W, lx = d.lx;
  const RecOff o = rec_off(d);
  const double a2cp = rec[o.aux];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = lane + 32 * k;
    if (j < nu) sc.L[j] = sc.U[j] - rec[o.lin + j] * a2cp;
  }
  __syncwarp();
  w_proj(d, op, sc.L, sc.PZ, sc.T, lane);  // PZ = P (u_anc - lin / (2c p))
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = lane + 32 * k;
    if (j < nu) {
      double u = rec[o.eoff + j] + sc.PZ[j];
      sc.U[j] = u;
      if (store_uv) d.U[(size_t)r * nu + j] = u;
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int j = lane + 32 * k;
    if (j < nt) {
      double bu = 0.0;
      for (int e = op.brp[j]; e < op.brp[j + 1]; ++e) bu = fma(sc.U[op.brc[e]], op.brv[e], bu);
      double x = (sc.X[j] + bu) + rec[o.g + j];
      sc.X[j] = x;
      if (store_uv) d.X[(size_t)r * lx + j] = x;
    }
  }
  __syncwarp();
  // prox (solver.py:461-475): v = w + gamma Hz, squared distances
  const double gamma = d.gamma, ig = f.inv_gamma;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = lane + 32 * k;
    if (c < W) {
      double y0 = rec[o.y + c];
      double w = dadd(y0, dmul(beta, dsub(y0, rec[o.ym + c])));
      double hz = c < nt ? sc.X[c] : (c < 2 * nt ? sc.X[c - nt] : sc.U[c - 2 * nt]);
      double v = dadd(w, dmul(gamma, hz));
      sc.V[c] = v;
      if (c < 2 * nt) {
        double V = div_by(v, gamma, ig);
        double df = c < nt ? dsub(V, np_clip(V, op.xmin[c], op.xmax[c])) : dsub(V, np_max(V, op.xsafe[c - nt]));
        sc.D2[c] = dmul(df, df);
      }
    }
  }
  __syncwarp();
  {
    // lanes 0-7: slot 1, lanes 8-15: slot 2 (numpy pairwise order)
    const int lane8 = lane & 7, slot = (lane >> 3) & 1;
    const unsigned mask = 0xffu << (lane & 24);
    double ssum = pw_group8(sc.D2 + slot * nt, nt, lane8, mask);
    if (lane < 16 && lane8 == 0) {
      double dist = __dsqrt_rn(ssum);
      double thr = dmul(ig, slot ? d.w_s : d.w_x);
      sc.S[slot] = dist > 0.0 ? np_min(1.0, div_exact(thr, dist)) : 0.0;
    }
  }
  __syncwarp();
  const double st1 = sc.S[0], st2 = sc.S[1];
  double* yn = ybuf_w(d, it + 1);
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = lane + 32 * k;
    if (c < W) {
      double v = sc.V[c];
      double V = div_by(v, gamma, ig);
      double O;
      if (c < nt) {
        O = dsub(V, dmul(st1, dsub(V, np_clip(V, op.xmin[c], op.xmax[c]))));
      } else if (c < 2 * nt) {
        O = dsub(V, dmul(st2, dsub(V, np_max(V, op.xsafe[c - nt]))));
      } else {
        O = np_clip(V, op.umin[c - 2 * nt], op.umax[c - 2 * nt]);
      }
      double yv = dsub(v, dmul(gamma, O));
      yn[(size_t)r * W + c] = yv;
      sc.V[c] = yv;
      bad |= !isfinite(yv);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(d.bad_nu, it);
  const double om = dsub(1.0, theta);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = lane + 32 * k;
    if (j < nu) {
      double u = sc.U[j];
      d.Ua[(size_t)r * nu + j] = it == 0 ? u : dadd(dmul(rec[o.ua + j], om), dmul(theta, u));
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int j = lane + 32 * k;
    if (j < nt) {
      double x = sc.X[j];
      d.Xa[(size_t)r * lx + j] = it == 0 ? x : dadd(dmul(rec[o.xa + j], om), dmul(theta, x));
    }
  }
  __syncwarp();
  if (next) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = lane + 32 * k;
      if (j < nt) {
        double p1 = sc.V[j], p2 = sc.V[nt + j];
        double w1 = dadd(p1, dmul(beta1, dsub(p1, rec[o.y + j])));
        double w2 = dadd(p2, dmul(beta1, dsub(p2, rec[o.y + nt + j])));
        d.Yc[(size_t)r * d.ly + j] = dadd(w1, w2);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = lane + 32 * k;
      if (j < nu) {
        double p3 = sc.V[2 * nt + j];
        d.Yc[(size_t)r * d.ly + lx + j] = dadd(p3, dmul(beta1, dsub(p3, rec[o.y + 2 * nt + j])));
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(FW_THREADS, 1) k_apg_warp(FastView f, const int* __restrict__ off_dev) {
  cg::grid_group grid = cg::this_grid();
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, ns = d.ns, H = d.H, lx = d.lx;
  const int bnnz = f.b_nnz;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int G = gridDim.x;
  const int TW = G * FW_WARPS;
  const int gw = wid * G + blockIdx.x;  // global warp id: spread over SMs first
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* slots_all = reinterpret_cast<double*>(smem_raw);        // FW_WARPS * nrow * rec
  double* scr_all = slots_all + (size_t)FW_WARPS * f.nrow * f.rec;  // FW_WARPS * FW_SCR
  double* s_bnd = scr_all + FW_WARPS * FW_SCR;                     // 3nt + 2nu
  double* s_ept = s_bnd + 3 * nt + 2 * nu;                         // ns*nu (E^+ transposed)
  double* s_ev = s_ept + nu * ns;
  double* s_bcv = s_ev + f.e_nnz;
  double* s_brv = s_bcv + bnnz;
  int* s_eptr = reinterpret_cast<int*>(s_brv + bnnz);
  int* s_ecol = s_eptr + ns + 1;
  int* s_bcp = s_ecol + f.e_nnz;
  int* s_bcr = s_bcp + nu + 1;
  int* s_brp = s_bcr + bnnz;
  int* s_brc = s_brp + nt + 1;
  int* offs = s_brc + bnnz;  // H+1

  for (int i = threadIdx.x; i <= H; i += blockDim.x) offs[i] = off_dev[i];
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
    int j = i / ns, k = i - j * ns;  // e_pinv is nu x ns; store transposed
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
  __syncthreads();
  const WOps op{s_ept, s_eptr, s_ecol, s_ev, s_bcp, s_bcr, s_bcv, s_brp, s_brc, s_brv,
                s_bnd, s_bnd + nt, s_bnd + 2 * nt, s_bnd + 3 * nt, s_bnd + 3 * nt + nu};
  const WScr sc = wscr(scr_all + wid * FW_SCR);
  double* slots = slots_all + (size_t)wid * f.nrow * f.rec;

  const int it0 = *d.iter;
  const int kstar = f.kstar, nst = H - kstar;
  // chains of this warp: gw, gw + TW, ...
  const int nmine = gw < f.nchain ? (f.nchain - gw + TW - 1) / TW : 0;
  const int nsteps = nmine * nst;
  const int depth = f.nrow - 1;
  auto step_node = [&](int k, bool backward, int& s) {
    int ci = k / nst, t = k - ci * nst;
    s = backward ? (H - 1 - t) : (kstar + t);
    return f.chain_node[(size_t)(s - kstar) * f.nchain + gw + ci * TW];
  };

  for (int il = 0; il < f.count; ++il) {
    const int it = it0 + il;
    const double beta = d.beta[it], theta = d.theta[it];
    const bool has_next = it + 1 < f.max_iter;
    const double beta1 = has_next ? d.beta[it + 1] : 0.0;
    const bool last = il == f.count - 1;

    // ---------------- A: chain backward ----------------
    for (int k = 0; k < depth; ++k) {
      if (k < nsteps) {
        int s;
        int r = step_node(k, true, s);
        w_issue_bwd(f, slots + (k % f.nrow) * f.rec, r, s < H - 1, lane);
      }
      cp_commit();
    }
    for (int k = 0; k < nsteps; ++k) {
      {
        const int kp = k + depth;
        if (kp < nsteps) {
          int s;
          int r = step_node(kp, true, s);
          w_issue_bwd(f, slots + (kp % f.nrow) * f.rec, r, s < H - 1, lane);
        }
        cp_commit();
      }
      int s;
      const int r = step_node(k, true, s);
      cp_wait_dyn(depth);
      __syncwarp();
      w_bwd(f, op, sc, slots + (k % f.nrow) * f.rec, r, s < H - 1, s == kstar, lane);
    }
    cp_wait<0>();
    grid.sync();

    // ---------------- B: branching backward, one node per warp ----------------
    for (int s = kstar - 1; s >= 0; --s) {
      const int cnt = offs[s + 1] - offs[s];
      for (int t = gw; t < cnt; t += TW) {
        const int r = offs[s] + t;
        w_issue_bwd(f, slots, r, true, lane);
        cp_commit();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int j = lane + 32 * k;
          if (j < nt) {
            double cs = 0.0;
            for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) cs += d.wbar[(size_t)d.cidx[e] * lx + j];
            sc.WB[j] = cs;
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = lane + 32 * k;
          if (j < nu) {
            double ls = 0.0;
            for (int e = d.cptr[r]; e < d.cptr[r + 1]; ++e) ls += d.lin[(size_t)d.cidx[e] * nu + j];
            sc.L[j] = ls;
          }
        }
        cp_wait<0>();
        __syncwarp();
        w_bwd(f, op, sc, slots, r, true, true, lane);
      }
      grid.sync();
    }

    // ---------------- C: branching forward + prox, one node per warp ----------------
    for (int s = 0; s < kstar; ++s) {
      const int cnt = offs[s + 1] - offs[s];
      for (int t = gw; t < cnt; t += TW) {
        const int r = offs[s] + t;
        w_issue_fwd(f, slots, r, it, lane);
        cp_commit();
        const int a = d.anc[r];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = lane + 32 * k;
          if (j < nu) sc.U[j] = a < 0 ? d.q[j] : d.U[(size_t)a * nu + j];
          if (k < 2 && j < nt) sc.X[j] = a < 0 ? d.p[j] : d.X[(size_t)a * lx + j];
        }
        cp_wait<0>();
        __syncwarp();
        w_fwd(f, op, sc, slots, r, it, beta, theta, beta1, has_next, true, lane);
      }
      grid.sync();
    }

    // ---------------- D: chain forward + prox ----------------
    for (int k = 0; k < depth; ++k) {
      if (k < nsteps) {
        int s;
        int r = step_node(k, false, s);
        w_issue_fwd(f, slots + (k % f.nrow) * f.rec, r, it, lane);
      }
      cp_commit();
    }
    for (int k = 0; k < nsteps; ++k) {
      {
        const int kp = k + depth;
        if (kp < nsteps) {
          int s;
          int r = step_node(kp, false, s);
          w_issue_fwd(f, slots + (kp % f.nrow) * f.rec, r, it, lane);
        }
        cp_commit();
      }
      int s;
      const int r = step_node(k, false, s);
      if (s == kstar) {  // chain top: ancestor state from the branching region
        const int a = d.anc[r];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int j = lane + 32 * kk;
          if (j < nu) sc.U[j] = a < 0 ? d.q[j] : d.U[(size_t)a * nu + j];
          if (kk < 2 && j < nt) sc.X[j] = a < 0 ? d.p[j] : d.X[(size_t)a * lx + j];
        }
      }
      cp_wait_dyn(depth);
      __syncwarp();
      w_fwd(f, op, sc, slots + (k % f.nrow) * f.rec, r, it, beta, theta, beta1, has_next, last && f.store_uv,
            lane);
    }
    cp_wait<0>();
    __threadfence();
    __syncwarp();
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *d.iter = it0 + f.count;
}

}  // namespace wmpc
