// wmpc_dp.cuh — one-kernel APG iteration for trees with many chains
// (k_chain_dp): down pass + Moreau prox of iteration it + up pass of it + 1,
// one warp per chain, rows streamed into shared memory by TMA bulk copies.
//
// The graph path (wmpc_scan.cuh) runs an iteration as up -> branch groups ->
// down -> prox, and moves U, X (down -> prox) and the collapsed dual Yc
// (prox -> next up) through HBM: 2.8 KB per node per iteration on top of the
// 10.0 KB the algorithm needs. Here the down pass walks each chain BOTTOM-UP,
// so the prox's output of a row (the next collapsed dual) feeds the next
// iteration's suffix scans (the up pass) in registers, and u, x feed the prox
// in registers: per chain row the kernel reads L, ut, g, y, y_prev, Ua, Xa and
// writes L', y_next, Ua, Xa — 11.9 KB per node, with no U, X or Yc round trip.
//
// Walking bottom-up needs the down pass's prefix sums (solver.py:276-287) at
// the chain's bottom row first. With N chain rows t = 0..N-1 below kb
// ancestors (root path rows m = 0..kb-1, then kb + t):
//   ls_t = LS_anc + sum_{t' <= t} L_t',     u_t = ut_t - P ls_t,
//   x_t  = x_a + sum_{t' <= t} (B u_t' + g_t'),
// so with the chain aggregates of the up pass LSc = sum_t L_t and
// LWc = sum_t (N - t) L_t (= sum_t of the prefix sums), and the per-solve
// constants SUT = sum_t ut_t, SG = sum_t g_t:
//   ls_{N-1} = LS_anc + LSc,
//   x_{N-1}  = x_a + B (SUT - P (N LS_anc + LWc)) + SG,
// and upwards ls_{t-1} = ls_t - L_t, x_{t-1} = (x_t - g_t) - B u_t.
// The same quantities as the reference's recursion in real arithmetic; the
// rounding differs (parity is checked against the reference at 1e-8, the
// north_star's tolerance, not bit-for-bit against the unfused kernels).
//
// Ancestor rows (branching stages) are walked top-down first, as in
// k_chain_down_r; the one chain that owns a branching row (cown, balanced per
// warp on the host) runs its prox and writes its Yc for the branch-group
// kernels of the next iteration. The kernel is persistent over chains: warp w
// handles chains w, w + NW, w + 2 NW, ...
//
// Per warp, a ring of DP_D stages [L | ut | g | y | y_prev | Ua | Xa] is filled
// by cp.async.bulk (one elected lane, one mbarrier per stage, expect_tx); a
// stage is re-armed as soon as the warp has read it into registers, so loads
// run DP_D - 1 rows ahead. fp32 mode: L, ut, g, Yc are fp32 (rows not 16-byte
// multiples, so those three are read with plain loads); the prox operands
// stay fp64 and go through the ring.
#pragma once
#include "wmpc_chainw.cuh"

namespace wmpc {

#ifndef DP_D_N
#define DP_D_N 3
#endif
constexpr int DP_D = DP_D_N;   // ring stages per warp
constexpr int DP_BND = 448;    // bounds table: xmin 64 | xmax 64 | xsafe 64 | umin 128 | umax 128
constexpr int DP_XCH = 352;    // per-warp exchange vectors (TG): wb 64 | zb 128 | ub 128 | tb 32
constexpr int DP_VSLOTS = 22;  // operator value table: bc 8 | ec 4 | kr 4 | br 6 (x 32 lanes)

struct DpArgs {
  void* agg;     // nchain x (3 nu + lx), TG: [LSc | LWc | SUT | SG]
  int cpw;       // chains per warp
  int mode;      // 0: iteration, 1: up pass only (Yc from memory: warm start)
};

__host__ __device__ inline int dp_stage(int nt, int nu, int lx) { return 3 * nu + 2 * lx + 2 * (2 * nt + nu); }
__host__ __device__ inline int dp_agg_w(int nu, int lx) { return 3 * nu + lx; }
template <typename TG>
__host__ __device__ inline size_t dp_smem(int wpc, int nt, int nu, int lx) {
  return sizeof(double) * (DP_BND + (size_t)wpc * DP_D * dp_stage(nt, nu, lx)) + 8 * (size_t)wpc * DP_D +
         sizeof(TG) * (size_t)wpc * DP_XCH + sizeof(double) * (size_t)wpc * 128 + 8 * DP_VSLOTS * 32 + 16;
}

__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{.reg .pred p; DPW%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra DPW%=;}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on mbarrier b (bytes % 16 == 0, both 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

template <typename TG>
__device__ __forceinline__ typename V2T<TG>::T ld2s(const TG* p) {  // shared or global, aligned pair
  return *reinterpret_cast<const typename V2T<TG>::T*>(p);
}

template <int WE, typename TG, bool VF>
__global__ void __launch_bounds__(256, 1) k_chain_dp(FastView f, DpArgs A) {
  using TB = std::conditional_t<VF && sizeof(TG) == 8, float, TG>;  // B, E value storage
  constexpr bool TMA_DG = sizeof(TG) == 8;  // L, ut, g, aggregates through the ring (fp64 rows are 16-byte multiples)
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly, W = d.W;
  const int kb = f.kstar, H = d.H, N = H - kb, S = H + 1;
  const int wpc = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int STG = dp_stage(nt, nu, lx), AW = dp_agg_w(nu, lx);
  const int oL = 0, oB = nu, oG = 2 * nu, oY = 2 * nu + lx, oYm = oY + W, oUa = oYm + W, oXa = oUa + nu;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* bnd = reinterpret_cast<double*>(smem_raw);
  double* ring_all = bnd + DP_BND;
  double* ring = ring_all + (size_t)warp * DP_D * STG;
  uint64_t* mbar_all = reinterpret_cast<uint64_t*>(ring_all + (size_t)wpc * DP_D * STG);
  uint64_t* mbar = mbar_all + warp * DP_D;
  TG* xch_all = reinterpret_cast<TG*>(mbar_all + wpc * DP_D);
  TG* wb = xch_all + (size_t)warp * DP_XCH;  // 64
  TG* zb = wb + 64;                          // 128
  TG* ub = zb + 128;                         // 128
  TG* tb = ub + 128;                         // 32
  double* sd2_all = reinterpret_cast<double*>(xch_all + (size_t)wpc * DP_XCH);
  double* sd2 = sd2_all + warp * 128;
  unsigned char* vtab = reinterpret_cast<unsigned char*>(sd2_all + wpc * 128);
  const GA<TG> G = ga<TG>(f);
  const int l2 = 2 * lane;
  const bool ok0 = l2 < nu, ok1 = 64 + l2 < nu, okx = l2 < nt, okx2 = l2 + 1 < nt;
  const unsigned o1 = ok1 ? 64 + l2 : 0;
  const unsigned nchain = f.nchain, nbr = f.n_branch;
  // ---- prologue (overlaps the predecessor under PDL): bounds, operators, barriers
  for (int i = threadIdx.x; i < DP_BND; i += blockDim.x) {
    double v = 0.0;
    if (i < 64) v = i < nt ? d.xmin[i] : 0.0;
    else if (i < 128) v = i - 64 < nt ? d.xmax[i - 64] : 0.0;
    else if (i < 192) v = i - 128 < nt ? d.xsafe[i - 128] : 0.0;
    else if (i < 320) v = i - 192 < nu ? d.umin[i - 192] : 0.0;
    else v = i - 320 < nu ? d.umax[i - 320] : 0.0;
    bnd[i] = v;
  }
  int voff = 0;
  (void)voff;
  EllRB<EllW<WE>::BC, TG, TB> bc[4];
  EllRE<EllW<WE>::EC, TG, TB> ec[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = cw_ku(lane, q);
    bc[q] = cw_bind<EllRB<EllW<WE>::BC, TG, TB>, TB>(ell_own<EllW<WE>::BC, TG>(f, own_bc(d, k), k < nu), wb, vtab,
                                                      voff, lane, warp == 0);
    ec[q] = cw_bind<EllRE<EllW<WE>::EC, TG, TB>, TB>(ell_own<EllW<WE>::EC, TG>(f, own_ec(d, k), k < nu), tb, vtab,
                                                      voff, lane, warp == 0);
  }
  const EllRK<EllW<WE>::KR, TG> kr = cw_bind<EllRK<EllW<WE>::KR, TG>, TG>(
      ell_own<EllW<WE>::KR, TG>(f, own_kr(d, lane), lane < d.ns), zb, vtab, voff, lane, warp == 0);
  EllRB<EllW<WE>::BR, TG, TB> br[2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
    br[h] = cw_bind<EllRB<EllW<WE>::BR, TG, TB>, TB>(ell_own<EllW<WE>::BR, TG>(f, own_br(d, l2 + h), l2 + h < nt),
                                                      ub, vtab, voff, lane, warp == 0);
  if (lane == 0) {
    for (int s = 0; s < DP_D; ++s) mbar_init(mbar + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // L of the branching rows comes from the last group kernel; iter from the first
  pdl_trigger();
  const bool up_only = A.mode == 1;
  const ProxIt P = up_only ? ProxIt{} : prox_it(f);
  const bool next = up_only || P.next;  // the up pass of the next iteration runs
  const bool store = !up_only && P.it == *f.store_it;
  const double* yb = up_only ? nullptr : ybuf(d, P.it);
  const double* ymb = up_only ? nullptr : ybuf(d, P.it + 2);
  double* ynb = up_only ? nullptr : ybuf_w(d, P.it + 1);
  TG* agg = reinterpret_cast<TG*>(A.agg);
  const int gw = blockIdx.x * wpc + warp, nw = gridDim.x * wpc;
  const int steps = A.cpw * S;
  // ---- the ring: step i = (chain slot i / S, step s = i % S): s < kb ancestor
  // row s, s == kb chain aggregates, s > kb chain row t = N - 1 - (s - kb - 1)
  auto issue = [&](int i) {
    if (lane != 0 || i >= steps || up_only) return;
    const int ci = gw + (i / S) * nw;
    if (ci >= (int)nchain) return;
    const int s = i % S;
    double* st = ring + (i % DP_D) * STG;
    uint64_t* b = mbar + (i % DP_D);
    unsigned r;
    bool dg = TMA_DG, px;
    if (s < kb) {
      r = (unsigned)f.cpath[(size_t)ci * kb + s];
      px = (f.cown[ci] >> s) & 1u;
    } else if (s == kb) {
      if (TMA_DG) {
        mbar_expect(b, (unsigned)(AW * 8));
        bulk_g2s(st, reinterpret_cast<const double*>(agg) + (size_t)ci * AW, AW * 8, b);
      } else {
        mbar_expect(b, 0u);
      }
      return;
    } else {
      r = nbr + (unsigned)(N - 1 - (s - kb - 1)) * nchain + (unsigned)ci;
      px = true;
    }
    const unsigned bytes = (dg ? (unsigned)(2 * nu + lx) * 8u : 0u) + (px ? (unsigned)(2 * W + nu + lx) * 8u : 0u);
    mbar_expect(b, bytes);
    if (dg) {
      bulk_g2s(st + oL, reinterpret_cast<const double*>(G.Lb) + (size_t)r * nu, nu * 8, b);
      bulk_g2s(st + oB, reinterpret_cast<const double*>(f.ut) + (size_t)r * nu, nu * 8, b);
      bulk_g2s(st + oG, reinterpret_cast<const double*>(G.g) + (size_t)r * lx, lx * 8, b);
    }
    if (px) {
      bulk_g2s(st + oY, yb + (size_t)r * W, W * 8, b);
      bulk_g2s(st + oYm, ymb + (size_t)r * W, W * 8, b);
      bulk_g2s(st + oUa, d.Ua + (size_t)r * nu, nu * 8, b);
      bulk_g2s(st + oXa, d.Xa + (size_t)r * lx, lx * 8, b);
    }
  };
  auto take = [&](int i) -> const double* {  // wait for step i's stage
    mbar_wait(mbar + (i % DP_D), (unsigned)((i / DP_D) & 1));
    return ring + (i % DP_D) * STG;
  };
  auto release = [&](int i) {  // the warp has read step i's stage: re-arm it with step i + DP_D
    __syncwarp();
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(i + DP_D);
  };
  for (int i = 0; i < DP_D; ++i) issue(i);
  // ---- the projector and operator products through the exchange vectors
  auto proj_neg = [&](const TG (&v)[4], const TG (&base)[4], TG (&out)[4]) {  // out = base + P(-v)
    TG z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) z[q] = -v[q];
    st2(zb + l2, z[0], z[1]);
    st2(zb + 64 + l2, z[2], z[3]);
    __syncwarp();
    tb[lane] = CW_DOT(kr);  // zero past ns
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = base[q] + (z[q] - CW_DOT(ec[q]));
  };
  auto bmul = [&](const TG (&u)[4], TG (&bu)[2]) {  // bu = B u (rows l2, l2 + 1)
    st2(ub + l2, u[0], u[1]);
    st2(ub + 64 + l2, u[2], u[3]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) bu[h] = CW_DOT(br[h]);
  };
  bool bad = false;
  // Moreau prox of one row (prox_x_warp / prox_u_warp arithmetic, bit-exact
  // with numpy per element), ergodic averages; returns the next collapsed dual
  auto prox = [&](const double* st, unsigned r, const TG (&u)[4], const TG (&x)[2], TG (&yx)[2], TG (&yu)[4]) {
    const double gamma = P.gamma, ig = P.ig;
    double* yn = ynb + (size_t)r * W;
    double xv[2] = {(double)x[0], (double)x[1]};
    double y1[2], y2[2], m1[2], m2[2], xa[2], V1[2], V2[2], v1[2], v2[2], c1[2], c2[2];
    {
      const double2 a = ld2s(st + oY + l2), b = ld2s(st + oYm + l2), c = ld2s(st + oXa + l2);
      y1[0] = a.x; y1[1] = a.y; m1[0] = b.x; m1[1] = b.y; xa[0] = c.x; xa[1] = c.y;
      y2[0] = st[oY + nt + l2]; y2[1] = st[oY + nt + l2 + 1];
      m2[0] = st[oYm + nt + l2]; m2[1] = st[oYm + nt + l2 + 1];
    }
    double xan[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = l2 + h;
      const bool ok = j < nt;
      xan[h] = P.it == 0 ? xv[h] : dadd(dmul(xa[h], P.om), dmul(P.theta, xv[h]));
      const double gx = dmul(gamma, xv[h]);
      v1[h] = dadd(dadd(y1[h], dmul(P.beta, dsub(y1[h], m1[h]))), gx);
      v2[h] = dadd(dadd(y2[h], dmul(P.beta, dsub(y2[h], m2[h]))), gx);
      V1[h] = div_by(v1[h], gamma, ig);
      V2[h] = div_by(v2[h], gamma, ig);
      c1[h] = np_clip(V1[h], bnd[j], bnd[64 + j]);
      c2[h] = np_max(V2[h], bnd[128 + j]);
      if (ok) {
        const double df1 = dsub(V1[h], c1[h]), df2 = dsub(V2[h], c2[h]);
        sd2[j] = dmul(df1, df1);
        sd2[64 + j] = dmul(df2, df2);
      }
    }
    double* xap = d.Xa + (size_t)r * lx + l2;
    if (okx2) st2(xap, xan[0], xan[1]);
    else if (okx) xap[0] = xan[0];
    // the u part while the norms' operands settle
    double y3[4], m3[4], ua[4];
    {
      const double2 a0 = ld2s(st + oY + 2 * nt + l2), a1 = ld2s(st + oY + 2 * nt + o1);
      const double2 b0 = ld2s(st + oYm + 2 * nt + l2), b1 = ld2s(st + oYm + 2 * nt + o1);
      const double2 c0 = ld2s(st + oUa + l2), c1v = ld2s(st + oUa + o1);
      y3[0] = a0.x; y3[1] = a0.y; y3[2] = a1.x; y3[3] = a1.y;
      m3[0] = b0.x; m3[1] = b0.y; m3[2] = b1.x; m3[3] = b1.y;
      ua[0] = c0.x; ua[1] = c0.y; ua[2] = c1v.x; ua[3] = c1v.y;
    }
    double uan[4], p3[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = cw_ku(lane, q);
      const double uq = (double)u[q];
      uan[q] = P.it == 0 ? uq : dadd(dmul(ua[q], P.om), dmul(P.theta, uq));
      const double v3 = dadd(dadd(y3[q], dmul(P.beta, dsub(y3[q], m3[q]))), dmul(gamma, uq));
      const double V3 = div_by(v3, gamma, ig);
      const int kk = k < nu ? k : 0;
      p3[q] = dsub(v3, dmul(gamma, np_clip(V3, bnd[192 + kk], bnd[320 + kk])));
      if (k < nu) bad |= !isfinite(p3[q]);
      yu[q] = next ? (TG)dadd(p3[q], dmul(P.beta1, dsub(p3[q], y3[q]))) : TG(0);
      if (k >= nu) yu[q] = TG(0);
    }
    if (ok0) {
      st2(d.Ua + (size_t)r * nu + l2, uan[0], uan[1]);
      st2(yn + 2 * nt + l2, p3[0], p3[1]);
    }
    if (ok1) {
      st2(d.Ua + (size_t)r * nu + 64 + l2, uan[2], uan[3]);
      st2(yn + 2 * nt + 64 + l2, p3[2], p3[3]);
    }
    __syncwarp();
    double stv = 0.0;
    if (lane < 16) {
      const int slot = lane >> 3;
      const double ssum = pw_group8(sd2 + 64 * slot, nt, lane & 7, 0xffu << (lane & 8));
      if ((lane & 7) == 0) {
        const double dist = __dsqrt_rn(ssum);
        const double thr = dmul(ig, slot ? d.w_s : d.w_x);  // prox parameter RN(1/gamma) (solver.py:571)
        stv = dist > 0.0 ? np_min(1.0, div_exact(thr, dist)) : 0.0;
      }
    }
    const double st1 = __shfl_sync(0xffffffffu, stv, 0), st2v = __shfl_sync(0xffffffffu, stv, 8);
    double p1[2], p2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = l2 + h;
      const double O1 = dsub(V1[h], dmul(st1, dsub(V1[h], c1[h])));
      const double O2 = dsub(V2[h], dmul(st2v, dsub(V2[h], c2[h])));
      p1[h] = dsub(v1[h], dmul(gamma, O1));
      p2[h] = dsub(v2[h], dmul(gamma, O2));
      if (j < nt) bad |= !isfinite(p1[h]) || !isfinite(p2[h]);
      yx[h] = (next && j < nt) ? (TG)dadd(dadd(p1[h], dmul(P.beta1, dsub(p1[h], y1[h]))),
                                          dadd(p2[h], dmul(P.beta1, dsub(p2[h], y2[h]))))
                               : TG(0);
    }
    if (okx2) st2(yn + l2, p1[0], p1[1]);
    else if (okx) yn[l2] = p1[0];
    if (okx) yn[nt + l2] = p2[0];
    if (okx2) yn[nt + l2 + 1] = p2[1];
  };
  auto store_ux = [&](unsigned r, const TG (&u)[4], const TG (&x)[2]) {
    TG* Up = G.U + (size_t)r * nu;
    if (ok0) st2(Up + l2, u[0], u[1]);
    if (ok1) st2(Up + 64 + l2, u[2], u[3]);
    TG* Xp = G.X + (size_t)r * lx + l2;
    if (okx2) st2(Xp, x[0], x[1]);
    else if (okx) Xp[0] = x[0];
  };
  auto row_dg = [&](const double* st, unsigned r, TG (&L)[4], TG (&b)[4], TG (&g)[2]) {
    if constexpr (TMA_DG) {
      const double2 a0 = ld2s(st + oL + l2), a1 = ld2s(st + oL + o1);
      const double2 b0 = ld2s(st + oB + l2), b1 = ld2s(st + oB + o1);
      const double2 g0 = ld2s(st + oG + l2);
      L[0] = (TG)a0.x; L[1] = (TG)a0.y; L[2] = (TG)a1.x; L[3] = (TG)a1.y;
      b[0] = (TG)b0.x; b[1] = (TG)b0.y; b[2] = (TG)b1.x; b[3] = (TG)b1.y;
      g[0] = (TG)g0.x; g[1] = (TG)g0.y;
    } else {
      const TG* base = sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32;
      const auto a0 = ldg2_if(G.Lb + (size_t)r * nu + l2, true), a1 = ldg2_if(G.Lb + (size_t)r * nu + o1, true);
      const auto b0 = ldg2_if(base + (size_t)r * nu + l2, true), b1 = ldg2_if(base + (size_t)r * nu + o1, true);
      const auto g0 = ldg2_if(G.g + (size_t)r * lx + l2, true);
      L[0] = a0.x; L[1] = a0.y; L[2] = a1.x; L[3] = a1.y;
      b[0] = b0.x; b[1] = b0.y; b[2] = b1.x; b[3] = b1.y;
      g[0] = g0.x; g[1] = g0.y;
    }
    if (!ok0) L[0] = L[1] = b[0] = b[1] = TG(0);
    if (!ok1) L[2] = L[3] = b[2] = b[3] = TG(0);
    if (!okx) g[0] = TG(0);
    if (!okx2) g[1] = TG(0);
  };
  int i = 0;  // ring step
  for (int cs = 0; cs < A.cpw; ++cs) {
    const int ci = gw + cs * nw;
    if (ci >= (int)nchain) break;
    const unsigned r_top = nbr + (unsigned)ci;
    TG ls[4] = {0, 0, 0, 0}, xs[2];
    if (!up_only) {
      // ---- ancestors, top-down (k_chain_down_r arithmetic)
      const unsigned own = kb > 0 ? f.cown[ci] : 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) xs[h] = l2 + h < nt ? (TG)d.p[l2 + h] : TG(0);
      for (int m = 0; m < kb; ++m, ++i) {
        const unsigned r = (unsigned)f.cpath[(size_t)ci * kb + m];
        const double* st = take(i);
        TG L[4], b[4], g[2];
        row_dg(st, r, L, b, g);
        const bool mine = (own >> m) & 1u;
        if (!mine) release(i);
#pragma unroll
        for (int q = 0; q < 4; ++q) ls[q] = m == 0 ? L[q] : ls[q] + L[q];
        TG u[4], bu[2];
        proj_neg(ls, b, u);
        bmul(u, bu);
#pragma unroll
        for (int h = 0; h < 2; ++h) xs[h] = (xs[h] + bu[h]) + g[h];
        if (mine) {
          TG yx[2], yu[4];
          prox(st, r, u, xs, yx, yu);
          release(i);
          if (next) {
            TG* yc = G.Yc + (size_t)r * ly;
            if (okx2) st2(yc + l2, yx[0], yx[1]);
            else if (okx) yc[l2] = yx[0];
            if (ok0) st2(yc + lx + l2, yu[0], yu[1]);
            if (ok1) st2(yc + lx + 64 + l2, yu[2], yu[3]);
          }
          if (store) store_ux(r, u, xs);
        }
      }
      // ---- chain aggregates: the bottom row's prefix sums
      {
        const double* st = take(i);
        TG LS[4], LW[4], SU[4], SG[2];
        if constexpr (TMA_DG) {
          const double* a = st;
          const double2 s0 = ld2s(a + l2), s1 = ld2s(a + o1), w0 = ld2s(a + nu + l2), w1 = ld2s(a + nu + o1);
          const double2 u0 = ld2s(a + 2 * nu + l2), u1 = ld2s(a + 2 * nu + o1), g0 = ld2s(a + 3 * nu + l2);
          LS[0] = s0.x; LS[1] = s0.y; LS[2] = s1.x; LS[3] = s1.y;
          LW[0] = w0.x; LW[1] = w0.y; LW[2] = w1.x; LW[3] = w1.y;
          SU[0] = u0.x; SU[1] = u0.y; SU[2] = u1.x; SU[3] = u1.y;
          SG[0] = g0.x; SG[1] = g0.y;
        } else {
          const TG* a = agg + (size_t)ci * AW;
          const auto s0 = ld2s(a + l2), s1 = ld2s(a + o1), w0 = ld2s(a + nu + l2), w1 = ld2s(a + nu + o1);
          const auto u0 = ld2s(a + 2 * nu + l2), u1 = ld2s(a + 2 * nu + o1), g0 = ld2s(a + 3 * nu + l2);
          LS[0] = s0.x; LS[1] = s0.y; LS[2] = s1.x; LS[3] = s1.y;
          LW[0] = w0.x; LW[1] = w0.y; LW[2] = w1.x; LW[3] = w1.y;
          SU[0] = u0.x; SU[1] = u0.y; SU[2] = u1.x; SU[3] = u1.y;
          SG[0] = g0.x; SG[1] = g0.y;
        }
        release(i);
        ++i;
        TG V[4], w[4], bw[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) V[q] = fma((TG)N, ls[q], LW[q]);
        proj_neg(V, SU, w);  // sum_t u_t
        bmul(w, bw);
#pragma unroll
        for (int h = 0; h < 2; ++h) xs[h] = (xs[h] + bw[h]) + SG[h];  // x_{N-1}
#pragma unroll
        for (int q = 0; q < 4; ++q) ls[q] = ls[q] + LS[q];  // ls_{N-1}
      }
    }
    // ---- chain rows, bottom-up: down of it, prox of it, up of it + 1
    TG wbr[2] = {0, 0}, acc[4] = {0, 0, 0, 0}, LSn[4] = {0, 0, 0, 0}, LWn[4] = {0, 0, 0, 0};
    for (int t = N - 1; t >= 0; --t) {
      const unsigned r = nbr + (unsigned)t * nchain + (unsigned)ci;
      const bool bottom = t == N - 1;
      TG yx[2], yu[4];
      if (!up_only) {
        const double* st = take(i);
        TG L[4], b[4], g[2], u[4];
        row_dg(st, r, L, b, g);
        proj_neg(ls, b, u);
        prox(st, r, u, xs, yx, yu);
        release(i);
        ++i;
        if (store) store_ux(r, u, xs);
        if (t > 0) {  // x and ls of the row above
          TG bu[2];
          bmul(u, bu);
#pragma unroll
          for (int h = 0; h < 2; ++h) xs[h] = (xs[h] - g[h]) - bu[h];
#pragma unroll
          for (int q = 0; q < 4; ++q) ls[q] = ls[q] - L[q];
        }
      } else {
        const TG* yc = G.Yc + (size_t)r * ly;
        const auto a = ldg2_if(yc + l2, okx), b0 = ldg2_if(yc + lx + l2, ok0), b1 = ldg2_if(yc + lx + o1, ok1);
        yx[0] = a.x; yx[1] = a.y;
        yu[0] = b0.x; yu[1] = b0.y; yu[2] = b1.x; yu[3] = b1.y;
      }
      if (!next) continue;
      // up pass of the next iteration (k_chain_up_r arithmetic, R-free)
#pragma unroll
      for (int h = 0; h < 2; ++h) wbr[h] = bottom ? yx[h] : yx[h] + wbr[h];
      st2(wb + l2, wbr[0], wbr[1]);
      __syncwarp();
      TG a[4], Sv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = yu[q] + CW_DOT(bc[q]);
        Sv[q] = acc[q];
        acc[q] = bottom ? a[q] : a[q] + acc[q];
      }
      TG l[4];
      if (!bottom) {
        st2(zb + l2, Sv[0], Sv[1]);
        st2(zb + 64 + l2, Sv[2], Sv[3]);
        __syncwarp();
        tb[lane] = CW_DOT(kr);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) l[q] = a[q] + (Sv[q] - CW_DOT(ec[q]));
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) l[q] = a[q];
      }
      const TG ax = G.aux[(size_t)r * 2];
      const TG wt = (TG)(N - t);
      TG Ln[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Ln[q] = l[q] * ax;
        LSn[q] = LSn[q] + Ln[q];
        LWn[q] = fma(wt, Ln[q], LWn[q]);
      }
      TG* Lp = G.Lb + (size_t)r * nu;
      if (ok0) st2(Lp + l2, Ln[0], Ln[1]);
      if (ok1) st2(Lp + 64 + l2, Ln[2], Ln[3]);
      __syncwarp();  // wb / zb / tb are rewritten by the next row
    }
    if (next) {  // chain totals for the branch groups, aggregates for the next iteration
      if (okx) G.wbar[(size_t)r_top * lx + l2] = wbr[0];
      if (okx2) G.wbar[(size_t)r_top * lx + l2 + 1] = wbr[1];
      if (ok0) st2(G.Asub + (size_t)r_top * nu + l2, acc[0], acc[1]);
      if (ok1) st2(G.Asub + (size_t)r_top * nu + 64 + l2, acc[2], acc[3]);
      TG* a = agg + (size_t)ci * AW;
      if (ok0) {
        st2(a + l2, LSn[0], LSn[1]);
        st2(a + nu + l2, LWn[0], LWn[1]);
      }
      if (ok1) {
        st2(a + 64 + l2, LSn[2], LSn[3]);
        st2(a + nu + 64 + l2, LWn[2], LWn[3]);
      }
    }
  }
  if (!up_only && __any_sync(0xffffffffu, bad) && lane == 0) atomicMin(d.bad_nu, P.it);
}

// Per-solve chain constants of k_chain_dp: SUT = sum_t ut_t, SG = sum_t g_t
// (chain rows), and zero running aggregates. One warp per chain.
template <typename TG>
__global__ void k_dp_agg_init(FastView f, TG* agg) {
  const DevView& d = f.d;
  const int nu = d.nu, lx = d.lx, N = d.H - f.kstar, AW = dp_agg_w(nu, lx);
  const int ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (ci >= f.nchain) return;
  const GA<TG> G = ga<TG>(f);
  const TG* base = sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32;
  TG* a = agg + (size_t)ci * AW;
  for (int c = lane; c < AW; c += 32) {
    TG s = 0;
    if (c >= 2 * nu && c < 3 * nu) {
      for (int t = 0; t < N; ++t) s += base[((size_t)f.n_branch + (size_t)t * f.nchain + ci) * nu + (c - 2 * nu)];
    } else if (c >= 3 * nu) {
      for (int t = 0; t < N; ++t) s += G.g[((size_t)f.n_branch + (size_t)t * f.nchain + ci) * lx + (c - 3 * nu)];
    }
    a[c] = s;
  }
}

}  // namespace wmpc
