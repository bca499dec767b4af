// wmpc_chainw.cuh — warp-per-chain variants of the graph's chain kernels.
//
// k_chain_up / k_chain_down (wmpc_scan.cuh) give a chain a 512-thread CTA,
// stage the whole chain in shared memory, and run each scan phase across the
// CTA with a barrier between phases: most threads idle at the barriers during
// the sequential scans. Here one warp walks one chain row by row, carrying the
// running sums in registers, with the same per-element arithmetic (identical
// results):
//   * lane l owns the element pairs (2l, 2l+1) and (64+2l, 65+2l) of the u
//     vectors, (2l, 2l+1) of the x vectors and row l of K, with their ELL
//     operator entries in registers (the _r kernels keep only the operand
//     addresses there and read the values from a per-CTA table: CW_SMV);
//   * rows stream through a per-warp shared-memory ring of PD rows filled by
//     cp.async; every lane copies exactly the pairs it reads, so the ring needs
//     no warp barrier (only the three small exchange vectors do: one
//     __syncwarp per cross-lane product);
//   * PD = 8 rows ahead (chains few per SM: latency-bound, C3); with many
//     chains the register-streamed _r kernels below replace the ring.
#pragma once
#include <type_traits>

#include "wmpc_scan.cuh"

namespace wmpc {

#ifndef CW_WARPS_N
#define CW_WARPS_N 4
#endif
constexpr int CW_WARPS = CW_WARPS_N;  // chains (warps) per CTA
#ifndef CW_MINB
#define CW_MINB 1
#endif

template <typename TG>
struct V2T;
template <>
struct V2T<double> { using T = double2; };
template <>
struct V2T<float> { using T = float2; };

// async copy of an fp64 element pair (16-byte cp.async.cg: L2 only, so a
// predecessor kernel's writes are never served from a stale L1 line)
template <typename TG>
__device__ __forceinline__ void cp_pair(TG* dst, const TG* src) {
  static_assert(sizeof(TG) == 8, "the ring kernels are fp64-only (fp32 mode streams rows through registers)");
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// predicated form: nothing is read (the pair is zero-filled) when !ok; src must
// still be a valid address
template <typename TG>
__device__ __forceinline__ void cp_pair_if(TG* dst, const TG* src, bool ok) {
  static_assert(sizeof(TG) == 8, "the ring kernels are fp64-only (fp32 mode streams rows through registers)");
  const unsigned n = ok ? 16u : 0u;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}
// ELL owner bound to one shared vector: entry addresses precomputed once
template <int W, typename TG>
struct EllS {
  unsigned a[W];
  TG v[W];
};
template <int W, typename TG>
__device__ __forceinline__ EllS<W, TG> ell_bind(const Ell<W, TG>& o, const TG* vec) {
  EllS<W, TG> b;
  const unsigned base = smem_u32(vec);
#pragma unroll
  for (int e = 0; e < W; ++e) {
    b.a[e] = base + (unsigned)o.idx[e] * (unsigned)sizeof(TG);
    b.v[e] = o.val[e];
  }
  return b;
}
__device__ __forceinline__ double lds_t(unsigned a, double) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
  return x;
}
__device__ __forceinline__ float lds_t(unsigned a, float) {
  float x;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a) : "memory");
  return x;
}
template <int W, typename TG>
__device__ __forceinline__ TG ells_dot(const EllS<W, TG>& b) {
  TG x[W];
#pragma unroll
  for (int e = 0; e < W; ++e) x[e] = lds_t(b.a[e], TG(0));
  TG s = 0;
#pragma unroll
  for (int e = 0; e < W; ++e) s = fma(b.v[e], x[e], s);
  return s;
}
template <typename TG>
__device__ __forceinline__ void ld2(const TG* p, TG& a, TG& b) {
  const typename V2T<TG>::T v = *reinterpret_cast<const typename V2T<TG>::T*>(p);
  a = v.x;
  b = v.y;
}
template <typename TG>
__device__ __forceinline__ void st2(TG* p, TG a, TG b) {
  typename V2T<TG>::T v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename V2T<TG>::T*>(p) = v;
}
// operator entries of an owner, zero (no contribution) when the owner is absent
template <int W, typename TG>
__device__ __forceinline__ Ell<W, TG> ell_own(const FastView& f, int owner, bool ok) {
  Ell<W, TG> o = ell_load<W, TG>(f, ok ? owner : 0);
  if (!ok) {
#pragma unroll
    for (int e = 0; e < W; ++e) {
      o.idx[e] = 0;
      o.val[e] = TG(0);
    }
  }
  return o;
}
// u-vector slot s of lane l: element 64*(s>>1) + 2l + (s&1)
__device__ __forceinline__ int cw_ku(int lane, int s) { return 64 * (s >> 1) + 2 * lane + (s & 1); }

// per-warp shared-memory sizes (elements)
__host__ __device__ inline int cw_up_rs(bool withR) { return 64 + 128 + 2 + (withR ? 128 : 0); }
__host__ __device__ inline int cw_up_warp(int pd, bool withR) { return pd * cw_up_rs(withR) + 64 + 128 + 32; }
constexpr int CW_DN_RS = 128 + 128 + 64;
__host__ __device__ inline int cw_dn_warp(int pd) { return pd * CW_DN_RS + 128 + 128 + 32; }

// ---------------------------------------------------------------- k_chain_up_w
// Bottom-up over the chain (t = nst-1 .. 0), as k_chain_up:
//   wbar_t = Yx_t + wbar_{t+1},  a_t = (Yu_t + wbar_t B) [+ R_t],
//   S_t = A_{t+1},  A_t = a_t + S_t,  L_t = (a_t + (S_t - E^T K S_t)) * aux_t
// (the bottom row: L = a * aux). Ring row: [Yx 64 | Yu 128 | aux 2 | R 128].
template <int WE, typename TG, int PD, bool RF>
__global__ void __launch_bounds__(CW_WARPS * 32, CW_MINB) k_chain_up_w(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly, ns = d.ns;
  const int nst = d.H - f.kstar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * CW_WARPS + warp;
  constexpr bool withR = !RF;  // f.rfree == RF
  const int rs = cw_up_rs(withR);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TG* ring = reinterpret_cast<TG*>(smem_raw) + (size_t)warp * cw_up_warp(PD, withR);
  TG* wb = ring + PD * rs;  // 64
  TG* sb = wb + 64;         // 128
  TG* tb = sb + 128;        // 32
  const GA<TG> G = ga<TG>(f);
  const int l2 = 2 * lane;
  const bool ok0 = l2 < nu, ok1 = 64 + l2 < nu, okx = l2 < nt;
  const unsigned o1 = ok1 ? 64 + l2 : 0;  // in-row offset of the second pair (clamped when absent)
  EllS<EllW<WE>::BC, TG> bc[4];
  EllS<EllW<WE>::EC, TG> ec[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = cw_ku(lane, q);
    bc[q] = ell_bind(ell_own<EllW<WE>::BC, TG>(f, own_bc(d, k), k < nu), wb);
    ec[q] = ell_bind(ell_own<EllW<WE>::EC, TG>(f, own_ec(d, k), k < nu), tb);
  }
  const EllS<EllW<WE>::KR, TG> kr = ell_bind(ell_own<EllW<WE>::KR, TG>(f, own_kr(d, lane), lane < ns), sb);
  pdl_wait();  // Yc comes from the prox of the previous iteration
  pdl_trigger();
  if (ci >= f.nchain) return;
  const unsigned r_top = (unsigned)f.n_branch + (unsigned)ci, r_step = (unsigned)f.nchain;
  auto issue = [&](int p) {  // processing position p = row t = nst-1-p
    if (p < nst) {
      const int t = nst - 1 - p;
      TG* s = ring + (p & (PD - 1)) * rs;
      const unsigned r = r_top + (unsigned)t * r_step;
      const TG* yc = G.Yc + r * (unsigned)ly;
      cp_pair_if(s + l2, yc + l2, okx);
      cp_pair_if(s + 64 + l2, yc + lx + l2, ok0);
      cp_pair_if(s + 128 + l2, yc + lx + o1, ok1);
      cp_pair_if(s + 192, G.aux + r * 2u, lane == 0);
      if (withR && t < nst - 1) {
        const TG* rp = G.R + r * (unsigned)nu;
        cp_pair_if(s + 194 + l2, rp + l2, ok0);
        cp_pair_if(s + 194 + 64 + l2, rp + o1, ok1);
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int p = 0; p < PD; ++p) issue(p);
  TG wbr[2] = {0, 0}, acc[4] = {0, 0, 0, 0};
  // one row; the bottom row (p == 0, no S/T part) is peeled off at compile time
  auto row = [&](int p, auto last_tag) {
    constexpr bool last = decltype(last_tag)::value;
    const int t = nst - 1 - p;
    cp_wait<PD - 1>();
    const TG* s = ring + (p & (PD - 1)) * rs;
    TG yx[2], yu[4], rr[4] = {0, 0, 0, 0};
    ld2(s + l2, yx[0], yx[1]);
    ld2(s + 64 + l2, yu[0], yu[1]);
    ld2(s + 128 + l2, yu[2], yu[3]);
    if constexpr (withR && !last) {
      ld2(s + 194 + l2, rr[0], rr[1]);
      ld2(s + 194 + 64 + l2, rr[2], rr[3]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) wbr[h] = last ? yx[h] : yx[h] + wbr[h];
    st2(wb + l2, wbr[0], wbr[1]);
    __syncwarp();
    const TG ax = s[192];  // lane 0's copy: read after the barrier
    TG a[4], S[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      TG v = yu[q] + ells_dot(bc[q]);
      if constexpr (withR && !last) v = v + rr[q];
      a[q] = v;
      S[q] = acc[q];
      acc[q] = last ? v : v + acc[q];
    }
    TG l[4];
    if constexpr (!last) {
      st2(sb + l2, S[0], S[1]);
      st2(sb + 64 + l2, S[2], S[3]);
      __syncwarp();
      tb[lane] = ells_dot(kr);  // zero past ns
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) l[q] = a[q] + (S[q] - ells_dot(ec[q]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) l[q] = a[q];
      __syncwarp();  // wb and the aux slot are rewritten next
    }
    TG* Lp = G.Lb + (r_top + (unsigned)t * r_step) * (unsigned)nu;
    if (ok0) st2(Lp + l2, l[0] * ax, l[1] * ax);
    if (ok1) st2(Lp + 64 + l2, l[2] * ax, l[3] * ax);
    issue(p + PD);
  };
  row(0, std::true_type{});
  for (int p = 1; p < nst; ++p) row(p, std::false_type{});
  if (l2 < nt) G.wbar[(size_t)r_top * lx + l2] = wbr[0];
  if (l2 + 1 < nt) G.wbar[(size_t)r_top * lx + l2 + 1] = wbr[1];
  if (ok0) st2(G.Asub + (size_t)r_top * nu + l2, acc[0], acc[1]);
  if (ok1) st2(G.Asub + (size_t)r_top * nu + 64 + l2, acc[2], acc[3]);
}

// ---------------------------------------------------------------- k_chain_down_w
// Top-down over the chain's whole root path (kstar ancestors, then the chain),
// as k_chain_down:
//   z_m = es_m - sum_{m' <= m} L_m',  u_m = base_m + (z_m - E^T K z_m),
//   x_m = (x_{m-1} + u_m B^T) + g_m,  x_{-1} = p,
// base = ut (R-free) or e_off with es the q + e_off prefix sums. Ancestor rows
// are written by the chain that owns them (cown). Ring row: [L 128 | base 128 | g 64].
template <int WE, typename TG, int PD, bool RF>
__global__ void __launch_bounds__(CW_WARPS * 32, CW_MINB) k_chain_down_w(FastView f) {
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ns = d.ns;
  const int kb = f.kstar, nr = d.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * CW_WARPS + warp;
  const bool live = ci < f.nchain;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TG* ring = reinterpret_cast<TG*>(smem_raw) + (size_t)warp * cw_dn_warp(PD);
  TG* zb = ring + PD * CW_DN_RS;  // 128
  TG* ub = zb + 128;              // 128
  TG* tb = ub + 128;              // 32
  const GA<TG> G = ga<TG>(f);
  constexpr bool rfree = RF;  // f.rfree == RF
  const TG* base = rfree ? (sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32) : G.e_off;
  const int l2 = 2 * lane;
  const bool ok0 = l2 < nu, ok1 = 64 + l2 < nu, okx = l2 < nt;
  const unsigned o1 = ok1 ? 64 + l2 : 0;  // in-row offset of the second pair (clamped when absent)
  const unsigned nchain = f.nchain, nbr = f.n_branch;
  auto grow = [&](int m) -> unsigned {
    return m < kb ? (unsigned)f.cpath[(size_t)ci * kb + m] : nbr + (unsigned)(m - kb) * nchain + (unsigned)ci;
  };
  auto issue_L = [&](TG* s, unsigned r) {
    const TG* p = G.Lb + r * (unsigned)nu;
    cp_pair_if(s + l2, p + l2, ok0);
    cp_pair_if(s + 64 + l2, p + o1, ok1);
  };
  auto issue_bg = [&](TG* s, unsigned r) {
    const TG* p = base + r * (unsigned)nu;
    cp_pair_if(s + 128 + l2, p + l2, ok0);
    cp_pair_if(s + 192 + l2, p + o1, ok1);
    cp_pair_if(s + 256 + l2, G.g + r * (unsigned)lx + l2, okx);
  };
  // before the predecessor finishes: base and g of the first PD rows, and the
  // chain rows' L when they predate the group kernels (f.lb_prewait)
  const int pre = PD < nr ? PD : nr;
  const bool lpre = f.lb_prewait;
  if (live)
    for (int m = 0; m < pre; ++m) {
      TG* s = ring + m * CW_DN_RS;
      const unsigned r = grow(m);
      issue_bg(s, r);
      if (m >= kb && lpre) issue_L(s, r);
    }
  cp_commit();
  EllS<EllW<WE>::EC, TG> ec[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = cw_ku(lane, q);
    ec[q] = ell_bind(ell_own<EllW<WE>::EC, TG>(f, own_ec(d, k), k < nu), tb);
  }
  const EllS<EllW<WE>::KR, TG> kr = ell_bind(ell_own<EllW<WE>::KR, TG>(f, own_kr(d, lane), lane < ns), zb);
  EllS<EllW<WE>::BR, TG> br[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) br[h] = ell_bind(ell_own<EllW<WE>::BR, TG>(f, own_br(d, l2 + h), l2 + h < nt), ub);
  pdl_wait();  // L of the branching rows comes from the last group kernel
  pdl_trigger();
  if (!live) return;
  for (int m = 0; m < pre; ++m)
    if (!(m >= kb && lpre)) issue_L(ring + m * CW_DN_RS, grow(m));
  cp_commit();
  const unsigned own = kb > 0 ? f.cown[ci] : 0u;
  TG ls[4] = {0, 0, 0, 0}, es[4] = {0, 0, 0, 0}, xs[2];
  if constexpr (!rfree) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = cw_ku(lane, q);
      es[q] = k < nu ? (TG)d.q[k] : TG(0);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) xs[h] = l2 + h < nt ? (TG)d.p[l2 + h] : TG(0);
  const bool x2 = l2 + 1 < nt;
  cp_wait<0>();
  auto row = [&](int m, auto first_tag) {  // the first row is peeled off at compile time
    constexpr bool first = decltype(first_tag)::value;
    if constexpr (!first) cp_wait<PD - 1>();
    const TG* s = ring + (m & (PD - 1)) * CW_DN_RS;
    TG L[4], b[4], g[2];
    ld2(s + l2, L[0], L[1]);
    ld2(s + 64 + l2, L[2], L[3]);
    ld2(s + 128 + l2, b[0], b[1]);
    ld2(s + 192 + l2, b[2], b[3]);
    ld2(s + 256 + l2, g[0], g[1]);
    TG z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ls[q] = first ? L[q] : ls[q] + L[q];
      z[q] = es[q] - ls[q];
      if constexpr (!rfree) es[q] = es[q] + b[q];
    }
    st2(zb + l2, z[0], z[1]);
    st2(zb + 64 + l2, z[2], z[3]);
    __syncwarp();
    tb[lane] = ells_dot(kr);  // zero past ns
    __syncwarp();
    TG u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = b[q] + (z[q] - ells_dot(ec[q]));
    const bool wr = m >= kb || ((own >> m) & 1u);
    const unsigned r = grow(m);
    TG* Up = G.U + r * (unsigned)nu;
    if (wr && ok0) st2(Up + l2, u[0], u[1]);
    if (wr && ok1) st2(Up + 64 + l2, u[2], u[3]);
    st2(ub + l2, u[0], u[1]);
    st2(ub + 64 + l2, u[2], u[3]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) xs[h] = (xs[h] + ells_dot(br[h])) + g[h];
    TG* Xp = G.X + r * (unsigned)lx + l2;
    if (wr && x2) st2(Xp, xs[0], xs[1]);
    if (wr && okx && !x2) Xp[0] = xs[0];
    if (m + PD < nr) {
      TG* sn = ring + (m & (PD - 1)) * CW_DN_RS;
      const unsigned rn = grow(m + PD);
      issue_L(sn, rn);
      issue_bg(sn, rn);
    }
    cp_commit();
  };
  row(0, std::true_type{});
  for (int m = 1; m < nr; ++m) row(m, std::false_type{});
}

// ---------------------------------------------------------------- register-streamed variants
// As k_chain_up_w / k_chain_down_w, but each lane loads its own pairs of the
// next row straight into registers (one row ahead) instead of through a
// shared-memory ring: half the L1 data-pipe traffic per row (no ring fill and
// re-read), which is what bounds the ring kernels when the GPU is full.
template <typename TG>
__device__ __forceinline__ typename V2T<TG>::T ldg2_if(const TG* p, bool ok) {
  typename V2T<TG>::T v;
  v.x = TG(0);
  v.y = TG(0);
  if (ok) v = __ldg(reinterpret_cast<const typename V2T<TG>::T*>(p));
  return v;
}
__host__ __device__ inline int cw_up_warp_r() { return 64 + 128 + 32; }
__host__ __device__ inline int cw_dn_warp_r() { return 128 + 128 + 32; }

// Register-light operators for the _r kernels (CW_SMV): the ELL values are the
// same for every chain, so one copy per CTA sits in a shared table laid out
// [slot][lane] (conflict-free); a lane keeps only its operand addresses and
// the address of its first value. Same products, same order: bit-identical to
// the register-resident form. CW_R_MINB caps registers for more resident
// chains per SM.
#ifndef CW_SMV
#define CW_SMV 1
#endif
#ifndef CW_R_MINB
#define CW_R_MINB 7
#endif
constexpr int CW_R_MB = CW_SMV ? CW_R_MINB : CW_MINB;
constexpr int CW_UP_SLOTS = 16, CW_DN_SLOTS = 14;  // bc 4x2 + ec 4x1 + kr 4 | ec 4x1 + kr 4 + br 2x3
// VF: the B and E values are stored as float when every one of them is exact
// in fp32 (wmpc_ctx::ell_vf, checked on the host; +-1 for the Barcelona-type
// networks): one shared wavefront per 32 lanes instead of two, and the
// float -> double conversion is exact, so the products are unchanged.
template <int W, typename TG, typename TV = TG>
struct EllV {
  unsigned a[W];
  unsigned v;  // shared address of entry 0's value; entry e at v + e * 32 * sizeof(TV)
};
template <typename TV, int W, typename TG>
__device__ __forceinline__ EllV<W, TG, TV> ellv_bind(const Ell<W, TG>& o, const TG* vec, unsigned char* tab, int& off,
                                                     int lane, bool writer) {
  EllV<W, TG, TV> b;
  const unsigned base = smem_u32(vec);
  TV* t = reinterpret_cast<TV*>(tab + off);
#pragma unroll
  for (int e = 0; e < W; ++e) {
    b.a[e] = base + (unsigned)o.idx[e] * (unsigned)sizeof(TG);
    if (writer) t[e * 32 + lane] = (TV)o.val[e];
  }
  b.v = smem_u32(t + lane);
  off += W * 32 * (int)sizeof(TV);
  return b;
}
template <int W, typename TG, typename TV>
__device__ __forceinline__ TG ellv_dot(const EllV<W, TG, TV>& b) {
  TG x[W], w[W];
#pragma unroll
  for (int e = 0; e < W; ++e) {
    x[e] = lds_t(b.a[e], TG(0));
    w[e] = (TG)lds_t(b.v + (unsigned)(e * 32 * sizeof(TV)), TV(0));
  }
  TG s = 0;
#pragma unroll
  for (int e = 0; e < W; ++e) s = fma(w[e], x[e], s);
  return s;
}
template <int W, typename TG, typename TV>
__device__ __forceinline__ TG cw_dot(const EllV<W, TG, TV>& b) { return ellv_dot(b); }
template <int W, typename TG>
__device__ __forceinline__ TG cw_dot(const EllS<W, TG>& b) { return ells_dot(b); }
// K values (TG) / B values (TB) / E values (TB; in fp32 the width-1 E
// operator keeps its values in registers: C4 fp32 203 -> 199 us, while in
// fp64 the 8 extra registers spill at 72, +3 us)
template <int W, typename TG>
using EllRK = std::conditional_t<CW_SMV, EllV<W, TG>, EllS<W, TG>>;
template <int W, typename TG, typename TB>
using EllRB = std::conditional_t<CW_SMV, EllV<W, TG, TB>, EllS<W, TG>>;
template <int W, typename TG, typename TB>
using EllRE = std::conditional_t<CW_SMV && sizeof(TG) == 8, EllV<W, TG, TB>, EllS<W, TG>>;
template <typename R, typename TV, int W, typename TG>
__device__ __forceinline__ R cw_bind(const Ell<W, TG>& o, const TG* vec, unsigned char* tab, int& off, int lane,
                                     bool writer) {
  if constexpr (std::is_same_v<R, EllS<W, TG>>) return ell_bind(o, vec);
  else return ellv_bind<TV>(o, vec, tab, off, lane, writer);
}
#define CW_DOT(b) cw_dot(b)

template <int WE, typename TG, bool RF, int RD, bool VF>
__global__ void __launch_bounds__(CW_WARPS * 32, CW_R_MB) k_chain_up_r(FastView f) {
  using TB = std::conditional_t<VF && sizeof(TG) == 8, float, TG>;  // B, E value storage
  using V = typename V2T<TG>::T;
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ly = d.ly, ns = d.ns;
  const int nst = d.H - f.kstar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * CW_WARPS + warp;
  constexpr bool withR = !RF;  // f.rfree == RF
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TG* wb = reinterpret_cast<TG*>(smem_raw) + (size_t)warp * cw_up_warp_r();  // 64
  TG* sb = wb + 64;                                                           // 128
  TG* tb = sb + 128;                                                          // 32
  unsigned char* vtab = smem_raw + sizeof(TG) * (size_t)CW_WARPS * cw_up_warp_r();  // <= CW_UP_SLOTS x 32 (CW_SMV)
  int voff = 0;
  (void)vtab;
  (void)voff;
  const GA<TG> G = ga<TG>(f);
  const int l2 = 2 * lane;
  const bool ok0 = l2 < nu, ok1 = 64 + l2 < nu, okx = l2 < nt;
  const unsigned o1 = ok1 ? 64 + l2 : 0;
  EllRB<EllW<WE>::BC, TG, TB> bc[4];
  EllRE<EllW<WE>::EC, TG, TB> ec[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = cw_ku(lane, q);
    bc[q] = cw_bind<EllRB<EllW<WE>::BC, TG, TB>, TB>(ell_own<EllW<WE>::BC, TG>(f, own_bc(d, k), k < nu), wb, vtab, voff, lane, warp == 0);
    ec[q] = cw_bind<EllRE<EllW<WE>::EC, TG, TB>, TB>(ell_own<EllW<WE>::EC, TG>(f, own_ec(d, k), k < nu), tb, vtab, voff, lane, warp == 0);
  }
  const EllRK<EllW<WE>::KR, TG> kr = cw_bind<EllRK<EllW<WE>::KR, TG>, TG>(ell_own<EllW<WE>::KR, TG>(f, own_kr(d, lane), lane < ns), sb, vtab, voff, lane, warp == 0);
#if CW_SMV
  __syncthreads();  // the value table is written by warp 0
#endif
  pdl_wait();  // Yc comes from the prox of the previous iteration
  pdl_trigger();
  if (ci >= f.nchain) return;
  const unsigned r_top = (unsigned)f.n_branch + (unsigned)ci, r_step = (unsigned)f.nchain;
  struct Row {
    V yx, yu0, yu1, r0, r1;
    TG ax;
  };
  auto load = [&](Row& R, int p) {  // processing position p = row t = nst-1-p
    const int t = nst - 1 - p;
    const unsigned r = r_top + (unsigned)t * r_step;
    const TG* yc = G.Yc + r * (unsigned)ly;
    R.yx = ldg2_if(yc + l2, okx);
    R.yu0 = ldg2_if(yc + lx + l2, ok0);
    R.yu1 = ldg2_if(yc + lx + o1, ok1);
    R.ax = __ldg(G.aux + r * 2u);
    if constexpr (withR) {
      const TG* rp = G.R + r * (unsigned)nu;
      const bool in = t < nst - 1;
      R.r0 = ldg2_if(rp + l2, ok0 && in);
      R.r1 = ldg2_if(rp + o1, ok1 && in);
    }
  };
  Row cur, n1;
  load(cur, 0);
  if constexpr (RD == 2) load(n1, nst > 1 ? 1 : 0);
  TG wbr[2] = {0, 0}, acc[4] = {0, 0, 0, 0};
  auto row = [&](int p, auto last_tag) {  // the bottom row (no S/T part) is peeled off at compile time
    constexpr bool last = decltype(last_tag)::value;
    const int t = nst - 1 - p;
    Row nxt;
    load(nxt, p + RD < nst ? p + RD : nst - 1);
    const TG yx[2] = {cur.yx.x, cur.yx.y};
    const TG yu[4] = {cur.yu0.x, cur.yu0.y, cur.yu1.x, cur.yu1.y};
#pragma unroll
    for (int h = 0; h < 2; ++h) wbr[h] = last ? yx[h] : yx[h] + wbr[h];
    st2(wb + l2, wbr[0], wbr[1]);
    __syncwarp();
    TG a[4], S[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      TG v = yu[q] + CW_DOT(bc[q]);
      if constexpr (withR && !last) {
        const TG rr[4] = {cur.r0.x, cur.r0.y, cur.r1.x, cur.r1.y};
        v = v + rr[q];
      }
      a[q] = v;
      S[q] = acc[q];
      acc[q] = last ? v : v + acc[q];
    }
    TG l[4];
    if constexpr (!last) {
      st2(sb + l2, S[0], S[1]);
      st2(sb + 64 + l2, S[2], S[3]);
      __syncwarp();
      tb[lane] = CW_DOT(kr);  // zero past ns
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) l[q] = a[q] + (S[q] - CW_DOT(ec[q]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) l[q] = a[q];
      __syncwarp();  // wb is rewritten next
    }
    const TG ax = cur.ax;
    TG* Lp = G.Lb + (r_top + (unsigned)t * r_step) * (unsigned)nu;
    if (ok0) st2(Lp + l2, l[0] * ax, l[1] * ax);
    if (ok1) st2(Lp + 64 + l2, l[2] * ax, l[3] * ax);
    if constexpr (RD == 2) {
      cur = n1;
      n1 = nxt;
    } else {
      cur = nxt;
    }
  };
  row(0, std::true_type{});
  for (int p = 1; p < nst; ++p) row(p, std::false_type{});
  if (l2 < nt) G.wbar[(size_t)r_top * lx + l2] = wbr[0];
  if (l2 + 1 < nt) G.wbar[(size_t)r_top * lx + l2 + 1] = wbr[1];
  if (ok0) st2(G.Asub + (size_t)r_top * nu + l2, acc[0], acc[1]);
  if (ok1) st2(G.Asub + (size_t)r_top * nu + 64 + l2, acc[2], acc[3]);
}

template <int WE, typename TG, bool RF, int RD, bool VF>
__global__ void __launch_bounds__(CW_WARPS * 32, CW_R_MB) k_chain_down_r(FastView f) {
  using TB = std::conditional_t<VF && sizeof(TG) == 8, float, TG>;  // B, E value storage
  using V = typename V2T<TG>::T;
  const DevView& d = f.d;
  const int nt = d.nt, nu = d.nu, lx = d.lx, ns = d.ns;
  const int kb = f.kstar, nr = d.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * CW_WARPS + warp;
  const bool live = ci < f.nchain;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TG* zb = reinterpret_cast<TG*>(smem_raw) + (size_t)warp * cw_dn_warp_r();  // 128
  TG* ub = zb + 128;                                                          // 128
  TG* tb = ub + 128;                                                          // 32
  const GA<TG> G = ga<TG>(f);
  constexpr bool rfree = RF;  // f.rfree == RF
  const TG* base = rfree ? (sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32) : G.e_off;
  const int l2 = 2 * lane;
  const bool ok0 = l2 < nu, ok1 = 64 + l2 < nu, okx = l2 < nt;
  const unsigned o1 = ok1 ? 64 + l2 : 0;
  const unsigned nchain = f.nchain, nbr = f.n_branch;
  auto grow = [&](int m) -> unsigned {
    return m < kb ? (unsigned)f.cpath[(size_t)ci * kb + m] : nbr + (unsigned)(m - kb) * nchain + (unsigned)ci;
  };
  struct Row {
    V L0, L1, b0, b1, g;
  };
  auto load_L = [&](Row& R, unsigned r) {
    const TG* p = G.Lb + r * (unsigned)nu;
    R.L0 = ldg2_if(p + l2, ok0);
    R.L1 = ldg2_if(p + o1, ok1);
  };
  auto load_bg = [&](Row& R, unsigned r) {
    const TG* p = base + r * (unsigned)nu;
    R.b0 = ldg2_if(p + l2, ok0);
    R.b1 = ldg2_if(p + o1, ok1);
    R.g = ldg2_if(G.g + r * (unsigned)lx + l2, okx);
  };
  // before the predecessor finishes: base and g of the first row, and its L
  // when it is a chain row that predates the group kernels (f.lb_prewait)
  const bool l0pre = kb == 0 && f.lb_prewait;
  Row cur;
  const unsigned r0 = live ? grow(0) : 0u;
  if (live) {
    load_bg(cur, r0);
    if (l0pre) load_L(cur, r0);
  }
  unsigned char* vtab = smem_raw + sizeof(TG) * (size_t)CW_WARPS * cw_dn_warp_r();  // <= CW_DN_SLOTS x 32 (CW_SMV)
  int voff = 0;
  (void)vtab;
  (void)voff;
  EllRE<EllW<WE>::EC, TG, TB> ec[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = cw_ku(lane, q);
    ec[q] = cw_bind<EllRE<EllW<WE>::EC, TG, TB>, TB>(ell_own<EllW<WE>::EC, TG>(f, own_ec(d, k), k < nu), tb, vtab, voff, lane, warp == 0);
  }
  const EllRK<EllW<WE>::KR, TG> kr = cw_bind<EllRK<EllW<WE>::KR, TG>, TG>(ell_own<EllW<WE>::KR, TG>(f, own_kr(d, lane), lane < ns), zb, vtab, voff, lane, warp == 0);
  EllRB<EllW<WE>::BR, TG, TB> br[2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
    br[h] = cw_bind<EllRB<EllW<WE>::BR, TG, TB>, TB>(ell_own<EllW<WE>::BR, TG>(f, own_br(d, l2 + h), l2 + h < nt), ub, vtab, voff, lane, warp == 0);
#if CW_SMV
  __syncthreads();  // the value table is written by warp 0
#endif
  pdl_wait();  // L of the branching rows comes from the last group kernel
  pdl_trigger();
  if (!live) return;
  if (!l0pre) load_L(cur, r0);
  Row n1;  // RD == 2: the row after next is loaded while this one is processed
  unsigned r1 = r0;
  if constexpr (RD == 2) {
    r1 = grow(nr > 1 ? 1 : 0);
    load_L(n1, r1);
    load_bg(n1, r1);
  }
  const unsigned own = kb > 0 ? f.cown[ci] : 0u;
  TG ls[4] = {0, 0, 0, 0}, es[4] = {0, 0, 0, 0}, xs[2];
  if constexpr (!rfree) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = cw_ku(lane, q);
      es[q] = k < nu ? (TG)d.q[k] : TG(0);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) xs[h] = l2 + h < nt ? (TG)d.p[l2 + h] : TG(0);
  const bool x2 = l2 + 1 < nt;
  unsigned r = r0;
  auto row = [&](int m, auto first_tag) {  // the first row is peeled off at compile time
    constexpr bool first = decltype(first_tag)::value;
    Row nxt;
    const int mn = m + RD < nr ? m + RD : nr - 1;
    const unsigned rn = grow(mn);
    load_L(nxt, rn);
    load_bg(nxt, rn);
    const TG L[4] = {cur.L0.x, cur.L0.y, cur.L1.x, cur.L1.y};
    const TG b[4] = {cur.b0.x, cur.b0.y, cur.b1.x, cur.b1.y};
    TG z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ls[q] = first ? L[q] : ls[q] + L[q];
      z[q] = es[q] - ls[q];
      if constexpr (!rfree) es[q] = es[q] + b[q];
    }
    st2(zb + l2, z[0], z[1]);
    st2(zb + 64 + l2, z[2], z[3]);
    __syncwarp();
    tb[lane] = CW_DOT(kr);  // zero past ns
    __syncwarp();
    TG u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = b[q] + (z[q] - CW_DOT(ec[q]));
    const bool wr = m >= kb || ((own >> m) & 1u);
    TG* Up = G.U + r * (unsigned)nu;
    if (wr && ok0) st2(Up + l2, u[0], u[1]);
    if (wr && ok1) st2(Up + 64 + l2, u[2], u[3]);
    st2(ub + l2, u[0], u[1]);
    st2(ub + 64 + l2, u[2], u[3]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) xs[h] = (xs[h] + CW_DOT(br[h])) + (h ? cur.g.y : cur.g.x);
    TG* Xp = G.X + r * (unsigned)lx + l2;
    if (wr && x2) st2(Xp, xs[0], xs[1]);
    if (wr && okx && !x2) Xp[0] = xs[0];
    if constexpr (RD == 2) {
      cur = n1;
      n1 = nxt;
      r = r1;
      r1 = rn;
    } else {
      cur = nxt;
      r = rn;
    }
  };
  row(0, std::true_type{});
  for (int m = 1; m < nr; ++m) row(m, std::false_type{});
}

}  // namespace wmpc
