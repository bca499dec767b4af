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
// The same aggregation covers the kb ancestor rows (branching stages): with
// W_anc = sum_{m < kb} ls_m and the per-solve path constants SUTp / SGp (sums
// of ut / g over the chain's whole root path),
//   x_{N-1} = p + B (SUTp - P (W_anc + N LS_anc + LWc)) + SGp,
// so an ancestor row costs one L-row read (L2) and two vector adds, not a
// projector; the one chain that owns a branching row (cown, balanced per warp
// on the host) also computes that row's u, x (from the per-branch-row path
// prefixes PUT / PG) and runs its prox, writing its Yc for the branch-group
// kernels of the next iteration. The kernel is persistent: warp w takes chains
// w, w + NW, w + 2 NW, ...
//
// Memory: per warp, a DP_D-stage ring of the prox operands [y | y_prev | Ua |
// Xa] (5.3 KB per row) filled by 16-byte cp.async.cg (L2 -> shared, no
// registers; released as soon as the row's prox has read it), and L, ut, g
// one row ahead in registers. 14 warps per SM (the bulk_stream microbenchmark:
// 12-16 warps per SM with one row in flight each reach the HBM ceiling).
// fp32 mode: L, ut, g and the aggregates are fp32; the prox operands fp64.
#pragma once
#include "wmpc_chainw.cuh"

namespace wmpc {

#ifndef DP_D_N
#define DP_D_N 2
#endif
constexpr int DP_D = DP_D_N;   // ring stages per warp
constexpr int DP_BND = 448;    // bounds table: xmin 64 | xmax 64 | xsafe 64 | umin 128 | umax 128
constexpr int DP_XCH = 512;    // per-warp exchange vectors (TG): wb 64 | zb 128 | ub 128 | tb 32 | zb2 128 | tb2 32
constexpr int DP_VSLOTS = 22;  // operator value table: bc 8 | ec 4 | kr 4 | br 6 (x 32 lanes)
#ifndef DP_MAXT
#define DP_MAXT 256  // up to 8 warps per CTA, one CTA per SM
#endif
#ifndef DP_SEG_NOOWN
#define DP_SEG_NOOWN 1  // segmented chains: the segment that does not run the owned branching rows' prox
#endif
#ifndef DP_MAXREG
#define DP_MAXREG 255  // <= 8 warps per SM: 2 per sub-partition, no spills (measured: 7 warps x 224 regs 236 us vs 10 warps x 168 regs (spills) 349 us at C4)
#endif

struct DpArgs {
  void* agg;         // nchain x (3 nu + lx), TG: [LSc | LWc | SUTp | SGp]
  const void* putg;  // n_branch x (nu + lx), TG: root-path prefix sums [PUT | PG] of each branching row
  int cpw;           // chains per warp
  int pro_w;         // doubles of a warp's chain-prologue scratch: kstar * nu + (3 nu + lx) [+ 2 nu]
  // Segmented chains (few chains per SM): seg_m > 0 splits every chain into an
  // upper segment (rows [0, seg_m), warp 2p) and a lower one ([seg_m, N),
  // warp 2p + 1) walked at the same time. The lower segment's L rows are
  // final; the upper segment stores its rows' L without the lower segment's
  // contribution (base). Whichever warp of the pair finishes second writes
  // the per-chain correction L_t = base_t + aux_t (c0 + n_t c1), n_t = seg_m - 1 - t
  // (applied where the rows are read next iteration), the upper segment's
  // corrected aggregates and the chain-top totals.
  int seg_m;
  void* aggu;   // nchain x (3 nu + lx): [LS_U | LW_U | SUT_U | SG_U] (upper segment; LW weights seg_m - t)
  void* corr;   // nchain x 2 nu: [c0 | c1]
  void* segx;   // nchain x DP_SXW: [lower: sum yx | sum a] [upper: sum yx | sum a | LS base | LW base]
  int* flag;    // nchain arrival counters (0 -> 1 -> 0 each iteration: the second warp corrects)
  const void* auxs;  // nchain x 4: sums over upper rows of aux, n aux, (m - t) aux, (m - t) n aux
  int sib;           // 1: a warp's chains hold every chain of their stage-(kstar-1) parents, whose
                     // up pass (k_branch_grp's first stage group) the warp runs after its last child
};

// Ring stage layout (doubles): every region starts on a 128-byte boundary so
// a warp's 512-byte cp.async rows and its 16-byte-per-lane reads take the
// minimum number of shared-memory wavefronts.
struct DpStage {
  int oYm, oUa, oXa, oL, oB, oG, oAx, stg;
};
__host__ __device__ constexpr int dp_p16(int x) { return (x + 15) & ~15; }
template <typename TG>
__host__ __device__ constexpr DpStage dp_stage_layout(int nt, int nu, int lx) {
  DpStage s{};
  const int w = 2 * nt + nu;
  s.oYm = dp_p16(w);
  s.oUa = s.oYm + dp_p16(w);
  s.oXa = s.oUa + dp_p16(nu);
  s.oL = s.oXa + dp_p16(lx);
  s.oB = s.oL + dp_p16(nu);
  s.oG = s.oB + dp_p16(nu);
  s.oAx = s.oG + dp_p16(lx);
  s.stg = sizeof(TG) == 8 ? dp_p16(s.oAx + 2) : s.oL;
  return s;
}
constexpr int DP_SD2 = 72;  // second tank-slot norm buffer (bank offset 16 from the first)
constexpr int DP_SD2W = 144;
__host__ __device__ inline int dp_agg_w(int nu, int lx) { return 3 * nu + lx; }
__host__ __device__ constexpr int DP_SXW(int nu, int lx) { return 2 * lx + 4 * nu; }
// Per-CTA pointer block of k_chain_dp in shared memory: under register
// pressure the compiler re-reads these from shared memory (short latency)
// instead of re-loading the bound node-state pointers from global memory.
template <typename TG>
struct alignas(16) DpPtrs {
  const double *yb, *ymb;
  double *ynb, *Ua, *Xa;
  TG *Lb, *U, *X, *Yc, *wbar, *Asub, *agg;
  const TG *UT, *g, *aux, *putg;
  const int* cpath;
  const unsigned* cown;
  int store, pad;
};

__host__ __device__ inline int dp_pro_w(int kstar, int nu, int lx, bool seg) {
  return kstar * nu + 3 * nu + lx + (seg ? 2 * nu : 0);
}
template <typename TG>
__host__ __device__ inline size_t dp_smem(int wpc, int nt, int nu, int lx, int kstar, bool seg = false) {
  return 128 + sizeof(double) * (DP_BND + 8 + DP_VSLOTS * 32) + sizeof(DpPtrs<TG>) +
         (size_t)wpc * (sizeof(double) * (DP_D * (size_t)dp_stage_layout<TG>(nt, nu, lx).stg + DP_SD2W) +
                        sizeof(TG) * DP_XCH) +
         sizeof(double) * (size_t)wpc * (size_t)dp_pro_w(kstar, nu, lx, seg);
}

template <typename TG>
__device__ __forceinline__ typename V2T<TG>::T ld2s(const TG* p) {  // aligned pair (shared or global)
  return *reinterpret_cast<const typename V2T<TG>::T*>(p);
}
template <typename TG>
__device__ __forceinline__ typename V2T<TG>::T ld2cg(const TG* p) {  // aligned pair, L2 (predecessor-written data)
  return __ldcg(reinterpret_cast<const typename V2T<TG>::T*>(p));
}
// numpy clip / maximum (numpy/_core _NPY_MIN/_NPY_MAX: NaN x propagates; bounds are never NaN)
// written with unordered comparisons: one compare and one select per bound
__device__ __forceinline__ double np_clip_u(double x, double lo, double hi) {
  const double m = !(x <= lo) ? x : lo;
  return !(m >= hi) ? m : hi;
}
__device__ __forceinline__ double np_max_u(double a, double b) { return !(a < b) ? a : b; }

// numpy pairwise sum of d2[0..n) (n <= 64) by an 8-lane group: lane8 g sums
// d2[g], d2[g+8], ... below n - n%8 in order, a 3-level tree, then the tail
// in order (pw_group8 of wmpc_fast.cuh with the loop bounds of n <= 64).
__device__ __forceinline__ double pw_group8_64(const double* d2, int n, int lane8, unsigned mask) {
  if (n < 8) {
    double res = 0.0;
    if (lane8 == 0)
      for (int i = 0; i < n; ++i) res = dadd(res, d2[i]);
    return res;
  }
  const int nb = n - (n % 8);
  double r = d2[lane8];
#pragma unroll
  for (int q = 1; q < 8; ++q)
    if (8 * q < nb) r = dadd(r, d2[lane8 + 8 * q]);
  double s = dadd(r, __shfl_down_sync(mask, r, 1, 8));
  double t = dadd(s, __shfl_down_sync(mask, s, 2, 8));
  double res = dadd(t, __shfl_down_sync(mask, t, 4, 8));
  if (lane8 == 0) {
    double tv[7];
#pragma unroll
    for (int q = 0; q < 7; ++q) tv[q] = nb + q < n ? d2[nb + q] : 0.0;
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (nb + q < n) res = dadd(res, tv[q]);
  }
  return res;
}

// The kernel's sparse operators, register-light: a lane's 22 ELL entries
// (slots: B by column q,e -> 2q+e; E by column q -> 8+q; K row e -> 12+e;
// B by row h,e -> 16+3h+e) keep only their column index, 8 bits each, packed
// four to a register (6 registers instead of 22 addresses); the values sit in
// a per-CTA [slot][lane] table. A gather is BFE + LEA + 2 LDS + DFMA.
struct DpOps {
  unsigned pk[6];  // packed entry indices
  unsigned vrow;   // shared address of this lane's value column (slot 0)
  unsigned xb;     // shared address of the warp's exchange vectors
};
template <typename TG>
__device__ __forceinline__ TG dp_gather(const DpOps& o, int slot0, int w, unsigned voff) {
  TG x[8], v[8];
#pragma unroll
  for (int e = 0; e < w; ++e) {
    const int sl = slot0 + e;
    const unsigned idx = (o.pk[sl >> 2] >> (8 * (sl & 3))) & 0xffu;
    x[e] = lds_t(o.xb + voff + idx * (unsigned)sizeof(TG), TG(0));
    v[e] = lds_t(o.vrow + (unsigned)(sl * 32 * sizeof(TG)), TG(0));
  }
  TG s = 0;
#pragma unroll
  for (int e = 0; e < w; ++e) s = fma(v[e], x[e], s);
  return s;
}

// the same entries applied to two exchange vectors (one value load per entry)
template <typename TG>
__device__ __forceinline__ void dp_gather2(const DpOps& o, int slot0, int w, unsigned voff, unsigned voff2, TG& s,
                                           TG& s2) {
  TG x[8], x2[8], v[8];
#pragma unroll
  for (int e = 0; e < w; ++e) {
    const int sl = slot0 + e;
    const unsigned idx = (o.pk[sl >> 2] >> (8 * (sl & 3))) & 0xffu;
    x[e] = lds_t(o.xb + voff + idx * (unsigned)sizeof(TG), TG(0));
    x2[e] = lds_t(o.xb + voff2 + idx * (unsigned)sizeof(TG), TG(0));
    v[e] = lds_t(o.vrow + (unsigned)(sl * 32 * sizeof(TG)), TG(0));
  }
  s = 0;
  s2 = 0;
#pragma unroll
  for (int e = 0; e < w; ++e) {
    s = fma(v[e], x[e], s);
    s2 = fma(v[e], x2[e], s2);
  }
}

// Compile-time network dimensions (NT tanks, NU flows; the instantiated shape
// is the Barcelona-dimension 63 / 114 network, other shapes run the graph
// path): every offset and loop bound is a constant, so no dimension or index
// is rematerialised under register pressure (the runtime-dimension version
// spent 30 % of its instructions on that and on runtime copy loops).
template <int NT, int NU, typename TG>
__global__ void __maxnreg__(DP_MAXREG) k_chain_dp(FastView f, DpArgs A) {
  static_assert(NT <= 64 && NU <= 128 && NU % 2 == 0 && NU > 64, "lane layout: pairs (2l, 2l+1) and (64+2l, 65+2l)");
  constexpr int LX = NT + (NT & 1), LY = LX + NU, W = 2 * NT + NU;
  // stage: [y W | y_prev W | Ua NU | Xa LX] and, in fp64, the chain row's down
  // operands [L NU | ut NU | g LX | aux 2] (fp32 rows are not 16-byte multiples:
  // those come through registers one row ahead)
  constexpr bool SDG = sizeof(TG) == 8;
  constexpr DpStage SL = dp_stage_layout<TG>(NT, NU, LX);
  constexpr int oYm = SL.oYm, oUa = SL.oUa, oXa = SL.oXa, oL = SL.oL, oB = SL.oB, oG = SL.oG, oAx = SL.oAx,
                STG = SL.stg;
  static_assert(!SDG || (oYm % 16 == 0 && STG % 16 == 0), "128-byte regions");
  constexpr int AW = 3 * NU + LX, PW = NU + LX;
  constexpr int WE = 4;
  constexpr int NB = NT - NT % 8;  // pairwise-sum block part of a tank norm
  const DevView& d = f.d;
  const int kb = f.kstar, N = d.H - kb;
  const int wpc = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* bnd = reinterpret_cast<double*>(smem_raw);         // DP_BND
  double* pv = bnd + DP_BND;                                 // 8: gamma, 1/gamma, beta, theta, 1-theta, beta1, w_x, w_s
  DpPtrs<TG>* PT = reinterpret_cast<DpPtrs<TG>*>(pv + 8);
  unsigned char* vtab = reinterpret_cast<unsigned char*>(PT + 1);  // DP_VSLOTS x 32 doubles
  unsigned char* wbase = smem_raw + ((vtab + 8 * DP_VSLOTS * 32 - smem_raw + 127) & ~(size_t)127);
  const size_t wbytes = sizeof(double) * (DP_D * STG + DP_SD2W) + sizeof(TG) * DP_XCH;
  double* ring = reinterpret_cast<double*>(wbase + warp * wbytes);
  double* sd2 = ring + DP_D * STG;  // DP_SD2W: tank-slot squares at 0 and DP_SD2
  double* pro = reinterpret_cast<double*>(wbase + (size_t)wpc * wbytes) + (size_t)warp * A.pro_w;  // chain prologue
  TG* wb = reinterpret_cast<TG*>(sd2 + DP_SD2W);  // 64
  TG* zb = wb + 64;                           // 128
  TG* ub = zb + 128;                          // 128
  TG* tb = ub + 128;                          // 32
  TG* zb2 = tb + 32;                          // 128
  TG* tb2 = zb2 + 128;                        // 32
  const int l2 = 2 * lane;
  const bool ok1 = 64 + l2 < NU, okx2 = l2 + 1 < NT;  // ok0 (l2 < NU) and okx (l2 < NT) hold for every lane
  const int o1 = ok1 ? 64 + l2 : l2;                   // second u pair (a valid in-row offset when absent)
  const unsigned nchain = f.nchain, nbr = f.n_branch;
  for (int i = threadIdx.x; i < DP_BND; i += blockDim.x) {
    double v = 0.0;
    if (i < 64) v = i < NT ? d.xmin[i] : 0.0;
    else if (i < 128) v = i - 64 < NT ? d.xmax[i - 64] : 0.0;
    else if (i < 192) v = i - 128 < NT ? d.xsafe[i - 128] : 0.0;
    else if (i < 320) v = i - 192 < NU ? d.umin[i - 192] : 0.0;
    else v = i - 320 < NU ? d.umax[i - 320] : 0.0;
    bnd[i] = v;
  }
  static_assert(EllW<WE>::BC == 2 && EllW<WE>::EC == 1 && EllW<WE>::KR == 4 && EllW<WE>::BR == 3, "slot map");
  DpOps ops;
  {
    TG* vt = reinterpret_cast<TG*>(vtab);
    unsigned pk[6] = {0, 0, 0, 0, 0, 0};
    auto put = [&](int sl, int idx, TG val) {
      pk[sl >> 2] |= ((unsigned)idx & 0xffu) << (8 * (sl & 3));
      if (warp == 0) vt[sl * 32 + lane] = val;
    };
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = cw_ku(lane, q);
      const Ell<2, TG> b = ell_own<2, TG>(f, own_bc(d, k), k < NU);
      put(2 * q, b.idx[0], b.val[0]);
      put(2 * q + 1, b.idx[1], b.val[1]);
      const Ell<1, TG> e = ell_own<1, TG>(f, own_ec(d, k), k < NU);
      put(8 + q, e.idx[0], e.val[0]);
    }
    const Ell<4, TG> kk = ell_own<4, TG>(f, own_kr(d, lane), lane < d.ns);
#pragma unroll
    for (int e = 0; e < 4; ++e) put(12 + e, kk.idx[e], kk.val[e]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const Ell<3, TG> b = ell_own<3, TG>(f, own_br(d, l2 + h), l2 + h < NT);
#pragma unroll
      for (int e = 0; e < 3; ++e) put(16 + 3 * h + e, b.idx[e], b.val[e]);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) ops.pk[i] = pk[i];
    ops.vrow = smem_u32(vt + lane);
    ops.xb = smem_u32(wb);
  }
  constexpr unsigned WB_OFF = 0, ZB_OFF = 64 * sizeof(TG), UB_OFF = 192 * sizeof(TG), TB_OFF = 320 * sizeof(TG),
                     ZB2_OFF = 352 * sizeof(TG), TB2_OFF = 480 * sizeof(TG);
  auto G_bc = [&](int q) { return dp_gather<TG>(ops, 2 * q, 2, WB_OFF); };   // (B^T wb)_k
  auto G_ec = [&](int q) { return dp_gather<TG>(ops, 8 + q, 1, TB_OFF); };   // (E^T tb)_k
  auto G_kr = [&]() { return dp_gather<TG>(ops, 12, 4, ZB_OFF); };           // (K zb)_lane
  auto G_br = [&](int h) { return dp_gather<TG>(ops, 16 + 3 * h, 3, UB_OFF); };  // (B ub)_j
  pdl_wait();  // L of the branching rows comes from the last group kernel; iter from the first
  pdl_trigger();
  const int it = *d.iter - 1;
  const bool next = it + 1 < f.max_iter;
  if (threadIdx.x == 0) {
    const ProxIt P = prox_it(f);
    pv[0] = P.gamma; pv[1] = P.ig; pv[2] = P.beta; pv[3] = P.theta; pv[4] = P.om; pv[5] = P.beta1;
    pv[6] = d.w_x; pv[7] = d.w_s;
    const GA<TG> G = ga<TG>(f);
    DpPtrs<TG> t;
    t.yb = ybuf(d, it); t.ymb = ybuf(d, it + 2); t.ynb = ybuf_w(d, it + 1); t.Ua = d.Ua; t.Xa = d.Xa;
    t.Lb = G.Lb; t.U = G.U; t.X = G.X; t.Yc = G.Yc; t.wbar = G.wbar; t.Asub = G.Asub;
    t.agg = reinterpret_cast<TG*>(A.agg);
    t.UT = sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32;
    t.g = G.g; t.aux = G.aux; t.putg = reinterpret_cast<const TG*>(A.putg);
    t.cpath = f.cpath; t.cown = f.cown;
    t.store = it == *f.store_it;
    t.pad = 0;
    *PT = t;
  }
  __syncthreads();
  const DpPtrs<TG> Q = *PT;  // in registers (no spill at <= 8 warps per SM)
  const double gamma = pv[0], ig = pv[1], beta = pv[2], theta = pv[3], om = pv[4], beta1 = pv[5];
  const double w_x = pv[6], w_s = pv[7];
  const int gw = blockIdx.x * wpc + warp;
  // whole chains (seg -1), or the upper (0) / lower (1) segment of a warp pair's chains
  const bool segd = A.seg_m > 0;
  const int seg = segd ? (gw & 1) : -1, gp = segd ? (gw >> 1) : gw;
  const int t_lo = seg == 1 ? A.seg_m : 0, t_hi = seg == 0 ? A.seg_m : N, NR = t_hi - t_lo;
  // ---- prox-row ring: owned ancestors then chain rows (bottom-up) of each
  // chain slot; one cp.async group per row (empty past the end)
  int ic_cs = 0, ic_pos = -2;  // the first ++ lands on chain slot 0's prologue
  unsigned ic_own = 0u;
  int ic_k = 0, ck = 0;
  // ring positions per chain: -1 the chain prologue (its ancestors' L rows and
  // its aggregates, into the warp's scratch, not a stage), 0..kb-1 the owned
  // ancestors, kb.. the chain rows bottom-up; one cp.async group each
  auto issue = [&]() {
    bool have = false, chain_row = false;
    unsigned r = 0;
    for (;;) {
      if (++ic_pos == kb + NR) {
        ic_pos = -1;
        ++ic_cs;
      }
      const int ci = gp * A.cpw + ic_cs;
      if (ic_cs >= A.cpw || ci >= (int)nchain) {
        ic_pos = kb + NR - 1;  // park past the end
        ic_cs = A.cpw;
        break;
      }
      if (ic_pos < 0) {  // prologue of chain ci
        ic_own = kb > 0 && seg != DP_SEG_NOOWN ? __ldg(Q.cown + ci) : 0u;
        for (int m = 0; m < kb; ++m) {
          const double* sl = reinterpret_cast<const double*>(Q.Lb) + (size_t)Q.cpath[(size_t)ci * kb + m] * NU +
                             2 * lane;
#pragma unroll
          for (int k = 0; k < (NU / 2 + 31) / 32; ++k)
            if (lane + 32 * k < NU / 2) cp16(pro + m * NU + 2 * lane + 64 * k, sl + 64 * k);
        }
        // aggregates: the chain's (whole / lower segment) or the upper segment's;
        // segmented: then the upper segment's corrections [c0 | c1] (upper) or
        // its corrected [LS_U | LW_U] (lower)
        const double* sa = reinterpret_cast<const double*>(seg == 0 ? A.aggu : Q.agg) + (size_t)ci * AW + 2 * lane;
#pragma unroll
        for (int k = 0; k < (AW / 2 + 31) / 32; ++k)
          if (lane + 32 * k < AW / 2) cp16(pro + kb * NU + 2 * lane + 64 * k, sa + 64 * k);
        if (segd) {
          const double* sc = seg == 0 ? reinterpret_cast<const double*>(A.corr) + (size_t)ci * 2 * NU + 2 * lane
                                      : reinterpret_cast<const double*>(A.aggu) + (size_t)ci * AW + 2 * lane;
#pragma unroll
          for (int k = 0; k < (NU + 31) / 32; ++k)
            if (lane + 32 * k < NU) cp16(pro + kb * NU + AW + 2 * lane + 64 * k, sc + 64 * k);
        }
        break;
      }
      if (ic_pos >= kb) {
        r = nbr + (unsigned)(t_hi - 1 - (ic_pos - kb)) * nchain + (unsigned)ci;
        have = chain_row = true;
        break;
      }
      if ((ic_own >> ic_pos) & 1u) {
        r = (unsigned)Q.cpath[(size_t)ci * kb + ic_pos];
        have = true;
        break;
      }
    }
    if (have) {
      double* st = ring + (ic_k & (DP_D - 1)) * STG;
      const double* s0 = Q.yb + (size_t)r * W + 2 * lane;
      const double* s1 = Q.ymb + (size_t)r * W + 2 * lane;
#pragma unroll
      for (int k = 0; k < (W / 2 + 31) / 32; ++k)
        if (lane + 32 * k < W / 2) {
          cp16(st + 2 * lane + 64 * k, s0 + 64 * k);
          cp16(st + oYm + 2 * lane + 64 * k, s1 + 64 * k);
        }
      const double* s2 = Q.Ua + (size_t)r * NU + 2 * lane;
#pragma unroll
      for (int k = 0; k < (NU / 2 + 31) / 32; ++k)
        if (lane + 32 * k < NU / 2) cp16(st + oUa + 2 * lane + 64 * k, s2 + 64 * k);
      const double* s3 = Q.Xa + (size_t)r * LX + 2 * lane;
#pragma unroll
      for (int k = 0; k < (LX / 2 + 31) / 32; ++k)
        if (lane + 32 * k < LX / 2) cp16(st + oXa + 2 * lane + 64 * k, s3 + 64 * k);
      if constexpr (SDG) {
        if (chain_row) {
          const double* s4 = reinterpret_cast<const double*>(Q.Lb) + (size_t)r * NU + 2 * lane;
          const double* s5 = reinterpret_cast<const double*>(Q.UT) + (size_t)r * NU + 2 * lane;
#pragma unroll
          for (int k = 0; k < (NU / 2 + 31) / 32; ++k)
            if (lane + 32 * k < NU / 2) {
              cp16(st + oL + 2 * lane + 64 * k, s4 + 64 * k);
              cp16(st + oB + 2 * lane + 64 * k, s5 + 64 * k);
            }
          const double* s6 = reinterpret_cast<const double*>(Q.g) + (size_t)r * LX + 2 * lane;
#pragma unroll
          for (int k = 0; k < (LX / 2 + 31) / 32; ++k)
            if (lane + 32 * k < LX / 2) cp16(st + oG + 2 * lane + 64 * k, s6 + 64 * k);
          if (lane == 0) cp16(st + oAx, reinterpret_cast<const double*>(Q.aux) + (size_t)r * 2);
        }
      }
    }
    cp_commit();
    ++ic_k;
  };
  auto take = [&]() -> const double* {
    cp_wait<DP_D - 1>();
    __syncwarp();
    return ring + (ck & (DP_D - 1)) * STG;
  };
  auto release = [&]() {  // every lane has read the stage: refill it with the row DP_D ahead
    __syncwarp();
    ++ck;
    issue();
  };
  if constexpr (SDG) {  // zero padding of the L / ut regions (the copies fill [0, NU) only)
    static_assert(oB - oL >= 128 && oG - oB >= 128, "128-wide L / ut regions");
    constexpr int PADN = 128 - NU;
    for (int i = lane; i < DP_D * 2 * PADN; i += 32) {
      const int stg = i / (2 * PADN), w = (i / PADN) & 1, j = i % PADN;
      ring[stg * STG + (w ? oB : oL) + NU + j] = 0.0;
    }
  }
  for (int k = 0; k < DP_D; ++k) issue();  // (not unrolled: measured 187.4 vs 189.0 us at C4, no spills)
  // ---- operator products through the exchange vectors
  auto proj_neg = [&](const TG (&v)[4], const TG (&base)[4], TG (&out)[4]) {  // out = base + P(-v)
    TG z[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) z[q] = -v[q];
    st2(zb + l2, z[0], z[1]);
    st2(zb + 64 + l2, z[2], z[3]);
    __syncwarp();
    tb[lane] = G_kr();  // zero past ns
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = base[q] + (z[q] - G_ec(q));
  };
  auto bmul = [&](const TG (&u)[4], TG (&bu)[2]) {  // bu = B u (rows l2, l2 + 1)
    st2(ub + l2, u[0], u[1]);
    st2(ub + 64 + l2, u[2], u[3]);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) bu[h] = G_br(h);
  };
  double badacc = 0.0;  // fma(p, 0, .): NaN once any output was not finite
  // Moreau prox of one row (prox_x_warp / prox_u_warp arithmetic per element,
  // bit-exact with numpy), ergodic averages, next collapsed dual
  // In the norms' shadow (the one long dependency chain of a row): bu = B u
  // (the x recursion of the row above) and wn = -P lsn (the down pass of the
  // row above: u = ut + wn, proj_neg's rounding).
  auto prox = [&](const double* st, unsigned r, const TG (&u)[4], const TG (&x)[2], TG (&yx)[2], TG (&yu)[4],
                  TG (&bu)[2], const TG (&lsn)[4], TG (&wn)[4], const TG (&sv)[4], TG (&ps)[4]) {
    double* yn = Q.ynb + (size_t)r * W;
    double v1[2], v2[2], V1[2], V2[2], c1[2], c2[2], y1[2], y2[2];
    {
      const double2 a = ld2s(st + l2), b = ld2s(st + oYm + l2), c = ld2s(st + oXa + l2);
      y1[0] = a.x; y1[1] = a.y;
      y2[0] = st[NT + l2]; y2[1] = st[NT + l2 + 1];
      const double m1[2] = {b.x, b.y}, m2[2] = {st[oYm + NT + l2], st[oYm + NT + l2 + 1]};
      const double xa[2] = {c.x, c.y};
      double xan[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double xv = (double)x[h];
        xan[h] = dadd(dmul(xa[h], om), dmul(theta, xv));  // iteration 0: Xa = 0, om = 0, theta = 1
        const double gx = dmul(gamma, xv);
        v1[h] = dadd(dadd(y1[h], dmul(beta, dsub(y1[h], m1[h]))), gx);
        v2[h] = dadd(dadd(y2[h], dmul(beta, dsub(y2[h], m2[h]))), gx);
        V1[h] = div_by(v1[h], gamma, ig);
        V2[h] = div_by(v2[h], gamma, ig);
      }
      const double2 lo = ld2s(bnd + l2), hi = ld2s(bnd + 64 + l2), sf = ld2s(bnd + 128 + l2);
      c1[0] = np_clip_u(V1[0], lo.x, hi.x);
      c1[1] = np_clip_u(V1[1], lo.y, hi.y);
      c2[0] = np_max_u(V2[0], sf.x);
      c2[1] = np_max_u(V2[1], sf.y);
      double* xap = Q.Xa + (size_t)r * LX + l2;
      if (okx2) st2(xap, xan[0], xan[1]);
      else xap[0] = xan[0];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double df1 = dsub(V1[h], c1[h]), df2 = dsub(V2[h], c2[h]);
        sd2[l2 + h] = dmul(df1, df1);  // slot 63 (past NT) is never read
        sd2[DP_SD2 + l2 + h] = dmul(df2, df2);
      }
    }
    {  // the u part (plain box) while the norms' operands settle
      double p3[4], uan[4];
#pragma unroll
      for (int hq = 0; hq < 2; ++hq) {
        const int o = hq ? o1 : l2;
        const double2 a = ld2s(st + 2 * NT + o), b = ld2s(st + oYm + 2 * NT + o), c = ld2s(st + oUa + o);
        const double2 lo = ld2s(bnd + 192 + o), hi = ld2s(bnd + 320 + o);
        const double y3[2] = {a.x, a.y}, m3[2] = {b.x, b.y}, ua[2] = {c.x, c.y}, l3[2] = {lo.x, lo.y},
                     h3[2] = {hi.x, hi.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int q = 2 * hq + h;
          const double uq = (double)u[q];
          uan[q] = dadd(dmul(ua[h], om), dmul(theta, uq));  // iteration 0: Ua = 0, om = 0, theta = 1
          const double v3 = dadd(dadd(y3[h], dmul(beta, dsub(y3[h], m3[h]))), dmul(gamma, uq));
          const double V3 = div_by(v3, gamma, ig);
          p3[q] = dsub(v3, dmul(gamma, np_clip_u(V3, l3[h], h3[h])));
          yu[q] = (TG)dadd(p3[q], dmul(beta1, dsub(p3[q], y3[h])));
        }
      }
      st2(Q.Ua + (size_t)r * NU + l2, uan[0], uan[1]);
      st2(yn + 2 * NT + l2, p3[0], p3[1]);
      badacc = fma(p3[0], 0.0, fma(p3[1], 0.0, badacc));
      if (ok1) {
        st2(Q.Ua + (size_t)r * NU + 64 + l2, uan[2], uan[3]);
        st2(yn + 2 * NT + 64 + l2, p3[2], p3[3]);
        badacc = fma(p3[2], 0.0, fma(p3[3], 0.0, badacc));
      } else {
        yu[2] = yu[3] = TG(0);
      }
    }
    if (Q.store) {  // the chunk's last iteration: U, X of the row reach HBM (one uniform branch)
      TG* Xp = Q.X + (size_t)r * LX + l2;
      if (okx2) st2(Xp, x[0], x[1]);
      else Xp[0] = x[0];
      st2(Q.U + (size_t)r * NU + l2, u[0], u[1]);
      if (ok1) st2(Q.U + (size_t)r * NU + 64 + l2, u[2], u[3]);
    }
    st2(ub + l2, u[0], u[1]);
    st2(ub + 64 + l2, u[2], u[3]);
    TG zn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) zn[q] = -lsn[q];
    st2(zb + l2, zn[0], zn[1]);
    st2(zb + 64 + l2, zn[2], zn[3]);
    st2(zb2 + l2, sv[0], sv[1]);
    st2(zb2 + 64 + l2, sv[2], sv[3]);
    __syncwarp();
    // the two tank-slot norms, numpy pairwise order (8-lane groups; lanes 16-31
    // repeat lanes 0-15 so the block has no branch and B u interleaves with it)
    const int slot = (lane >> 3) & 1, g = lane & 7;
    const double* s2 = sd2 + DP_SD2 * slot;
    double r8 = s2[g];
#pragma unroll
    for (int q = 1; q < NB / 8; ++q) r8 = dadd(r8, s2[g + 8 * q]);
#pragma unroll
    for (int h = 0; h < 2; ++h) bu[h] = G_br(h);
    {
      TG k1, k2;
      dp_gather2<TG>(ops, 12, 4, ZB_OFF, ZB2_OFF, k1, k2);  // (K zb, K zb2)_lane, zero past ns
      tb[lane] = k1;
      tb2[lane] = k2;
    }
    __syncwarp();
    double ssum = dadd(r8, __shfl_down_sync(0xffffffffu, r8, 1, 8));
    ssum = dadd(ssum, __shfl_down_sync(0xffffffffu, ssum, 2, 8));
    ssum = dadd(ssum, __shfl_down_sync(0xffffffffu, ssum, 4, 8));
#pragma unroll
    for (int q = NB; q < NT; ++q) ssum = dadd(ssum, s2[q]);  // complete on g == 0 only
    const double dist = __dsqrt_rn(ssum);
    const double thr = dmul(ig, slot ? w_s : w_x);  // prox parameter RN(1/gamma) (solver.py:571)
    const double stv = dist > 0.0 ? np_min(1.0, div_exact(thr, dist)) : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      TG e1, e2;
      dp_gather2<TG>(ops, 8 + q, 1, TB_OFF, TB2_OFF, e1, e2);
      wn[q] = zn[q] - e1;
      ps[q] = sv[q] - e2;  // P sv
    }
    const double st1 = __shfl_sync(0xffffffffu, stv, 0), st2v = __shfl_sync(0xffffffffu, stv, 8);
    double p1[2], p2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double O1 = dsub(V1[h], dmul(st1, dsub(V1[h], c1[h])));
      const double O2 = dsub(V2[h], dmul(st2v, dsub(V2[h], c2[h])));
      p1[h] = dsub(v1[h], dmul(gamma, O1));
      p2[h] = dsub(v2[h], dmul(gamma, O2));
      yx[h] = (TG)dadd(dadd(p1[h], dmul(beta1, dsub(p1[h], y1[h]))), dadd(p2[h], dmul(beta1, dsub(p2[h], y2[h]))));
    }
    yn[NT + l2] = p2[0];
    if (okx2) {
      st2(yn + l2, p1[0], p1[1]);
      yn[NT + l2 + 1] = p2[1];
      badacc = fma(p1[0], 0.0, fma(p1[1], 0.0, fma(p2[0], 0.0, fma(p2[1], 0.0, badacc))));
    } else {
      yn[l2] = p1[0];
      badacc = fma(p1[0], 0.0, fma(p2[0], 0.0, badacc));
      yx[1] = TG(0);
    }
  };

  int sib0 = gp * A.cpw;  // first chain of the current stage-(kstar-1) parent
  for (int cs = 0; cs < A.cpw; ++cs) {
    const int ci = gp * A.cpw + cs;
    if (ci >= (int)nchain) break;
    const unsigned r_top = nbr + (unsigned)ci;
    // the chain prologue (a ring group): its ancestors' L rows and its aggregates, in the scratch
    take();
    release();  // occupies no stage: the next group goes out right away
    TG LSc[4], LWc[4], SU[4], SG[2];
    {
      const double* a = pro + kb * NU;
      const double2 s0 = ld2s(a + l2), s1 = ld2s(a + o1), w0 = ld2s(a + NU + l2), w1 = ld2s(a + NU + o1);
      const double2 u0 = ld2s(a + 2 * NU + l2), u1 = ld2s(a + 2 * NU + o1), g0 = ld2s(a + 3 * NU + l2);
      LSc[0] = s0.x; LSc[1] = s0.y; LSc[2] = ok1 ? s1.x : TG(0); LSc[3] = ok1 ? s1.y : TG(0);
      LWc[0] = w0.x; LWc[1] = w0.y; LWc[2] = ok1 ? w1.x : TG(0); LWc[3] = ok1 ? w1.y : TG(0);
      SU[0] = u0.x; SU[1] = u0.y; SU[2] = ok1 ? u1.x : TG(0); SU[3] = ok1 ? u1.y : TG(0);
      SG[0] = g0.x; SG[1] = okx2 ? g0.y : TG(0);
      if (seg == 1) {  // lower segment: whole-chain aggregates from both segments' (the upper's corrected)
        const double2 su0 = ld2s(a + AW + l2), su1 = ld2s(a + AW + o1), wu0 = ld2s(a + AW + NU + l2),
                      wu1 = ld2s(a + AW + NU + o1);
        const TG LSu[4] = {su0.x, su0.y, ok1 ? su1.x : TG(0), ok1 ? su1.y : TG(0)};
        const TG LWu[4] = {wu0.x, wu0.y, ok1 ? wu1.x : TG(0), ok1 ? wu1.y : TG(0)};
        const TG dn = (TG)(N - A.seg_m);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          LWc[q] = fma(dn, LSu[q], LWc[q] + LWu[q]);
          LSc[q] = LSu[q] + LSc[q];
        }
      }
    }
    // ---- ancestors, top-down: ls = running sum of L, Ws = running sum of ls
    TG ls[4] = {0, 0, 0, 0}, Ws[4] = {0, 0, 0, 0};
    const unsigned own = kb > 0 && seg != DP_SEG_NOOWN ? __ldg(Q.cown + ci) : 0u;
    for (int m = 0; m < kb; ++m) {
      const unsigned r = (unsigned)Q.cpath[(size_t)ci * kb + m];
      const double2 a0 = ld2s(pro + m * NU + l2), a1 = ld2s(pro + m * NU + o1);
      const TG La[4] = {a0.x, a0.y, ok1 ? a1.x : TG(0), ok1 ? a1.y : TG(0)};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ls[q] = ls[q] + La[q];
        Ws[q] = Ws[q] + ls[q];
      }
      if ((own >> m) & 1u) {  // this chain owns branching row r: its u, x and prox
        TG ua[4], xa[2], sw[4], bw[2];
        const auto b0 = ld2cg(Q.UT + (size_t)r * NU + l2), b1 = ld2cg(Q.UT + (size_t)r * NU + o1);
        const TG* pg = Q.putg + (size_t)r * PW;
        const auto p0 = ld2cg(pg + l2), p1 = ld2cg(pg + o1), q0 = ld2cg(pg + NU + l2);
        const TG bu[4] = {b0.x, b0.y, ok1 ? b1.x : TG(0), ok1 ? b1.y : TG(0)};
        const TG PU[4] = {p0.x, p0.y, ok1 ? p1.x : TG(0), ok1 ? p1.y : TG(0)};
        proj_neg(ls, bu, ua);  // u_m = ut_m - P ls_m
        proj_neg(Ws, PU, sw);  // sum_{m' <= m} u_m'
        bmul(sw, bw);
        xa[0] = ((TG)d.p[l2] + bw[0]) + q0.x;
        xa[1] = okx2 ? ((TG)d.p[l2 + 1] + bw[1]) + q0.y : TG(0);
        TG yx[2], yu[4], bx[2], wx[4], px[4];
        prox(take(), r, ua, xa, yx, yu, bx, ls, wx, ls, px);
        release();
        if (next) {
          TG* yc = Q.Yc + (size_t)r * LY;
          if (okx2) st2(yc + l2, yx[0], yx[1]);
          else yc[l2] = yx[0];
          st2(yc + LX + l2, yu[0], yu[1]);
          if (ok1) st2(yc + LX + 64 + l2, yu[2], yu[3]);
        }
      }
    }
    // ---- the bottom chain row's prefix sums from the aggregates
    TG xs[2];
    {
      TG V[4], w[4], bw[2];
#pragma unroll
      for (int q = 0; q < 4; ++q) V[q] = fma((TG)t_hi, ls[q], LWc[q]) + Ws[q];
      proj_neg(V, SU, w);  // sum of u over the root path
      bmul(w, bw);
      xs[0] = ((TG)d.p[l2] + bw[0]) + SG[0];
      xs[1] = okx2 ? ((TG)d.p[l2 + 1] + bw[1]) + SG[1] : TG(0);
#pragma unroll
      for (int q = 0; q < 4; ++q) ls[q] = ls[q] + LSc[q];  // ls of the warp's bottom row
    }
    TG wn[4];  // -P ls of the next row down the walk
    {
      TG z[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = -ls[q];
      st2(zb + l2, z[0], z[1]);
      st2(zb + 64 + l2, z[2], z[3]);
      __syncwarp();
      tb[lane] = G_kr();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) wn[q] = z[q] - G_ec(q);
    }
    // ---- chain rows, bottom-up: down of it, prox of it, up of it + 1
    TG wbr[2] = {0, 0}, acc[4] = {0, 0, 0, 0}, LSn[4] = {0, 0, 0, 0}, LWn[4] = {0, 0, 0, 0};
    for (int t = t_hi - 1; t >= t_lo; --t) {
      const unsigned r = nbr + (unsigned)t * nchain + (unsigned)ci;
      TG L[4], b[4], g[2], ax, u[4], yx[2], yu[4];
      const double* st = take();
      {
        // the L / ut regions are 128 wide with zero padding past NU: no masks
        const double2 a0 = ld2s(st + oL + l2), a1 = ld2s(st + oL + 64 + l2), b0 = ld2s(st + oB + l2),
                      b1 = ld2s(st + oB + 64 + l2), g0 = ld2s(st + oG + l2);
        L[0] = a0.x; L[1] = a0.y; L[2] = a1.x; L[3] = a1.y;
        b[0] = b0.x; b[1] = b0.y; b[2] = b1.x; b[3] = b1.y;
        g[0] = g0.x; g[1] = g0.y;  // (the padding column of g is zero: k_pad_rows)
        ax = st[oAx];
        if (seg == 0) {  // upper segment: L_t = base_t + aux_t (c0 + n_t c1) (previous iteration's correction)
          const double* cb = pro + kb * NU + AW;
          const double2 c00 = ld2s(cb + l2), c01 = ld2s(cb + o1), c10 = ld2s(cb + NU + l2), c11 = ld2s(cb + NU + o1);
          const TG c0[4] = {c00.x, c00.y, c01.x, c01.y}, c1[4] = {c10.x, c10.y, c11.x, c11.y};
          const TG nt = (TG)(t_hi - 1 - t);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < 2 || ok1) L[q] = fma(ax, fma(nt, c1[q], c0[q]), L[q]);
        }
      }
      TG bu[2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u[q] = b[q] + wn[q];
        ls[q] = ls[q] - L[q];  // ls of the row above
      }
      TG pS[4];  // P (sum of a below), for the up pass
      prox(st, r, u, xs, yx, yu, bu, ls, wn, acc, pS);
      release();
      if (t > t_lo) {  // x of the row above
        xs[0] = (xs[0] - g[0]) - bu[0];
        xs[1] = (xs[1] - g[1]) - bu[1];
      }
      if (!next) continue;
      // up pass of the next iteration (k_chain_up_r arithmetic, R-free)
      // wbr, acc start at zero and pS = P 0 = 0 at the bottom row: the sums need no
      // bottom-row case (up to the sign of an exact zero)
      wbr[0] = yx[0] + wbr[0];
      wbr[1] = yx[1] + wbr[1];
      st2(wb + l2, wbr[0], wbr[1]);
      __syncwarp();
      TG a[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = yu[q] + G_bc(q);
        acc[q] = a[q] + acc[q];
        l[q] = a[q] + pS[q];
      }
      const TG wt = (TG)(t_hi - t);  // LW weight from the warp's bottom row
      TG Ln[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Ln[q] = l[q] * ax;
        LSn[q] = LSn[q] + Ln[q];
        LWn[q] = fma(wt, Ln[q], LWn[q]);
      }
      TG* Lp = Q.Lb + (size_t)r * NU;
      st2(Lp + l2, Ln[0], Ln[1]);
      if (ok1) st2(Lp + 64 + l2, Ln[2], Ln[3]);
    }
    if (next && seg < 0) {  // chain totals for the branch groups, L aggregates for the next iteration
      if (okx2) st2(Q.wbar + (size_t)r_top * LX + l2, wbr[0], wbr[1]);
      else Q.wbar[(size_t)r_top * LX + l2] = wbr[0];
      st2(Q.Asub + (size_t)r_top * NU + l2, acc[0], acc[1]);
      if (ok1) st2(Q.Asub + (size_t)r_top * NU + 64 + l2, acc[2], acc[3]);
      TG* a = Q.agg + (size_t)ci * AW;
      st2(a + l2, LSn[0], LSn[1]);
      st2(a + NU + l2, LWn[0], LWn[1]);
      if (ok1) {
        st2(a + 64 + l2, LSn[2], LSn[3]);
        st2(a + NU + 64 + l2, LWn[2], LWn[3]);
      }
    }
    if (next && seg >= 0) {  // segmented: the second warp of the pair to finish applies the lower totals
                             // to the upper rows (no waiting: any order). A warp that finds its partner
                             // done (counter 1 -> 0) needs no record of its own; otherwise it publishes
                             // its totals (fenced) and arrives (0 -> 1, or 1 -> 0 if the partner came
                             // in between: then it is the second after all).
      TG* sx = reinterpret_cast<TG*>(A.segx) + (size_t)ci * DP_SXW(NU, LX);
      TG* own = sx + (seg == 1 ? 0 : LX + NU);  // [lower: wbar | a] [upper: wbar | a | LS base | LW base]
      if (seg == 1) {  // the lower segment's L rows are final: its aggregates in any case
        TG* ag = Q.agg + (size_t)ci * AW;
        st2(ag + l2, LSn[0], LSn[1]);
        st2(ag + NU + l2, LWn[0], LWn[1]);
        if (ok1) {
          st2(ag + 64 + l2, LSn[2], LSn[3]);
          st2(ag + NU + 64 + l2, LWn[2], LWn[3]);
        }
      }
      unsigned* cnt = reinterpret_cast<unsigned*>(A.flag) + ci;
      unsigned second = 0u;
      if (lane == 0) second = atomicCAS(cnt, 1u, 0u) == 1u;
      second = __shfl_sync(0xffffffffu, second, 0);
      if (!second) {
        if (okx2) st2(own + l2, wbr[0], wbr[1]);
        else own[l2] = wbr[0];
        st2(own + LX + l2, acc[0], acc[1]);
        if (ok1) st2(own + LX + 64 + l2, acc[2], acc[3]);
        if (seg == 0) {
          TG* ag = own + LX + NU;
          st2(ag + l2, LSn[0], LSn[1]);
          st2(ag + NU + l2, LWn[0], LWn[1]);
          if (ok1) {
            st2(ag + 64 + l2, LSn[2], LSn[3]);
            st2(ag + NU + 64 + l2, LWn[2], LWn[3]);
          }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) second = atomicInc(cnt, 1u) == 1u;  // 0 -> 1 (first), 1 -> 0 (second)
        second = __shfl_sync(0xffffffffu, second, 0);
      }
      __syncwarp();  // every lane is past the last row's reads of the exchange vectors
      if (second) {
        __threadfence();
        const TG* lo = sx;
        const TG* up = sx + LX + NU;
        auto pair4 = [&](const TG* v, TG (&o)[4]) {
          const auto p0 = ld2cg(v + l2), p1 = ld2cg(v + o1);
          o[0] = p0.x; o[1] = p0.y; o[2] = ok1 ? p1.x : TG(0); o[3] = ok1 ? p1.y : TG(0);
        };
        // this warp's own totals from registers, the other segment's from its record (the same bits)
        TG WBd[2], WBu[2], AD[4], AU[4], LSb[4], LWb[4];
        if (seg == 1) {
          const auto wu = ld2cg(up + l2);
          WBu[0] = wu.x; WBu[1] = okx2 ? wu.y : TG(0);
          pair4(up + LX, AU);
          pair4(up + LX + NU, LSb);
          pair4(up + LX + 2 * NU, LWb);
#pragma unroll
          for (int q = 0; q < 4; ++q) AD[q] = acc[q];
          WBd[0] = wbr[0]; WBd[1] = okx2 ? wbr[1] : TG(0);
        } else {
          const auto wd = ld2cg(lo + l2);
          WBd[0] = wd.x; WBd[1] = okx2 ? wd.y : TG(0);
          pair4(lo + LX, AD);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            AU[q] = acc[q];
            LSb[q] = LSn[q];
            LWb[q] = LWn[q];
          }
          WBu[0] = wbr[0]; WBu[1] = okx2 ? wbr[1] : TG(0);
        }
        st2(wb + l2, WBd[0], WBd[1]);
        __syncwarp();
        TG c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = G_bc(q);  // c = B' WB_D
        st2(zb + l2, c[0], c[1]);
        st2(zb + 64 + l2, c[2], c[3]);
        st2(zb2 + l2, AD[0], AD[1]);
        st2(zb2 + 64 + l2, AD[2], AD[3]);
        __syncwarp();
        {
          TG k1, k2;
          dp_gather2<TG>(ops, 12, 4, ZB_OFF, ZB2_OFF, k1, k2);
          tb[lane] = k1;
          tb2[lane] = k2;
        }
        __syncwarp();
        TG c0[4], c1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          TG e1, e2;
          dp_gather2<TG>(ops, 8 + q, 1, TB_OFF, TB2_OFF, e1, e2);
          c1[q] = c[q] - e1;             // P c
          c0[q] = c[q] + (AD[q] - e2);   // c + P A_D
        }
        TG* cr = reinterpret_cast<TG*>(A.corr) + (size_t)ci * 2 * NU;
        st2(cr + l2, c0[0], c0[1]);
        st2(cr + NU + l2, c1[0], c1[1]);
        if (ok1) {
          st2(cr + 64 + l2, c0[2], c0[3]);
          st2(cr + NU + 64 + l2, c1[2], c1[3]);
        }
        const TG* as = reinterpret_cast<const TG*>(A.auxs) + (size_t)ci * 4;
        const TG A0 = as[0], A1 = as[1], A2 = as[2], A3 = as[3];
        const TG mm = (TG)A.seg_m;
        TG* au = reinterpret_cast<TG*>(A.aggu) + (size_t)ci * AW;
        TG LSu[4], LWu[4], At[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          LSu[q] = LSb[q] + (A0 * c0[q] + A1 * c1[q]);
          LWu[q] = LWb[q] + (A2 * c0[q] + A3 * c1[q]);
          At[q] = fma(mm, c[q], AU[q]) + AD[q];
        }
        st2(au + l2, LSu[0], LSu[1]);
        st2(au + NU + l2, LWu[0], LWu[1]);
        if (ok1) {
          st2(au + 64 + l2, LSu[2], LSu[3]);
          st2(au + NU + 64 + l2, LWu[2], LWu[3]);
        }
        const TG Wt[2] = {WBu[0] + WBd[0], WBu[1] + WBd[1]};
        if (okx2) st2(Q.wbar + (size_t)r_top * LX + l2, Wt[0], Wt[1]);
        else Q.wbar[(size_t)r_top * LX + l2] = Wt[0];
        st2(Q.Asub + (size_t)r_top * NU + l2, At[0], At[1]);
        if (ok1) st2(Q.Asub + (size_t)r_top * NU + 64 + l2, At[2], At[3]);
      }
    }
    if (A.sib && next) {  // after the parent's last chain: its up pass (k_branch_grp arithmetic, R-free,
                          // no branching descendants: W2 = 0), from its own Yc and the chains' totals
      const unsigned p = (unsigned)Q.cpath[(size_t)ci * kb + kb - 1];
      const int cn = ci + 1;
      const bool fin = cs + 1 >= A.cpw || cn >= (int)nchain || (unsigned)Q.cpath[(size_t)cn * kb + kb - 1] != p;
      if (fin) {
        // this warp wrote every operand below (same lanes, same addresses)
        TG W1[2] = {0, 0}, Su[4] = {0, 0, 0, 0};
        for (int c = sib0; c <= ci; ++c) {
          const size_t rt = nbr + (size_t)c;
          const auto w = ld2cg(Q.wbar + rt * LX + l2);
          const auto s0 = ld2cg(Q.Asub + rt * NU + l2), s1 = ld2cg(Q.Asub + rt * NU + o1);
          W1[0] += w.x;
          W1[1] += okx2 ? w.y : TG(0);
          Su[0] += s0.x; Su[1] += s0.y; Su[2] += ok1 ? s1.x : TG(0); Su[3] += ok1 ? s1.y : TG(0);
        }
        const TG* yc = Q.Yc + (size_t)p * LY;
        const auto ox = ld2cg(yc + l2), ou0 = ld2cg(yc + LX + l2), ou1 = ld2cg(yc + LX + o1);
        W1[0] = ox.x + W1[0];
        W1[1] = okx2 ? ox.y + W1[1] : TG(0);
        const TG yu[4] = {ou0.x, ou0.y, ok1 ? ou1.x : TG(0), ok1 ? ou1.y : TG(0)};
        const TG axp = Q.aux[(size_t)p * 2];
        __syncwarp();  // every lane is past the last row's reads of wb
        st2(wb + l2, W1[0], W1[1]);
        st2(zb + l2, Su[0], Su[1]);
        st2(zb + 64 + l2, Su[2], Su[3]);
        __syncwarp();
        TG a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = yu[q] + G_bc(q);
        tb[lane] = G_kr();
        __syncwarp();
        TG Lp[4], Ap[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          Lp[q] = (a[q] + (Su[q] - G_ec(q))) * axp;
          Ap[q] = a[q] + Su[q];
        }
        if (okx2) st2(Q.wbar + (size_t)p * LX + l2, W1[0], W1[1]);
        else Q.wbar[(size_t)p * LX + l2] = W1[0];
        st2(Q.Lb + (size_t)p * NU + l2, Lp[0], Lp[1]);
        st2(Q.Asub + (size_t)p * NU + l2, Ap[0], Ap[1]);
        if (ok1) {
          st2(Q.Lb + (size_t)p * NU + 64 + l2, Lp[2], Lp[3]);
          st2(Q.Asub + (size_t)p * NU + 64 + l2, Ap[2], Ap[3]);
        }
        sib0 = cn;
      }
    }
  }
  cp_wait<0>();
  if (__any_sync(0xffffffffu, isnan(badacc)) && lane == 0) atomicMin(d.bad_nu, it);
}

// Per-solve constants of k_chain_dp: per chain SUTp / SGp (ut / g summed over
// the whole root path, ancestors and chain rows), per branching row the root
// path prefixes PUT / PG (including the row); the running L aggregates are
// zeroed (L = 0 at Yc = 0). Segmented chains (segm > 0): also the upper
// segment's SUT_U / SG_U (ancestors + rows [0, segm)) and its aux sums
// [sum aux, sum n aux, sum (segm - t) aux, sum (segm - t) n aux], n = segm - 1 - t.
// One warp per chain / branching row.
template <typename TG>
__global__ void k_dp_agg_init(FastView f, TG* agg, TG* putg, TG* aggu, TG* auxs, int segm) {
  const DevView& d = f.d;
  const int nu = d.nu, lx = d.lx, kb = f.kstar, N = d.H - kb, AW = dp_agg_w(nu, lx), PW = nu + lx;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const GA<TG> G = ga<TG>(f);
  const TG* UT = sizeof(TG) == 8 ? (const TG*)f.ut : (const TG*)f.ut32;
  auto crow = [&](int ci, int t) { return (size_t)f.n_branch + (size_t)t * f.nchain + ci; };
  if (w < f.nchain) {
    const int ci = w;
    for (int part = 0; part < (segm > 0 ? 2 : 1); ++part) {
      const int tend = part == 0 ? N : segm;
      TG* a = (part == 0 ? agg : aggu) + (size_t)ci * AW;
      for (int c = lane; c < AW; c += 32) {
        TG s = 0;
        if (c >= 2 * nu) {
          const bool isg = c >= 3 * nu;
          const int cc = isg ? c - 3 * nu : c - 2 * nu;
          const TG* base = isg ? G.g : UT;
          const int stride = isg ? lx : nu;
          for (int m = 0; m < kb; ++m) s += base[(size_t)f.cpath[(size_t)ci * kb + m] * stride + cc];
          for (int t = 0; t < tend; ++t) s += base[crow(ci, t) * stride + cc];
        }
        a[c] = s;
      }
    }
    if (segm > 0 && lane == 0) {
      TG s0 = 0, s1 = 0, s2 = 0, s3 = 0;
      for (int t = 0; t < segm; ++t) {
        const TG ax = G.aux[crow(ci, t) * 2], n = (TG)(segm - 1 - t), wt = (TG)(segm - t);
        s0 += ax;
        s1 += n * ax;
        s2 += wt * ax;
        s3 += wt * n * ax;
      }
      auxs[(size_t)ci * 4] = s0;
      auxs[(size_t)ci * 4 + 1] = s1;
      auxs[(size_t)ci * 4 + 2] = s2;
      auxs[(size_t)ci * 4 + 3] = s3;
    }
  } else if (w < f.nchain + f.n_branch) {
    const int r = w - f.nchain;
    for (int c = lane; c < PW; c += 32) {
      const bool isg = c >= nu;
      const int cc = isg ? c - nu : c;
      const TG* base = isg ? G.g : UT;
      const int stride = isg ? lx : nu;
      TG s = 0;
      for (int a = r; a >= 0; a = d.anc[a]) s += base[(size_t)a * stride + cc];
      putg[(size_t)r * PW + c] = s;
    }
  }
}

// Warm start: L aggregates of the chains from L (written by the up pass; the
// segment corrections are zero): [LS | LW] over rows [segm, N) with weights
// N - t into agg and, segmented, over rows [0, segm) with weights segm - t into aggu.
template <typename TG>
__global__ void k_dp_agg_L(FastView f, TG* agg, TG* aggu, int segm) {
  const DevView& d = f.d;
  const int nu = d.nu, lx = d.lx, N = d.H - f.kstar, AW = dp_agg_w(nu, lx);
  const int ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (ci >= f.nchain) return;
  const GA<TG> G = ga<TG>(f);
  for (int part = 0; part < (segm > 0 ? 2 : 1); ++part) {
    const int t0 = part == 0 ? segm : 0, t1 = part == 0 ? N : segm;
    TG* a = (part == 0 ? agg : aggu) + (size_t)ci * AW;
    for (int c = lane; c < nu; c += 32) {
      TG s = 0, w = 0;
      for (int t = t1 - 1; t >= t0; --t) {
        const TG L = G.Lb[((size_t)f.n_branch + (size_t)t * f.nchain + ci) * nu + c];
        s = s + L;
        w = fma((TG)(t1 - t), L, w);
      }
      a[c] = s;
      a[nu + c] = w;
    }
  }
}

}  // namespace wmpc
