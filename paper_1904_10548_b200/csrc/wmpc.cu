// wmpc.cu — C ABI (include/wmpc.h) over the sm_100a kernels.
//
// The context owns every device buffer of one tree structure; the APG
// iteration (2H stage kernels + 1 counter kernel) is captured once per
// wmpc_apg_begin into a CUDA graph and replayed; nothing leaves HBM between
// iterations except the scalars read at check iterations.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved at run time (the process may already hold torch's)

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "wmpc.h"
#include "wmpc_scan.cuh"
#include "wmpc_chainw.cuh"
#include "wmpc_dp.cuh"

// k_chain_dp's instantiated network shape (the Barcelona-dimension network of
// BASELINE.json; other shapes run the graph path)
constexpr int DP_NT = 63, DP_NU = 114;

using namespace wmpc;

static thread_local std::string g_global_err;

struct wmpc_nodes {
  int dev = 0;
  size_t n = 0;
  double *u_part = nullptr, *e_off = nullptr, *R = nullptr, *shift = nullptr, *g = nullptr, *ebar = nullptr;
  bool ready = false;
};

struct wmpc_ctx {
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream_rd = nullptr;  // result readout (wmpc_apg_read_async), overlapping the certificate
  cudaEvent_t ev_rd = nullptr;
  double *rb_u0 = nullptr, *rb_p = nullptr, *rb_a = nullptr;  // readout staging (device)
  int n = 0, H = 0, nt = 0, nu = 0, nd = 0, ns = 0, W = 0, P = 0, lx = 0, ly = 0;
  int a_identity = 0, w_scalar = 0;
  double w_c = 0.0;
  std::vector<int> off;  // H+1
  bool have_structure = false, have_nodes = false, have_bounds = false;
  // device buffers
  int *stage_of = nullptr, *anc = nullptr, *cptr = nullptr, *cidx = nullptr;
  double *prob = nullptr, *A = nullptr, *At = nullptr, *Bt = nullptr, *Wu = nullptr;
  double *T = nullptr, *Lam = nullptr, *Mb = nullptr, *Mf = nullptr, *E = nullptr, *e_pinv = nullptr;
  wmpc_nodes* nodes = nullptr;  // bound per-node state (not owned)
  NodePtrs* d_np = nullptr;     // device copy of the bound node pointers
  double *econ = nullptr, *tmp = nullptr, *demand = nullptr, *Ed = nullptr;
  double *xmin = nullptr, *xmax = nullptr, *xsafe = nullptr, *umin = nullptr, *umax = nullptr;
  double *p = nullptr, *q = nullptr;
  double w_x = 0.0, w_s = 0.0;
  double *Y[3] = {nullptr, nullptr, nullptr};
  double *U = nullptr, *X = nullptr, *Ua = nullptr, *Xa = nullptr;
  double *Uc = nullptr, *Xc = nullptr, *Uf = nullptr, *Xf = nullptr, *U0 = nullptr, *X0 = nullptr;
  double *wbar = nullptr, *lin = nullptr, *Yc = nullptr;
  double *ys = nullptr, *gv = nullptr, *vv = nullptr, *zbuf = nullptr;
  double* gd_stage = nullptr;  // factor step: demand_gd as uploaded (n x nt)
  double *theta = nullptr, *beta = nullptr;
  int max_iter = 0;
  int *iter = nullptr, *bad_nu = nullptr, *bad_row = nullptr;
  double *part = nullptr, *scal = nullptr;
  int part_blocks = 0;
  double gamma = 0.0;
  int it_host = 0;
  int64_t launches = 0;
  double graph_gamma = -1.0;
  // structured fast path (wmpc_fast.cuh)
  bool fast = false;
  int kstar = 0, nchain = 0, fast_mc = 1, fast_cpc = 1, fast_gs = 1, fast_grid = 0;
  int fast_nrow = 2, fast_rec = 0, fast_enz = 0, fast_bnz = 0, fast_knz = 0;
  int use_scan = 0, scan_work = 0;
  size_t scan_smem = 0;
  // graph-of-kernels scan path (wmpc_scan.cuh)
  // sparse projector operands (K = (E E^T)^{-1} E by rows, E by columns)
  int *pj_kp = nullptr, *pj_kc = nullptr, *pj_ecp = nullptr, *pj_ecr = nullptr;
  double *pj_kv = nullptr, *pj_ecv = nullptr;
  unsigned long long* dk_mv = nullptr;
  int* dk_sweeps = nullptr;
  int* dk_free = nullptr;                      // inputs in no coupling row (E column empty)
  int dk_nfree = 0;
  int* dk_list = nullptr;                      // block Dykstra pass 2: [count | block indices]
  int* dk_fix = nullptr;                       // certificate Dykstra: settled sweep per node (k_dyk_warp) or per (node, coupling row) (k_dyk_block)
  int use_graphk = 0, n_branch = 0;
  int* store_it = nullptr;
  int store_it_host = 0;
  double *Lb = nullptr, *Asub = nullptr;
  unsigned char* blob = nullptr;
  int blob16 = 0;
  int *gi_ptr = nullptr, *gi_item = nullptr, *gi_w = nullptr, *cpath = nullptr;
  unsigned* cown = nullptr;
  std::vector<std::pair<int, int>> gk_groups;  // (first row, rows) per stage group, bottom-up
  std::pair<int, int> rep_group{0, 0};         // subtree sharding: replicated rows (first, count)
  std::vector<int> h_cptr, h_cidx;             // host CSR children
  std::vector<int> h_cpath;                    // host copy of cpath (nchain x kstar)
  double* Yc_save = nullptr;                   // certificate: APG state while Yc holds collapse(y)
  int* acct = nullptr;                         // subtree sharding: rows counted in global sums
  int* rep_gidx = nullptr;                     // per local row: global replicated index or -1
  double* xbuf = nullptr;                      // exchange buffer (caller-owned device memory)
  int n_rep_global = 0, shard_k = -1, kstar_min = 0;
  ncclComm_t nccl = nullptr;                   // subtree sharding: exchange inside the iteration graph
  size_t sm_up = 0, sm_grp = 0, sm_grp128 = 0, sm_down = 0, sm_prox = 0;
  int up_threads = 512, down_threads = 512, prox_warp = 1;
  int fp32 = 0;                                 // SolverConfig.precision == "fp32"
  int pdl = 1;                                  // programmatic dependent launch between graph kernels
  int chain_occ = 0;                            // chain kernels: register cap for occupancy (many chains)
  int chainw = 0, cw_pd = 8;                   // warp-per-chain kernels (wmpc_chainw.cuh): 8-row ring or registers (1)
  int chainw32 = 0;                             // ... also in fp32 mode (register variant only)
  int rfree = 1;                                // R-free iteration form (graph path, unsharded, unfused)
  double* ut = nullptr;                         // u at Yc = 0 (rfree), per solve
  float* ut32 = nullptr;
#ifndef GRP_ITEMS_CAP
#define GRP_ITEMS_CAP 16
#endif
  int grp_items = GRP_ITEMS_CAP;                           // max items per row in one branching stage group (measured)
  int grp_items_few = 16;                       // ... when the stage has at most one row per SM
  float *f32_Yc = nullptr, *f32_Lb = nullptr, *f32_Asub = nullptr, *f32_wbar = nullptr, *f32_U = nullptr,
        *f32_X = nullptr, *f32_eoff = nullptr, *f32_R = nullptr, *f32_g = nullptr, *f32_aux = nullptr,
        *f32_ell = nullptr;
  size_t ell_len = 0;
  int *ell_cnt = nullptr, *ell_idx = nullptr;
  double* ell_val = nullptr;
  int ell_w = 4;
  int ell_vf = 0;                               // B, E ELL values exact in fp32 (WMPC_ELL_VF=0 disables)
  // fused one-kernel iteration for many chains (wmpc_dp.cuh)
  int use_dp = 0, dp_wpc = 0, dp_grid = 0, dp_cpw = 1;
  int dp_sib = 0;  // k_chain_dp runs the up pass of the stage-(kstar-1) rows (gk_groups[0] skipped)
  size_t dp_sm = 0;
  double* dp_agg = nullptr;  // nchain x (3 nu + lx): [LSc | LWc | SUTp | SGp]
  double* dp_putg = nullptr;  // n_branch x (nu + lx): root-path prefixes [PUT | PG]
  int dp_segm = 0;            // > 0: segmented chains (upper rows [0, dp_segm) on their own warp)
  double *dp_aggu = nullptr, *dp_corr = nullptr, *dp_segx = nullptr, *dp_auxs = nullptr;  // see DpArgs
  int* dp_flag = nullptr;
  double *dp_Lc = nullptr, *dp_Ac = nullptr, *dp_wc = nullptr;  // certificate scratch (the iteration state stays)
  cudaGraphExec_t gk_exec1 = nullptr, gk_exec8 = nullptr;
  double gk_gamma = -1.0;
  int gk_maxit = -1;
  unsigned long long* prof = nullptr;
  float last_debug_ms = 0.f;
  int prof_on = 0;
  size_t fast_smem = 0;
  int *chain_node = nullptr, *bc_ptr = nullptr, *bc_row = nullptr, *br_ptr = nullptr, *br_col = nullptr;
  int *e_ptr = nullptr, *e_col = nullptr;
  double *e_val = nullptr, *aux = nullptr;
  std::vector<double> prob_host;
  int* off_dev = nullptr;
  double *bc_val = nullptr, *br_val = nullptr;
  int sms = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  std::string err;
};

namespace {

struct Fail {};

// NCCL entry points, resolved on first use from the libnccl already in the
// process (torch's) or the system one: libwmpc does not link NCCL, so loading
// it never pins an NCCL version ahead of torch.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
  api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.get_unique_id && api.init_rank && api.all_reduce && api.destroy && api.error_string;
  return api;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ctx->err = std::string("CUDA error ") + cudaGetErrorString(e_) + " at " #call;    \
      throw Fail{};                                                                     \
    }                                                                                   \
  } while (0)

#define ARG(cond, msg)        \
  do {                        \
    if (!(cond)) {            \
      ctx->err = (msg);       \
      return WMPC_E_ARG;      \
    }                         \
  } while (0)

template <class T>
void dalloc(wmpc_ctx* ctx, T** p, size_t count) {
  CK(cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T)));
  CK(cudaMemsetAsync(*p, 0, std::max<size_t>(count, 1) * sizeof(T), ctx->stream));
}

void h2d(wmpc_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}
void d2h(wmpc_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}
void sync(wmpc_ctx* ctx) { CK(cudaStreamSynchronize(ctx->stream)); }
void check_launch(wmpc_ctx* ctx) { CK(cudaGetLastError()); }

DevView view(const wmpc_ctx* c) {
  DevView d;
  d.n = c->n; d.H = c->H; d.nt = c->nt; d.nu = c->nu; d.nd = c->nd; d.ns = c->ns;
  d.W = c->W; d.P = c->P; d.lx = c->lx; d.ly = c->ly; d.Yc = c->Yc;
  d.a_identity = c->a_identity; d.w_scalar = c->w_scalar; d.w_c = c->w_c;
  d.stage_of = c->stage_of; d.anc = c->anc; d.cptr = c->cptr; d.cidx = c->cidx; d.prob = c->prob;
  d.A = c->A; d.At = c->At; d.Bt = c->Bt; d.Wu = c->Wu; d.T = c->T; d.Lam = c->Lam;
  d.Mb = c->Mb; d.Mf = c->Mf; d.E = c->E; d.e_pinv = c->e_pinv;
  d.np = c->d_np;
  d.econ = c->econ;
  d.xmin = c->xmin; d.xmax = c->xmax; d.xsafe = c->xsafe; d.umin = c->umin; d.umax = c->umax;
  d.p = c->p; d.q = c->q; d.w_x = c->w_x; d.w_s = c->w_s;
  d.Y0 = c->Y[0]; d.Y1 = c->Y[1]; d.Y2 = c->Y[2];
  d.U = c->U; d.X = c->X; d.Ua = c->Ua; d.Xa = c->Xa; d.wbar = c->wbar; d.lin = c->lin;
  d.theta = c->theta; d.beta = c->beta; d.iter = c->iter; d.bad_nu = c->bad_nu;
  d.gamma = c->gamma;
  d.acct = c->acct;
  return d;
}

int grid_for(size_t len, int threads = 256) {
  size_t b = (len + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 1184) b = 1184;
  return (int)b;
}

size_t smem_bwd(const wmpc_ctx* c, int s) {
  int K = c->nt + (s < c->H - 1 ? c->nu : 0);
  return sizeof(double) * (size_t)TM * (K + c->nu + c->nt);
}
size_t smem_fwd(const wmpc_ctx* c) {
  return sizeof(double) * ((size_t)TM * (2 * c->nu + c->nu + 2 * c->nt + c->W) + 2 * TM);
}

// Dual gradient over all stages: backward H..1 then forward 1..H.
void launch_dg(wmpc_ctx* ctx, const DevView& d, const double* ysrc, int mode) {
  for (int s = ctx->H - 1; s >= 0; --s) {
    int cnt = ctx->off[s + 1] - ctx->off[s];
    if (cnt <= 0) continue;
    k_bwd_stage<<<(cnt + TM - 1) / TM, NTHR, smem_bwd(ctx, s), ctx->stream>>>(d, s, ctx->off[s], cnt, ysrc);
  }
  for (int s = 0; s < ctx->H; ++s) {
    int cnt = ctx->off[s + 1] - ctx->off[s];
    if (cnt <= 0) continue;
    k_fwd_stage<<<(cnt + TM - 1) / TM, NTHR, smem_fwd(ctx), ctx->stream>>>(d, s, ctx->off[s], cnt, mode);
  }
  check_launch(ctx);
  ctx->launches += 2 * ctx->H;
}

// Sum-reduce the 4 cost terms of (Uin, Xin[, y]) -> host[4].
void cost_terms(wmpc_ctx* ctx, const DevView& d, const double* Uin, const double* Xin, const double* y,
                int pen, double out[4]) {
  int nb = std::min(ctx->part_blocks, std::max(1, (ctx->n + 7) / 8));
  ctx->launches++;
  k_cost_partial<<<nb, 256, 0, ctx->stream>>>(d, Uin, Xin, y, pen, ctx->part);
  ctx->launches++;
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 4, 0, 4, ctx->scal);
  check_launch(ctx);
  d2h(ctx, out, ctx->scal, 4 * sizeof(double));
  sync(ctx);
}

// Device-side variants for the certificate: results stay in device memory
// (out[0..3] cost terms; out[0] g* value, out[1] > 0 when y is outside dom g*)
// so the whole certificate needs one host round trip.
void cost_terms_dev(wmpc_ctx* ctx, const DevView& d, const double* Uin, const double* Xin, const double* y, int pen,
                    double* out) {
  int nb = std::min(ctx->part_blocks, std::max(1, (ctx->n + 7) / 8));
  ctx->launches += 2;
  k_cost_partial<<<nb, 256, 0, ctx->stream>>>(d, Uin, Xin, y, pen, ctx->part);
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 4, 0, 4, out);
}
void gconj_dev(wmpc_ctx* ctx, const DevView& d, const double* y, double* out) {
  int nb = std::min(ctx->part_blocks, std::max(1, (ctx->n + 7) / 8));
  ctx->launches += 3;
  k_gconj_partial<<<nb, 256, 0, ctx->stream>>>(d, y, 1e-9, ctx->part);
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 0, 1, out);
  k_finish<1><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 1, 1, out);
}

double gconj_value(wmpc_ctx* ctx, const DevView& d, const double* y) {
  int nb = std::min(ctx->part_blocks, std::max(1, (ctx->n + 7) / 8));
  ctx->launches++;
  k_gconj_partial<<<nb, 256, 0, ctx->stream>>>(d, y, 1e-9, ctx->part);
  ctx->launches++;
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 0, 1, ctx->scal);
  ctx->launches++;
  k_finish<1><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 1, 1, ctx->scal);
  check_launch(ctx);
  double h[2];
  d2h(ctx, h, ctx->scal, 2 * sizeof(double));
  sync(ctx);
  return h[1] > 0.0 ? INFINITY : h[0];
}

// Dykstra operators: CSR always; the structured path's ELL copy (width 4,
// zero-padded, the same entries) keeps them in registers across the sweeps.
DykOps dyk_ops(const wmpc_ctx* ctx) {
  DykOps po{ctx->pj_kp, ctx->pj_kc, ctx->pj_ecp, ctx->pj_ecr, ctx->pj_kv, ctx->pj_ecv, nullptr, nullptr, 0, 0, 0,
            ctx->dk_free, ctx->dk_nfree};
  if (ctx->fast && ctx->use_graphk && ctx->ell_idx && ctx->ell_w == 4) {
    po.eidx = ctx->ell_idx;
    po.eval = ctx->ell_val;
    po.ew = ctx->ell_w;
    po.ec0 = ctx->nu + ctx->nt;
    po.kr0 = 2 * ctx->nu + ctx->nt;
  }
  return po;
}

template <typename... A>
void launch_dyk(wmpc_ctx* ctx, int grid, const DykOps& po, A... args) {
  (void)grid;  // one warp per node, DYK_WPB nodes per CTA
  const int g = (ctx->n + DYK_WPB - 1) / DYK_WPB;
  if (po.eidx) k_dyk_warp<true><<<g, DYK_WPB * 32, 0, ctx->stream>>>(args...);
  else k_dyk_warp<false><<<g, DYK_WPB * 32, 0, ctx->stream>>>(args...);
}

void gconj_raw(wmpc_ctx* ctx, const DevView& d, const double* y, double out[2]) {
  int nb = std::min(ctx->part_blocks, std::max(1, (ctx->n + 7) / 8));
  ctx->launches += 3;
  k_gconj_partial<<<nb, 256, 0, ctx->stream>>>(d, y, 1e-9, ctx->part);
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 0, 1, ctx->scal);
  k_finish<1><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 1, 1, ctx->scal);
  check_launch(ctx);
  d2h(ctx, out, ctx->scal, 2 * sizeof(double));
  sync(ctx);
}

template <class T>
void upload_vec(wmpc_ctx* ctx, T** dst, const std::vector<T>& v) {
  if (*dst) cudaFree(*dst);
  *dst = nullptr;
  dalloc(ctx, dst, v.size());
  h2d(ctx, *dst, v.data(), sizeof(T) * v.size());
}

template <int MC>
void fast_attr(wmpc_ctx* ctx, size_t smem) {
  CK(cudaFuncSetAttribute(k_apg_fast<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

size_t fast_smem_bytes(const wmpc_ctx* c, int MC, int nrow, int rec, int cpc, int enz, int bnz) {
  const int nst = c->H - c->kstar, nu = c->nu, nt = c->nt, lx = c->lx, ns = c->ns;
  size_t dbl = (size_t)nrow * MC * rec + 2 * (size_t)MC * nu + 3 * (size_t)MC * lx + (size_t)MC * FAST_MAXNS +
               (size_t)MC * 2 * nt + 2 * MC + (3 * nt + 2 * nu) + (size_t)nu * ns + enz + 2 * (size_t)bnz;
  size_t ints = (ns + 1) + enz + (nu + 1) + bnz + (nt + 1) + bnz + (size_t)nrow * MC + c->H + 1 +
                (size_t)cpc * nst;
  return dbl * sizeof(double) + ints * sizeof(int) + 64;
}

// Decide whether the structured persistent kernel applies and lay out its data:
// A = I, W = cI, n_u even, n_s <= 32, and every stage factor equal to the
// null(E) projector (T_s = P/(2c), D_s = P up to 1e-12 relative).
// Launch with programmatic stream serialization (PDL) when enabled: the kernel
// may start while its predecessor drains; griddepcontrol.wait in the kernel
// orders the dependent loads (captured into the graph as programmatic edges).
template <typename... KArgs, typename... Args>
void launch_pdl(wmpc_ctx* ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

template <int WE, typename TG, int PD, bool RF>
void cw_attrs1(wmpc_ctx* ctx) {
  CK(cudaFuncSetAttribute(k_chain_up_w<WE, TG, PD, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(TG) * CW_WARPS * cw_up_warp(PD, !RF))));
  CK(cudaFuncSetAttribute(k_chain_down_w<WE, TG, PD, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(TG) * CW_WARPS * cw_dn_warp(PD))));
}
template <int WE, typename TG, int PD>
void cw_attrs(wmpc_ctx* ctx) {
  cw_attrs1<WE, TG, PD, true>(ctx);
  cw_attrs1<WE, TG, PD, false>(ctx);
}
template <int WE, typename TG, bool RF>
void cw_up_r(wmpc_ctx* ctx, const FastView& f) {
  const dim3 grid((ctx->nchain + CW_WARPS - 1) / CW_WARPS), block(CW_WARPS * 32);
  const size_t sm = sizeof(TG) * (CW_WARPS * cw_up_warp_r() + (CW_SMV ? CW_UP_SLOTS * 32 : 0));
  if (ctx->ell_vf) launch_pdl(ctx, k_chain_up_r<WE, TG, RF, 1, true>, grid, block, sm, f);
  else launch_pdl(ctx, k_chain_up_r<WE, TG, RF, 1, false>, grid, block, sm, f);
}
template <int WE, typename TG, bool RF>
void cw_down_r(wmpc_ctx* ctx, const FastView& f) {
  const dim3 grid((ctx->nchain + CW_WARPS - 1) / CW_WARPS), block(CW_WARPS * 32);
  const size_t sm = sizeof(TG) * (CW_WARPS * cw_dn_warp_r() + (CW_SMV ? CW_DN_SLOTS * 32 : 0));
  if (ctx->ell_vf) launch_pdl(ctx, k_chain_down_r<WE, TG, RF, 1, true>, grid, block, sm, f);
  else launch_pdl(ctx, k_chain_down_r<WE, TG, RF, 1, false>, grid, block, sm, f);
}
template <int WE, typename TG>
void gk_attrs_t(wmpc_ctx* ctx, size_t up, size_t down, size_t grp) {
  if constexpr (WE == 4 && sizeof(TG) == 8) cw_attrs<WE, TG, 8>(ctx);  // the ring: fp64 only
  CK(cudaFuncSetAttribute(k_chain_up<WE, TG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)up));
  CK(cudaFuncSetAttribute(k_chain_down<WE, TG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down));
  CK(cudaFuncSetAttribute(k_chain_up<WE, TG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)up));
  CK(cudaFuncSetAttribute(k_chain_down<WE, TG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down));
  CK(cudaFuncSetAttribute(k_branch_grp<WE, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grp));
  CK(cudaFuncSetAttribute(k_branch_grp<WE, TG, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)grp));
}
template <int WE>
void gk_attrs(wmpc_ctx* ctx, size_t up, size_t down, size_t grp) {
  CK(cudaFuncSetAttribute(k_chain_rollout<WE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(double) * (size_t)ctx->H * (ctx->nu + ctx->lx) + sizeof(int) * 32)));
  gk_attrs_t<WE, double>(ctx, up, down, grp);
  gk_attrs_t<WE, float>(ctx, up, down, grp);
}
template <int WE, typename TG, int PD>
void cw_up(wmpc_ctx* ctx, const FastView& f) {
  const dim3 grid((ctx->nchain + CW_WARPS - 1) / CW_WARPS), block(CW_WARPS * 32);
  const size_t sm = sizeof(TG) * CW_WARPS * cw_up_warp(PD, !f.rfree);
  if (f.rfree) launch_pdl(ctx, k_chain_up_w<WE, TG, PD, true>, grid, block, sm, f);
  else launch_pdl(ctx, k_chain_up_w<WE, TG, PD, false>, grid, block, sm, f);
}
template <int WE, typename TG, int PD>
void cw_down(wmpc_ctx* ctx, const FastView& f) {
  const dim3 grid((ctx->nchain + CW_WARPS - 1) / CW_WARPS), block(CW_WARPS * 32);
  const size_t sm = sizeof(TG) * CW_WARPS * cw_dn_warp(PD);
  if (f.rfree) launch_pdl(ctx, k_chain_down_w<WE, TG, PD, true>, grid, block, sm, f);
  else launch_pdl(ctx, k_chain_down_w<WE, TG, PD, false>, grid, block, sm, f);
}
template <int WE, typename TG = double>
void gk_up(wmpc_ctx* ctx, const FastView& f) {
  if constexpr (WE == 4)
    if (ctx->chainw && (sizeof(TG) == 8 || ctx->chainw32)) {
      // the 8-row cp.async ring (fp64, 16-byte .cg copies) or rows streamed
      // through registers; both bit-identical to the CTA kernels
      // (tests/test_gpu_fast_path.py). fp32 mode: registers only (round 1's
      // 8-byte cp.async.ca ring variant was deleted).
      if constexpr (sizeof(TG) == 8)
        if (ctx->cw_pd == 8) {
          cw_up<WE, TG, 8>(ctx, f);
          return;
        }
      if (f.rfree) cw_up_r<WE, TG, true>(ctx, f);
      else cw_up_r<WE, TG, false>(ctx, f);
      return;
    }
  if (ctx->chain_occ)
    launch_pdl(ctx, k_chain_up<WE, TG, true>, dim3(ctx->nchain), dim3(ctx->up_threads), ctx->sm_up, f);
  else
    launch_pdl(ctx, k_chain_up<WE, TG, false>, dim3(ctx->nchain), dim3(ctx->up_threads), ctx->sm_up, f);
}
bool dp_on(const wmpc_ctx* ctx);
// stage groups [g0, g1) of gk_groups (g1 < 0: to the end)
template <int WE, typename TG = double>
void gk_grp(wmpc_ctx* ctx, const FastView& f, int bump, int first_flags = 0, int g0 = 0, int g1 = -1) {
  const int ng = (int)ctx->gk_groups.size();
  for (int gi = g0; gi < (g1 < 0 ? ng : std::min(g1, ng)); ++gi) {
    const auto& g = ctx->gk_groups[gi];
    if (dp_on(ctx))  // 4-warp CTAs next to k_chain_dp
      launch_pdl(ctx, k_branch_grp<WE, TG, 128>, dim3(g.second), dim3(128), ctx->sm_grp128, f, g.first, bump,
                 (int)GRP_FULL | first_flags);
    else
      launch_pdl(ctx, k_branch_grp<WE, TG>, dim3(g.second), dim3(GRP_THREADS), ctx->sm_grp, f, g.first, bump,
                 (int)GRP_FULL | first_flags);
    bump = 0;
    first_flags = 0;
  }
}
// fp64 only: in fp32 mode the four-kernel graph measured faster (C4 200 vs 258 us)
bool dp_on(const wmpc_ctx* ctx) {
  return ctx->use_dp && !ctx->fp32 && ctx->shard_k < 0 && ctx->rfree;
}
void launch_dp(wmpc_ctx* ctx, const FastView& f) {  // fp64 only (dp_on)
  DpArgs a{(void*)ctx->dp_agg, (const void*)ctx->dp_putg, ctx->dp_cpw,
           dp_pro_w(ctx->kstar, ctx->nu, ctx->lx, ctx->dp_segm > 0), ctx->dp_segm, (void*)ctx->dp_aggu,
           (void*)ctx->dp_corr, (void*)ctx->dp_segx, ctx->dp_flag, (const void*)ctx->dp_auxs, ctx->dp_sib};
  const dim3 grid(ctx->dp_grid), block(ctx->dp_wpc * 32);
  launch_pdl(ctx, k_chain_dp<DP_NT, DP_NU, double>, grid, block, ctx->dp_sm, f, a);
}
template <int WE>
void gk_rep(wmpc_ctx* ctx, const FastView& f, int mode, int bump) {
  if (ctx->rep_group.second > 0)
    k_branch_grp<WE, double><<<ctx->rep_group.second, GRP_THREADS, ctx->sm_grp, ctx->stream>>>(
        f, ctx->rep_group.first, bump, mode);
}
template <int WE, typename TG = double>
void gk_down(wmpc_ctx* ctx, const FastView& f) {
  if constexpr (WE == 4)
    if (ctx->chainw && (sizeof(TG) == 8 || ctx->chainw32)) {
      if constexpr (sizeof(TG) == 8)
        if (ctx->cw_pd == 8) {
          cw_down<WE, TG, 8>(ctx, f);
          return;
        }
      if (f.rfree) cw_down_r<WE, TG, true>(ctx, f);
      else cw_down_r<WE, TG, false>(ctx, f);
      return;
    }
  if (ctx->chain_occ)
    launch_pdl(ctx, k_chain_down<WE, TG, true>, dim3(ctx->nchain), dim3(ctx->down_threads), ctx->sm_down, f);
  else
    launch_pdl(ctx, k_chain_down<WE, TG, false>, dim3(ctx->nchain), dim3(ctx->down_threads), ctx->sm_down, f);
}
template <typename TG>
void gk_prox(wmpc_ctx* ctx, const FastView& f) {
  if (ctx->prox_warp)
    launch_pdl(ctx, k_prox_warp<TG>, dim3((ctx->n + PW_ROWS - 1) / PW_ROWS), dim3(64 * PW_ROWS), 0, f);
  else
    k_prox_nodes<<<(ctx->n + SC_NPB - 1) / SC_NPB, SC_THREADS, ctx->sm_prox, ctx->stream>>>(f);
}
template <int WE, typename TG>
void gk_iteration(wmpc_ctx* ctx, const FastView& f) {
  gk_up<WE, TG>(ctx, f);
  gk_grp<WE, TG>(ctx, f, 1);
  gk_down<WE, TG>(ctx, f);
  gk_prox<TG>(ctx, f);
}

// Branching-region stage groups, bottom-up, with <= 32 items per row, and
// their item lists. Stages < k_rep (subtree sharding) form the replicated
// group: its in-group items are limited to the rows this rank accounts for
// (acct), its frontier is this rank's own stage-k_rep rows.
void build_groups(wmpc_ctx* ctx, int k_rep, const int* acct) {
  const int kstar = ctx->kstar;
  const std::vector<int>& off = ctx->off;
  const std::vector<int>& cptr = ctx->h_cptr;
  const std::vector<int>& cidx = ctx->h_cidx;
  const int nb = off[kstar];
  std::vector<int> stage(std::max(nb, 1), 0);
  for (int s = 0; s < kstar; ++s)
    for (int r = off[s]; r < off[s + 1]; ++r) stage[r] = s;
  auto items_of = [&](int r, int s_hi, std::vector<int>* it, std::vector<int>* wt) {
    int cnt = 0;
    std::vector<int> st(cidx.begin() + cptr[r], cidx.begin() + cptr[r + 1]);
    std::vector<int> dep(st.size(), 1);
    while (!st.empty()) {
      const int e = st.back(), de = dep.back();
      st.pop_back();
      dep.pop_back();
      const bool frontier = e >= off[s_hi + 1];
      const bool counted = frontier || !acct || acct[e];
      if (counted) ++cnt;
      if (it && counted) {
        it->push_back(e * 2 + (frontier ? 1 : 0));
        wt->push_back(frontier ? de - 1 : de);
      }
      if (!frontier)
        for (int c = cptr[e]; c < cptr[e + 1]; ++c) {
          st.push_back(cidx[c]);
          dep.push_back(de + 1);
        }
    }
    return cnt;
  };
  ctx->gk_groups.clear();
  ctx->rep_group = {0, 0};
  std::vector<int> gip(nb + 1, 0), gii, giw;
  std::vector<std::pair<int, int>> groups;  // (s_lo, s_hi), bottom-up
  int s_hi = kstar - 1;
  while (s_hi >= k_rep) {
    int s_lo = s_hi;
    while (s_lo > k_rep) {
      int mx = 0;
      for (int r = off[s_lo - 1]; r < off[s_lo]; ++r) mx = std::max(mx, items_of(r, s_hi, nullptr, nullptr));
      // a stage of few rows is latency-bound: more items per row cost less than one more kernel
      const int lim = off[s_lo] - off[s_lo - 1] <= ctx->sms ? ctx->grp_items_few : ctx->grp_items;
      if (mx > lim) break;
      --s_lo;
    }
    groups.push_back({s_lo, s_hi});
    s_hi = s_lo - 1;
  }
  std::vector<int> ghi(std::max(kstar, 1), 0);
  for (auto& g : groups)
    for (int st = g.first; st <= g.second; ++st) ghi[st] = g.second;
  for (int st = 0; st < k_rep; ++st) ghi[st] = k_rep - 1;  // replicated group, frontier = stage k_rep
  for (int r = 0; r < nb; ++r) {
    items_of(r, ghi[stage[r]], &gii, &giw);
    gip[r + 1] = (int)gii.size();
  }
  for (auto& g : groups) ctx->gk_groups.push_back({off[g.first], off[g.second + 1] - off[g.first]});
  if (k_rep > 0) ctx->rep_group = {0, off[k_rep]};
  if (gii.empty()) { gii.push_back(0); giw.push_back(0); }
  upload_vec(ctx, &ctx->gi_ptr, gip);
  upload_vec(ctx, &ctx->gi_item, gii);
  upload_vec(ctx, &ctx->gi_w, giw);
}

// Fused one-kernel iteration (k_chain_dp, wmpc_dp.cuh) for trees with many
// chains: persistent warps, DP_WPS warps per SM, each over cpw chains
// (strided: warp w takes chains w, w + NW, ...). Branching rows are owned
// (prox + Yc) by one chain below them, balanced over warps.
#ifndef DP_WPS
#define DP_WPS 7
#endif
void dp_attr(wmpc_ctx* ctx, size_t sm) {
  CK(cudaFuncSetAttribute(k_chain_dp<DP_NT, DP_NU, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
}
void configure_dp(wmpc_ctx* ctx) {
  ctx->use_dp = 0;
  ctx->dp_sib = 0;
  ctx->dp_segm = 0;
  const int nt = ctx->nt, nu = ctx->nu, lx = ctx->lx, nchain = ctx->nchain, kstar = ctx->kstar;
  const bool fits = ctx->ell_w == 4 && nt == DP_NT && nu == DP_NU && ctx->ns <= 32 && kstar <= 30;
  const int sms = std::max(ctx->sms, 1), N = ctx->H - kstar;
  // many chains per SM (C4: 4,096 chains, 27.7 per SM: 236 vs 256 us per iteration); at C3 (512 chains,
  // 3.5 per SM) one warp per whole chain is latency-bound (51 vs 52 us): segmented chains (two warps
  // per chain) where every pair fits in one wave
  // (measured, us per iteration: C3 graph 52.1, whole chains 50.0, segmented 42.5 with 10 of 19 rows
  // up; C2, 128 chains: graph 19.4, segmented 28.0, whole 42.2; 1,024 chains [4,4,4,4,2,2]: graph 95.8,
  // whole chains 62.4; [8,8,8,2]: 100.2 vs 63.8): k_chain_dp from 2 chains per SM
  const bool many = nchain >= 8 * sms;
  const bool few = 2 * nchain <= sms * DP_WPS && N >= 6 && kstar > 0;
  const bool seg_default = few && nchain >= 2 * sms;
  bool want = fits && nchain >= 2 * sms;
  if (const char* e = getenv("WMPC_DP")) want = fits && e[0] == '1';
  if (!want) return;
  int segm = few && !many && seg_default ? (N + 1) / 2 : 0;
  if (few && !many) {
    if (const char* e = getenv("WMPC_DP_SEG")) segm = e[0] == '1' ? (N + 1) / 2 : 0;
    if (const char* e = getenv("WMPC_DP_SEGM")) segm = std::min(std::max(atoi(e), 1), N - 1);
  }
  const int lanes = segm > 0 ? 2 : 1;  // warps per chain slot
  const int cpw = (lanes * nchain + sms * DP_WPS - 1) / (sms * DP_WPS);
  const int nw = lanes * ((nchain + cpw - 1) / cpw);
  const int wpc = std::min(DP_MAXT / 32, std::max(1, (nw + sms - 1) / sms));
  const int grid = (nw + wpc - 1) / wpc;
  if (segm > 0 && grid > sms) return;  // segments pay in one resident wave only (not reached: few chains)
  const size_t sm = dp_smem<double>(wpc, nt, nu, lx, kstar, segm > 0);
  if (sm > 227 * 1024) return;
  dp_attr(ctx, sm);
  // ownership of the branching rows balanced over the persistent warps
  const int nwt = grid * wpc, nb = ctx->off[kstar];
  if (kstar > 0) {
    std::vector<int> lo(nb, INT_MAX), hi(nb, -1), cntw(nwt, 0), cntc(nchain, 0);
    for (int i = 0; i < nchain; ++i)
      for (int m = 0; m < kstar; ++m) {
        const int a = ctx->h_cpath[(size_t)i * kstar + m];
        lo[a] = std::min(lo[a], i);
        hi[a] = std::max(hi[a], i + 1);
      }
    std::vector<unsigned> cown(nchain, 0u);
    for (int st = kstar - 1; st >= 0; --st)
      for (int a = ctx->off[st]; a < ctx->off[st + 1]; ++a) {
        if (hi[a] < 0) continue;
        int best = lo[a];
        for (int i = lo[a]; i < hi[a]; ++i) {
          const int ci = cntw[i / cpw], cb = cntw[best / cpw];
          if (ci < cb || (ci == cb && cntc[i] < cntc[best])) best = i;
        }
        cntw[best / cpw]++;
        cntc[best]++;
        cown[best] |= 1u << st;
      }
    upload_vec(ctx, &ctx->cown, cown);
    // the stage-(kstar-1) rows' up pass moves into k_chain_dp when each such
    // row's chains are all on one warp (contiguous chains per warp) and that
    // stage is exactly the first branch group (identical item lists)
    bool sib = segm == 0 && ctx->gk_groups.size() >= 2 && ctx->gk_groups[0].first == ctx->off[kstar - 1] &&
               ctx->gk_groups[0].second == ctx->off[kstar] - ctx->off[kstar - 1];
    for (int a = ctx->off[kstar - 1]; sib && a < ctx->off[kstar]; ++a)
      sib = hi[a] > 0 && lo[a] / cpw == (hi[a] - 1) / cpw;
    ctx->dp_sib = sib ? 1 : 0;
    if (const char* e = getenv("WMPC_DP_SIB")) ctx->dp_sib &= e[0] != '0';
  }
  const size_t aw = (size_t)nchain * dp_agg_w(nu, lx);
  for (double** p : {&ctx->dp_agg, &ctx->dp_putg, &ctx->dp_aggu, &ctx->dp_corr, &ctx->dp_segx, &ctx->dp_auxs}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (ctx->dp_flag) cudaFree(ctx->dp_flag);
  ctx->dp_flag = nullptr;
  dalloc(ctx, &ctx->dp_agg, aw);
  dalloc(ctx, &ctx->dp_putg, (size_t)std::max(nb, 1) * (nu + lx));
  if (segm > 0) {
    dalloc(ctx, &ctx->dp_aggu, aw);
    dalloc(ctx, &ctx->dp_corr, (size_t)nchain * 2 * nu);
    dalloc(ctx, &ctx->dp_segx, (size_t)nchain * DP_SXW(nu, lx));
    dalloc(ctx, &ctx->dp_auxs, (size_t)nchain * 4);
    CK(cudaMalloc(&ctx->dp_flag, sizeof(int) * nchain));
    CK(cudaMemset(ctx->dp_flag, 0, sizeof(int) * nchain));
  }
  ctx->dp_segm = segm;
  if (!ctx->dp_Lc) {
    dalloc(ctx, &ctx->dp_Lc, (size_t)ctx->n * nu);
    dalloc(ctx, &ctx->dp_wc, (size_t)ctx->n * lx);
  }
  if (ctx->dp_Ac) cudaFree(ctx->dp_Ac);
  ctx->dp_Ac = nullptr;
  dalloc(ctx, &ctx->dp_Ac, (size_t)(nb + nchain) * nu);
  ctx->dp_cpw = cpw;
  ctx->dp_wpc = wpc;
  ctx->dp_grid = grid;
  ctx->dp_sm = sm;
  ctx->use_dp = 1;
}

// Graph-of-kernels scan path: operator blob, stage groups of the branching
// region with per-row item lists, chain root paths. Default when it fits.
void configure_graphk(wmpc_ctx* ctx, const std::vector<int>& cptr, const std::vector<int>& cidx,
                      const std::vector<double>& ept, const std::vector<int>& ep, const std::vector<int>& ec,
                      const std::vector<double>& ev, const std::vector<int>& bcp, const std::vector<int>& bcr,
                      const std::vector<double>& bcv, const std::vector<int>& brp, const std::vector<int>& brc,
                      const std::vector<double>& brv, int enz, int bnz) {
  ctx->use_graphk = 0;
  if (ctx->gk_exec1) cudaGraphExecDestroy(ctx->gk_exec1);
  if (ctx->gk_exec8) cudaGraphExecDestroy(ctx->gk_exec8);
  ctx->gk_exec1 = ctx->gk_exec8 = nullptr;
  ctx->gk_gamma = -1.0;
  const char* ek = getenv("WMPC_KERNEL");
  if (ek && std::string(ek) != "graph") return;
  const int H = ctx->H, kstar = ctx->kstar, nst = H - kstar, nt = ctx->nt, nu = ctx->nu, ns = ctx->ns;
  const int lx = ctx->lx, ly = ctx->ly;
  if (H > SC_THREADS || kstar > SC_MAXK) return;
  const std::vector<int>& off = ctx->off;
  const int nb = off[kstar], nchain = off[kstar + 1] - off[kstar];
  // chains must be stage-major contiguous: row = nb + t * nchain + chain
  for (int i = 0; i < nchain; ++i) {
    int r = nb + i;
    for (int t = 1; t < nst; ++t) {
      if (cptr[r + 1] - cptr[r] != 1 || cidx[cptr[r]] != nb + t * nchain + i) return;
      r = cidx[cptr[r]];
    }
  }
  // sparse projector operands: K = (E E^T)^{-1} E = (E^+)^T (entries below
  // 1e-14 max|K| are rounding noise of the SVD), E by columns
  std::vector<int> kp(ns + 1, 0), kc, ecp(nu + 1, 0), ecr;
  std::vector<double> kv, ecv;
  {
    double kmax = 0.0;
    for (size_t i = 0; i < ept.size(); ++i) kmax = std::max(kmax, std::fabs(ept[i]));
    for (int i = 0; i < ns; ++i) {
      for (int k = 0; k < nu; ++k) {
        const double v = ept[(size_t)k * ns + i];
        if (std::fabs(v) > 1e-14 * kmax) {
          kc.push_back(k);
          kv.push_back(v);
        }
      }
      kp[i + 1] = (int)kc.size();
    }
    std::vector<std::vector<std::pair<int, double>>> cols(nu);
    for (int i = 0; i < ns; ++i)
      for (int e = ep[i]; e < ep[i + 1]; ++e) cols[ec[e]].push_back({i, ev[e]});
    for (int k = 0; k < nu; ++k) {
      for (auto& pr : cols[k]) {
        ecr.push_back(pr.first);
        ecv.push_back(pr.second);
      }
      ecp[k + 1] = (int)ecr.size();
    }
  }
  const int knz = (int)kc.size();
  ctx->fast_knz = knz;
  const BlobLayout bl = blob_layout(nt, nu, ns, knz, enz, bnz);
  const size_t cap = 227 * 1024;
  const size_t up = sizeof(double) * (size_t)nst * (ly + nu + 2 + FAST_MAXNS);
  const size_t grp = sizeof(double) * ((size_t)(GRP_THREADS / 32) * 256 + 2 * lx + 2 * nu + FAST_MAXNS);
  ctx->sm_grp128 = sizeof(double) * ((size_t)(128 / 32) * 256 + 2 * lx + 2 * nu + FAST_MAXNS);
  const size_t down = sizeof(double) * (size_t)H * (2 * nu + lx + FAST_MAXNS) + sizeof(int) * ((H + 3) & ~3);
  const size_t prox = sizeof(double) * ((size_t)SC_NPB * (ctx->fast_rec + nu + lx + 2) + 3 * nt + 2 * nu) +
                      sizeof(int) * SC_NPB + 16;
  if (std::max(std::max(up, down), std::max(grp, prox)) > cap) return;
  // operator blob
  std::vector<unsigned char> blob(bl.bytes, 0);
  {
    double* dp = reinterpret_cast<double*>(blob.data());
    int* ip = reinterpret_cast<int*>(blob.data());
    for (int e = 0; e < knz; ++e) { dp[bl.kv + e] = kv[e]; ip[bl.kcol + e] = kc[e]; }
    for (int i = 0; i <= ns; ++i) ip[bl.kptr + i] = kp[i];
    for (int e = 0; e < enz; ++e) { dp[bl.ecv + e] = ecv[e]; ip[bl.ecr + e] = ecr[e]; }
    for (int k = 0; k <= nu; ++k) ip[bl.ecp + k] = ecp[k];
    for (int e = 0; e < bnz; ++e) {
      dp[bl.bcv + e] = bcv[e]; ip[bl.bcr + e] = bcr[e];
      dp[bl.brv + e] = brv[e]; ip[bl.brc + e] = brc[e];
    }
    for (int j = 0; j <= nu; ++j) ip[bl.bcp + j] = bcp[j];
    for (int i = 0; i <= nt; ++i) ip[bl.brp + i] = brp[i];
  }
  upload_vec(ctx, &ctx->blob, blob);
  // ELL operators, owners [B cols | B rows | E cols | K rows], width = max entries per owner
  {
    std::vector<std::vector<std::pair<int, double>>> owners((size_t)2 * nu + nt + ns);
    for (int k = 0; k < nu; ++k)
      for (int e = bcp[k]; e < bcp[k + 1]; ++e) owners[k].push_back({bcr[e], bcv[e]});
    for (int j = 0; j < nt; ++j)
      for (int e = brp[j]; e < brp[j + 1]; ++e) owners[nu + j].push_back({brc[e], brv[e]});
    for (int k = 0; k < nu; ++k)
      for (int e = ecp[k]; e < ecp[k + 1]; ++e) owners[nu + nt + k].push_back({ecr[e], ecv[e]});
    for (int i = 0; i < ns; ++i)
      for (int e = kp[i]; e < kp[i + 1]; ++e) owners[2 * nu + nt + i].push_back({kc[e], kv[e]});
    size_t w = 1, wbc = 0, wbr = 0, wec = 0, wkr = 0;
    for (size_t o = 0; o < owners.size(); ++o) {
      const size_t c = owners[o].size();
      w = std::max(w, c);
      if (o < (size_t)nu) wbc = std::max(wbc, c);
      else if (o < (size_t)(nu + nt)) wbr = std::max(wbr, c);
      else if (o < (size_t)(2 * nu + nt)) wec = std::max(wec, c);
      else wkr = std::max(wkr, c);
    }
    if (w > 8) return;  // wide operators: the persistent kernels handle them
    // variant 4: per-operator widths (2, 3, 1, 4), stored with stride 4
    const int we = (wbc <= 2 && wbr <= 3 && wec <= 1 && wkr <= 4) ? 4 : 8;
    std::vector<int> cnt(owners.size()), idx(owners.size() * we, 0);
    std::vector<double> val(owners.size() * we, 0.0);
    for (size_t o = 0; o < owners.size(); ++o) {
      cnt[o] = (int)owners[o].size();
      for (size_t e = 0; e < owners[o].size(); ++e) {
        idx[o * we + e] = owners[o][e].first;
        val[o * we + e] = owners[o][e].second;
      }
    }
    upload_vec(ctx, &ctx->ell_cnt, cnt);
    upload_vec(ctx, &ctx->ell_idx, idx);
    upload_vec(ctx, &ctx->ell_val, val);
    // B and E values (owners before the K rows) exact in fp32: the warp chain
    // kernels store them as float in their shared operator table
    ctx->ell_vf = 1;
    for (size_t i = 0; i < (size_t)(2 * nu + nt) * we && i < val.size(); ++i)
      ctx->ell_vf &= (double)(float)val[i] == val[i];
    ctx->ell_w = we;
    ctx->ell_len = val.size();
  }
  ctx->h_cptr = cptr;
  ctx->h_cidx = cidx;
  // measured (us per iteration, 16 -> 64): C2 19.8 -> 22.6 (few chains: keep 16),
  // C3 52.4 -> 51.0, C4 269.7 -> 268.0
#ifndef GRP_FEW_CAP
#define GRP_FEW_CAP 32  // round 2, k_chain_dp paths (us per iteration, 64 -> 32): C3 42.8 -> 40.8, C4 191.7 -> 191.1
#endif
  ctx->grp_items_few = nchain > ctx->sms ? std::max(ctx->grp_items, GRP_FEW_CAP) : ctx->grp_items;
  build_groups(ctx, 0, nullptr);
  // chain root paths and ancestor ownership (first chain below a row writes it)
  std::vector<int> cpath((size_t)std::max(nchain * kstar, 1), 0);
  std::vector<unsigned> cown(nchain, 0u);
  if (kstar > 0) {
    std::vector<int> anc(ctx->n, -1);
    for (int r = 0; r < ctx->n; ++r)
      for (int c = cptr[r]; c < cptr[r + 1]; ++c) anc[cidx[c]] = r;
    // ownership: every branching row is written (U, X, prox) by one chain
    // below it, balanced so that a chain owns as few ancestors as possible
    std::vector<int> lo(nb, INT_MAX), hi(nb, -1), cnt(nchain, 0);
    for (int i = 0; i < nchain; ++i) {
      int a = anc[nb + i];
      for (int m = kstar - 1; m >= 0; --m) {
        cpath[(size_t)i * kstar + m] = a;
        lo[a] = std::min(lo[a], i);
        hi[a] = std::max(hi[a], i + 1);
        a = anc[a];
      }
    }
    for (int st = kstar - 1; st >= 0; --st)
      for (int a = off[st]; a < off[st + 1]; ++a) {
        if (hi[a] < 0) continue;
        int best = lo[a];
        for (int i = lo[a]; i < hi[a]; ++i)
          if (cnt[i] < cnt[best]) best = i;
        cnt[best]++;
        cown[best] |= 1u << st;
      }
  }
  ctx->h_cpath = cpath;
  upload_vec(ctx, &ctx->cpath, cpath);
  upload_vec(ctx, &ctx->cown, cown);
  std::vector<double> zl((size_t)ctx->n * nu, 0.0), za((size_t)(nb + nchain) * nu, 0.0);
  upload_vec(ctx, &ctx->Lb, zl);
  upload_vec(ctx, &ctx->Asub, za);
  if (ctx->Yc_save) cudaFree(ctx->Yc_save);
  ctx->Yc_save = nullptr;
  dalloc(ctx, &ctx->Yc_save, (size_t)ctx->n * ly);
  if (ctx->ut) cudaFree(ctx->ut);
  ctx->ut = nullptr;
  dalloc(ctx, &ctx->ut, (size_t)ctx->n * nu);
  if (ctx->ell_w == 4) gk_attrs<4>(ctx, up, down, grp);
  else gk_attrs<8>(ctx, up, down, grp);
  CK(cudaFuncSetAttribute(k_prox_nodes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prox));
  ctx->sm_up = up; ctx->sm_down = down; ctx->sm_grp = grp; ctx->sm_prox = prox;
  ctx->up_threads = ctx->down_threads = 512;  // measured: 512 beats 256 on C2 and C4
  ctx->chain_occ = ctx->nchain > 4 * ctx->sms ? 1 : 0;  // measured: C4 (4096 chains) +4 %; C2, C3 (<= 512) better without
  {  // warp-per-chain kernels (wmpc_chainw.cuh). Measured (us per iteration, CTA kernels ->
     // warp kernels): C2 128 chains 19.7 -> 27 (latency-bound: the CTA kernels run the
     // phases of all rows in parallel), C3 512 chains 55.4 -> 53.4 (8-row ring),
     // C4 4096 chains 331 -> 270 (ring of 2 or registers, equal; registers chosen).
    const bool fits = ctx->ell_w == 4 && nu <= 128 && nu % 2 == 0 && nt <= 64 && lx % 2 == 0 && ly % 2 == 0 &&
                      ctx->ns <= 32;
    const int wps = (ctx->nchain + ctx->sms - 1) / std::max(ctx->sms, 1);
    ctx->chainw = ctx->nchain > 2 * ctx->sms ? 1 : 0;
    ctx->cw_pd = wps <= 4 ? 8 : 1;
    // tests / tools force a variant: WMPC_CHAINW=0|1, WMPC_CWPD=1 (registers) | 8 (ring)
    if (const char* e = getenv("WMPC_CWPD")) ctx->cw_pd = atoi(e) >= 8 ? 8 : 1;
    // fp32 mode (register variant only): C3 47 (CTA) vs 52 us, C4 279 vs 226 us
    ctx->chainw32 = wps > 4 ? 1 : 0;
    if (const char* e = getenv("WMPC_CHAINW")) ctx->chainw = ctx->chainw32 = e[0] == '1';
    if (!fits) ctx->chainw = ctx->chainw32 = 0;
  }
  configure_dp(ctx);
  ctx->prox_warp = nt <= 64 && nu <= 128 ? 1 : 0;
  ctx->blob16 = bl.bytes / 16;
  ctx->n_branch = nb;
  ctx->use_graphk = 1;
}

void configure_fast(wmpc_ctx* ctx, const double* B, const double* E, const double* e_pinv, const double* T,
                    const double* D, const std::vector<int>& cptr, const std::vector<int>& cidx) {
  ctx->fast = false;
  const char* env = getenv("WMPC_DISABLE_FAST");
  if (env && env[0] == '1') return;
  const int H = ctx->H, nt = ctx->nt, nu = ctx->nu, ns = ctx->ns;
  if (!ctx->a_identity || !ctx->w_scalar || (nu % 2) || ns > FAST_MAXNS || ctx->w_c <= 0.0) return;
  if (nt > 64 || nu > 128 || ctx->W > 256 || (ctx->ly / 2) > 128) return;  // division-free layouts
  // projector check against the host recursion's factors
  std::vector<double> P((size_t)nu * nu);
  for (int i = 0; i < nu; ++i)
    for (int j = 0; j < nu; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < ns; ++k) s -= e_pinv[(size_t)i * ns + k] * E[(size_t)k * nu + j];
      P[(size_t)i * nu + j] = s;
    }
  const double c2 = 2.0 * ctx->w_c;
  for (int s = 0; s < H; ++s) {
    double tmax = 0.0, terr = 0.0, derr = 0.0;
    for (size_t k = 0; k < (size_t)nu * nu; ++k) {
      const double t = T[(size_t)s * nu * nu + k], dv = D[(size_t)s * nu * nu + k];
      tmax = std::max(tmax, std::fabs(t));
      terr = std::max(terr, std::fabs(t - P[k] / c2));
      derr = std::max(derr, std::fabs(dv - P[k]));
    }
    if (terr > 1e-12 * std::max(tmax, 1e-300) || derr > 1e-12) return;
  }
  // first chain stage: from the leaves up, stages whose nodes all have one child and equal counts
  const std::vector<int>& off = ctx->off;
  int kstar = H - 1;
  while (kstar > 0) {
    int s = kstar - 1;
    if (off[s + 1] - off[s] != off[s + 2] - off[s + 1]) break;
    bool ok = true;
    for (int r = off[s]; r < off[s + 1] && ok; ++r) ok = (cptr[r + 1] - cptr[r]) == 1;
    if (!ok) break;
    kstar = s;
  }
  kstar = std::max(kstar, std::min(ctx->kstar_min, H - 1));  // shards: replicated rows stay branching rows
  const int nchain = off[kstar + 1] - off[kstar];
  std::vector<int> chain((size_t)(H - kstar) * nchain);
  for (int i = 0; i < nchain; ++i) {
    int r = off[kstar] + i;
    for (int s = kstar; s < H; ++s) {
      chain[(size_t)(s - kstar) * nchain + i] = r;
      if (s + 1 < H) r = cidx[cptr[r]];
    }
  }
  // sparse B (both orientations) and E (rows)
  std::vector<int> bcp(nu + 1, 0), bcr, brp(nt + 1, 0), brc, ep(ns + 1, 0), ec;
  std::vector<double> bcv, brv, ev;
  for (int j = 0; j < nu; ++j) {
    for (int i = 0; i < nt; ++i)
      if (B[(size_t)i * nu + j] != 0.0) {
        bcr.push_back(i);
        bcv.push_back(B[(size_t)i * nu + j]);
      }
    bcp[j + 1] = (int)bcr.size();
  }
  for (int i = 0; i < nt; ++i) {
    for (int j = 0; j < nu; ++j)
      if (B[(size_t)i * nu + j] != 0.0) {
        brc.push_back(j);
        brv.push_back(B[(size_t)i * nu + j]);
      }
    brp[i + 1] = (int)brc.size();
  }
  for (int i = 0; i < ns; ++i) {
    for (int j = 0; j < nu; ++j)
      if (E[(size_t)i * nu + j] != 0.0) {
        ec.push_back(j);
        ev.push_back(E[(size_t)i * nu + j]);
      }
    ep[i + 1] = (int)ec.size();
  }
  const int bnz = (int)bcr.size(), enz = (int)ec.size();
  if (bcr.empty()) {
    bcr.push_back(0); bcv.push_back(0.0); brc.push_back(0); brv.push_back(0.0);
  }
  if (ec.empty()) {
    ec.push_back(0); ev.push_back(0.0);
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
  ctx->sms = sms;
  int cpc = (nchain + sms - 1) / sms;
  int MC = 1;
  while (MC < 8 && MC < cpc) MC *= 2;
  int ngroups = (cpc + MC - 1) / MC;
  int gs = (cpc + ngroups - 1) / ngroups;
  ctx->kstar = kstar;  // fast_smem_bytes reads it
  const int W = ctx->W, lx = ctx->lx, ly = ctx->ly;
  const int rec = std::max(ly + nu, 2 * W + 3 * nu + 2 * lx + 2);
  const size_t cap = 227 * 1024;
  int nrow = 0;
  for (int nr = 2; nr <= 8; ++nr)
    if (fast_smem_bytes(ctx, MC, nr, rec, cpc, enz, bnz) <= cap) nrow = nr;
  if (nrow < 2) return;
  size_t smem = fast_smem_bytes(ctx, MC, nrow, rec, cpc, enz, bnz);
  switch (MC) {
    case 1: fast_attr<1>(ctx, smem); break;
    case 2: fast_attr<2>(ctx, smem); break;
    case 4: fast_attr<4>(ctx, smem); break;
    default: fast_attr<8>(ctx, smem); break;
  }
  upload_vec(ctx, &ctx->chain_node, chain);
  upload_vec(ctx, &ctx->bc_ptr, bcp);
  upload_vec(ctx, &ctx->bc_row, bcr);
  upload_vec(ctx, &ctx->bc_val, bcv);
  upload_vec(ctx, &ctx->br_ptr, brp);
  upload_vec(ctx, &ctx->br_col, brc);
  upload_vec(ctx, &ctx->br_val, brv);
  upload_vec(ctx, &ctx->e_ptr, ep);
  upload_vec(ctx, &ctx->e_col, ec);
  upload_vec(ctx, &ctx->e_val, ev);
  upload_vec(ctx, &ctx->off_dev, off);
  {
    std::vector<double> aux((size_t)2 * ctx->n, 0.0);
    for (int r = 0; r < ctx->n; ++r) aux[2 * r] = 1.0 / (2.0 * ctx->w_c * ctx->prob_host[r]);
    upload_vec(ctx, &ctx->aux, aux);
  }
  ctx->nchain = nchain;
  ctx->fast_mc = MC;
  ctx->fast_cpc = cpc;
  ctx->fast_gs = gs;
  ctx->fast_grid = sms;  // one persistent CTA per SM
  ctx->fast_smem = smem;
  ctx->fast_nrow = nrow;
  ctx->fast_rec = rec;
  ctx->fast_enz = enz;
  ctx->fast_bnz = bnz;
  // scan-form kernel (default when the chain fits in shared memory)
  {
    const int nst = H - kstar;
    const size_t dA = (size_t)nst * (ly + nu + lx + nu + FAST_MAXNS);
    const size_t dD = (size_t)nst * (rec + nu + nu + lx + FAST_MAXNS) + nu + lx + 2 * nst;
    const size_t dB = (size_t)MC * rec + 2 * (size_t)MC * nu + 3 * (size_t)MC * lx + (size_t)MC * FAST_MAXNS +
                      (size_t)MC * 2 * nt + 2 * MC;
    const size_t work = std::max(dA, std::max(dD, dB));
    const size_t shared = (3 * nt + 2 * nu) + (size_t)nu * ns + enz + 2 * (size_t)bnz;
    const size_t ints = (ns + 1) + enz + (nu + 1) + bnz + (nt + 1) + bnz + std::max(MC, nst) + H + 1 +
                        (size_t)cpc * nst;
    const size_t bytes = (work + shared) * sizeof(double) + ints * sizeof(int) + 64;
    const char* ek = getenv("WMPC_KERNEL");
    const bool want = !(ek && (std::string(ek) == "cta" || std::string(ek) == "warp"));
    ctx->use_scan = 0;
    if (want && bytes <= cap && nst <= FAST_THREADS) {
      ctx->scan_work = (int)work;
      ctx->scan_smem = bytes;
      switch (MC) {
        case 1: CK(cudaFuncSetAttribute(k_apg_scan<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)); break;
        case 2: CK(cudaFuncSetAttribute(k_apg_scan<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)); break;
        case 4: CK(cudaFuncSetAttribute(k_apg_scan<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)); break;
        default: CK(cudaFuncSetAttribute(k_apg_scan<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)); break;
      }
      ctx->use_scan = 1;
    }
  }
  configure_graphk(ctx, cptr, cidx, std::vector<double>(e_pinv, e_pinv + (size_t)nu * ns), ep, ec, ev, bcp, bcr,
                   bcv, brp, brc, brv, enz, bnz);
  ctx->fast = true;
}

template <int MC>
void launch_scan_mc(wmpc_ctx* ctx, FastView& f) {
  void* args[] = {(void*)&f, (void*)&ctx->off_dev};
  CK(cudaLaunchCooperativeKernel((void*)k_apg_scan<MC>, dim3(ctx->fast_grid), dim3(FAST_THREADS), args,
                                 ctx->scan_smem, ctx->stream));
}

template <int MC>
void launch_fast_mc(wmpc_ctx* ctx, FastView& f) {
  void* args[] = {(void*)&f, (void*)&ctx->off_dev};
  CK(cudaLaunchCooperativeKernel((void*)k_apg_fast<MC>, dim3(ctx->fast_grid), dim3(FAST_THREADS), args,
                                 ctx->fast_smem, ctx->stream));
}

FastView make_fastview(wmpc_ctx* ctx, int count);

int graphk_kernels(const wmpc_ctx* ctx) {
  const int g = (int)ctx->gk_groups.size();
  if (ctx->shard_k > 0) return 3 + g + 2 * (ctx->rep_group.second > 0) + (g == 0 && ctx->rep_group.second == 0);
  if (dp_on(ctx)) return g - ctx->dp_sib + 1 + (g == 0 ? 1 : 0);
  return 3 + g + (g == 0 ? 1 : 0);
}

// One APG iteration of the graph-of-kernels path, enqueued on ctx->stream.
void enqueue_graphk_iteration(wmpc_ctx* ctx, const FastView& f) {
  cudaStream_t st = ctx->stream;
  if (ctx->gk_groups.empty()) k_advance<<<1, 32, 0, st>>>(ctx->iter);  // else the first group kernel counts
  if (dp_on(ctx)) {  // branch groups (the first reads Yc the previous k_chain_dp wrote) + k_chain_dp
    gk_grp<4, double>(ctx, f, 1, GRP_LATE, ctx->dp_sib);
    launch_dp(ctx, f);
    return;
  }
  if (ctx->fp32) {
    if (ctx->ell_w == 4) gk_iteration<4, float>(ctx, f); else gk_iteration<8, float>(ctx, f);
  } else {
    if (ctx->ell_w == 4) gk_iteration<4, double>(ctx, f); else gk_iteration<8, double>(ctx, f);
  }
}

void enqueue_shard_iteration(wmpc_ctx* ctx, const FastView& f);

void capture_graphk(wmpc_ctx* ctx) {
  if (ctx->shard_k > 0 && !ctx->nccl) return;  // host-mediated exchange: wmpc_shard_step, no graph
  if (ctx->gk_exec1 && ctx->gk_gamma == ctx->gamma && ctx->gk_maxit == ctx->max_iter) return;
  if (ctx->gk_exec1) cudaGraphExecDestroy(ctx->gk_exec1);
  if (ctx->gk_exec8) cudaGraphExecDestroy(ctx->gk_exec8);
  ctx->gk_exec1 = ctx->gk_exec8 = nullptr;
  FastView f = make_fastview(ctx, 1);
  for (int reps : {1, 8}) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    try {
      for (int i = 0; i < reps; ++i) {
        if (ctx->shard_k > 0) enqueue_shard_iteration(ctx, f);
        else enqueue_graphk_iteration(ctx, f);
      }
    } catch (Fail&) {  // leave the stream usable
      cudaStreamEndCapture(ctx->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(ctx->stream, &g));
    CK(cudaGraphInstantiate(reps == 1 ? &ctx->gk_exec1 : &ctx->gk_exec8, g, 0));
    cudaGraphDestroy(g);
  }
  ctx->gk_gamma = ctx->gamma;
  ctx->gk_maxit = ctx->max_iter;
}

void launch_graphk(wmpc_ctx* ctx, int count) {
  ctx->store_it_host = ctx->it_host + count - 1;  // U, X of the chunk's last iteration reach HBM
  CK(cudaMemcpyAsync(ctx->store_it, &ctx->store_it_host, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  int i = 0;
  for (; i + 8 <= count; i += 8) CK(cudaGraphLaunch(ctx->gk_exec8, ctx->stream));
  for (; i < count; ++i) CK(cudaGraphLaunch(ctx->gk_exec1, ctx->stream));
  ctx->launches += (int64_t)count * graphk_kernels(ctx);
}

// Dual-function minimiser z*(y) for the certificate (solver.py:454-456) with
// the chain/branch kernels: Yc is saved, replaced by collapse(y), and the
// up/branch/down passes write U, X into Uc, Xc. phase 0: up to the exchange
// point (sharded: partial sums in xbuf); phase 1: the rest; -1: both.
template <int WE>
void dual_eval_graph(wmpc_ctx* ctx, const double* y, int phase, double* Uout = nullptr, double* Xout = nullptr) {
  FastView f = make_fastview(ctx, 1);
  f.d.U = Uout ? Uout : ctx->Uc;
  f.d.X = Xout ? Xout : ctx->Xc;
  f.rfree = 0;  // the minimiser of an arbitrary y: the full form with R
  if (dp_on(ctx)) {  // L, subtree totals and wbar are k_chain_dp's iteration state: use scratch
    f.Lb = ctx->dp_Lc;
    f.Asub = ctx->dp_Ac;
    f.d.wbar = ctx->dp_wc;
  }
  const int nthr = 256;
  if (phase <= 0) {
    CK(cudaMemcpyAsync(ctx->Yc_save, ctx->Yc, sizeof(double) * (size_t)ctx->n * ctx->ly, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    k_collapse<<<grid_for((size_t)ctx->n * ctx->ly), nthr, 0, ctx->stream>>>(f.d, y, ctx->Yc);
    gk_up<WE>(ctx, f);
    gk_grp<WE>(ctx, f, 0);
    if (ctx->rep_group.second > 0) {
      CK(cudaMemsetAsync(ctx->xbuf, 0, sizeof(double) * 256 * (size_t)ctx->n_rep_global, ctx->stream));
      gk_rep<WE>(ctx, f, GRP_PARTIAL, 0);
    }
    ctx->launches += 2 + ctx->gk_groups.size() + (ctx->rep_group.second > 0);
  }
  if (phase != 0) {
    if (ctx->rep_group.second > 0) gk_rep<WE>(ctx, f, GRP_FINISH, 0);
    if (WE == 4 && ctx->chainw)
      gk_down<WE>(ctx, f);
    else if (ctx->chain_occ)
      k_chain_down<WE, double, true><<<ctx->nchain, ctx->down_threads, ctx->sm_down, ctx->stream>>>(f);
    else
      k_chain_down<WE, double, false><<<ctx->nchain, ctx->down_threads, ctx->sm_down, ctx->stream>>>(f);
    CK(cudaMemcpyAsync(ctx->Yc, ctx->Yc_save, sizeof(double) * (size_t)ctx->n * ctx->ly, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    ctx->launches += 1 + (ctx->rep_group.second > 0);
  }
  check_launch(ctx);
}

// Dual-function minimiser (U, X) of a device-resident y for the public
// dual_gradient and the power iteration: the graph kernels when the
// structured path is bound (one launch per kernel of the iteration graph
// instead of 2H per-stage launches), the general per-stage kernels otherwise.
void dual_gradient_dev(wmpc_ctx* ctx, const double* y, double* Uout, double* Xout) {
  if (ctx->fast && ctx->use_graphk && ctx->shard_k < 0) {
    if (ctx->ell_w == 4) dual_eval_graph<4>(ctx, y, -1, Uout, Xout);
    else dual_eval_graph<8>(ctx, y, -1, Uout, Xout);
    return;
  }
  DevView d = view(ctx);
  d.U = Uout;
  d.X = Xout;
  launch_dg(ctx, d, y, 0);
}

// x from u along every root path: one chain-parallel launch in graph mode
// (H <= 32), else one launch per stage.
void rollout(wmpc_ctx* ctx, const DevView& d, const double* U, double* X) {
  if (ctx->fast && ctx->use_graphk && ctx->H <= 32) {
    FastView f = make_fastview(ctx, 1);
    const size_t smem = sizeof(double) * (size_t)ctx->H * (ctx->nu + ctx->lx) + sizeof(int) * 32;
    ctx->launches++;
    if (ctx->ell_w == 4)
      k_chain_rollout<4><<<ctx->nchain, 256, smem, ctx->stream>>>(f, U, X);
    else
      k_chain_rollout<8><<<ctx->nchain, 256, smem, ctx->stream>>>(f, U, X);
    return;
  }
  for (int s = 0; s < ctx->H; ++s) {
    int cnt = ctx->off[s + 1] - ctx->off[s];
    ctx->launches++;
    k_rollout_stage<<<grid_for((size_t)cnt * ctx->nt), 256, 0, ctx->stream>>>(d, ctx->off[s], cnt, U, X);
  }
}

FastView make_fastview(wmpc_ctx* ctx, int count) {
  FastView f;
  f.d = view(ctx);
  f.kstar = ctx->kstar;
  f.nchain = ctx->nchain;
  f.chain_node = ctx->chain_node;
  f.bc_ptr = ctx->bc_ptr; f.bc_row = ctx->bc_row; f.bc_val = ctx->bc_val;
  f.br_ptr = ctx->br_ptr; f.br_col = ctx->br_col; f.br_val = ctx->br_val;
  f.e_ptr = ctx->e_ptr; f.e_col = ctx->e_col; f.e_val = ctx->e_val;
  f.aux = ctx->aux;
  f.e_nnz = ctx->fast_enz;
  f.b_nnz = ctx->fast_bnz;
  f.k_nnz = ctx->fast_knz;
  f.inv_2c = 1.0 / (2.0 * ctx->w_c);
  f.inv_gamma = 1.0 / ctx->gamma;
  f.cpc = ctx->fast_cpc;
  f.gs = ctx->fast_gs;
  f.nrow = ctx->fast_nrow;
  f.rec = ctx->fast_rec;
  f.max_iter = ctx->max_iter;
  f.count = count;
  f.store_uv = 1;
  f.prof = ctx->prof_on ? ctx->prof : nullptr;
  f.n_branch = ctx->n_branch;
  f.Lb = ctx->Lb;
  f.Asub = ctx->Asub;
  f.blob = reinterpret_cast<const double*>(ctx->blob);
  f.blob16 = ctx->blob16;
  f.gi_ptr = ctx->gi_ptr; f.gi_item = ctx->gi_item; f.gi_w = ctx->gi_w;
  f.cpath = ctx->cpath;
  f.cown = ctx->cown;
  f.store_it = ctx->store_it;
  f.ell_cnt = ctx->ell_cnt;
  f.ell_idx = ctx->ell_idx;
  f.ell_val = ctx->ell_val;
  f.ell_w = ctx->ell_w;
  f.lb_prewait = ctx->gk_groups.empty() ? 0 : 1;
  f.rfree = ctx->rfree && ctx->shard_k < 0 ? 1 : 0;
  f.ut = ctx->ut;
  f.ut32 = ctx->ut32;
  f.g32 = G32{ctx->f32_Yc, ctx->f32_Lb, ctx->f32_Asub, ctx->f32_wbar, ctx->f32_U, ctx->f32_X,
              ctx->f32_eoff, ctx->f32_R, ctx->f32_g, ctx->f32_aux, ctx->f32_ell};
  f.xbuf = ctx->xbuf;
  f.rep_gidx = ctx->rep_gidx;
  f.work_doubles = ctx->scan_work;
  return f;
}

void launch_fast(wmpc_ctx* ctx, int count) {
  if (ctx->use_graphk) {
    launch_graphk(ctx, count);
    return;
  }
  FastView f = make_fastview(ctx, count);
  if (ctx->use_scan) {
    f.work_doubles = ctx->scan_work;
    switch (ctx->fast_mc) {
      case 1: launch_scan_mc<1>(ctx, f); break;
      case 2: launch_scan_mc<2>(ctx, f); break;
      case 4: launch_scan_mc<4>(ctx, f); break;
      default: launch_scan_mc<8>(ctx, f); break;
    }
    ctx->launches += 1;
    return;
  }
  switch (ctx->fast_mc) {
    case 1: launch_fast_mc<1>(ctx, f); break;
    case 2: launch_fast_mc<2>(ctx, f); break;
    case 4: launch_fast_mc<4>(ctx, f); break;
    default: launch_fast_mc<8>(ctx, f); break;
  }
  ctx->launches += 1;
}

void point_nodes(wmpc_ctx* ctx, wmpc_nodes* nd) {
  NodePtrs h{nd->e_off, nd->R, nd->g, nd->shift, nd->ebar};
  CK(cudaMemcpyAsync(ctx->d_np, &h, sizeof(NodePtrs), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->nodes = nd;
}

template <class F>
int run(wmpc_ctx* ctx, F&& f) {
  if (!ctx) {
    g_global_err = "null context";
    return WMPC_E_ARG;
  }
  try {
    return f();
  } catch (Fail&) {
    return WMPC_E_CUDA;
  }
}

void free_all(wmpc_ctx* c) {
  void* ptrs[] = {c->stage_of, c->anc, c->cptr, c->cidx, c->prob, c->A, c->At, c->Bt, c->Wu, c->T,
                  c->Lam, c->Mb, c->Mf, c->E, c->e_pinv, c->econ, c->tmp, c->demand, c->Ed, c->xmin, c->xmax, c->xsafe, c->umin, c->umax,
                  c->p, c->q, c->Y[0], c->Y[1], c->Y[2], c->U, c->X, c->Ua, c->Xa, c->Uc, c->Xc,
                  c->Uf, c->Xf, c->U0, c->X0, c->wbar, c->lin, c->Yc, c->ys, c->gv, c->vv, c->zbuf,
                  c->theta, c->beta, c->iter, c->bad_nu,
                  c->bad_row, c->part, c->scal, c->d_np, c->chain_node,
                  c->bc_ptr, c->bc_row, c->br_ptr, c->br_col, c->off_dev, c->bc_val, c->br_val,
                  c->e_ptr, c->e_col, c->e_val, c->aux,
                  c->Lb, c->Asub, c->blob, c->store_it, c->ut, c->ut32, c->f32_Yc, c->f32_Lb, c->f32_Asub, c->f32_wbar, c->f32_U,
                  c->f32_X, c->f32_eoff, c->f32_R, c->f32_g, c->f32_aux, c->f32_ell, c->Yc_save, c->acct, c->rep_gidx, c->ell_cnt, c->ell_idx, c->ell_val, c->pj_kp, c->pj_kc, c->pj_ecp, c->pj_ecr, c->pj_kv,
                  c->pj_ecv, c->dk_mv, c->dk_sweeps, c->dk_fix, c->dk_list, c->dk_free, c->gi_ptr, c->gi_item, c->gi_w, c->cpath, c->cown,
                  c->prof, c->rb_u0, c->rb_p, c->rb_a, c->gd_stage, c->dp_agg, c->dp_putg, c->dp_aggu, c->dp_corr, c->dp_segx, c->dp_auxs, c->dp_flag, c->dp_Lc,
                  c->dp_Ac, c->dp_wc};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->nccl) nccl_api().destroy(c->nccl);
  if (c->gk_exec1) cudaGraphExecDestroy(c->gk_exec1);
  if (c->gk_exec8) cudaGraphExecDestroy(c->gk_exec8);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev2) cudaEventDestroy(c->ev2);
  if (c->ev3) cudaEventDestroy(c->ev3);
  if (c->stream_rd) {
    cudaStreamSynchronize(c->stream_rd);
    cudaStreamDestroy(c->stream_rd);
  }
  if (c->ev_rd) cudaEventDestroy(c->ev_rd);
  if (c->stream) cudaStreamDestroy(c->stream);
}

template <int WE>
void shard_phase(wmpc_ctx* ctx, const FastView& f, int phase) {
  const bool rep = ctx->rep_group.second > 0;
  if (phase == 0) {
    int bump = 1;
    if (ctx->gk_groups.empty() && !rep) {
      k_advance<<<1, 32, 0, ctx->stream>>>(ctx->iter);
      bump = 0;
    }
    gk_up<WE>(ctx, f);
    gk_grp<WE>(ctx, f, bump);
    if (rep) {
      CK(cudaMemsetAsync(ctx->xbuf, 0, sizeof(double) * 256 * (size_t)ctx->n_rep_global, ctx->stream));
      gk_rep<WE>(ctx, f, GRP_PARTIAL, ctx->gk_groups.empty() ? 1 : 0);
    }
    ctx->launches += 1 + ctx->gk_groups.size() + rep;
  } else {
    if (rep) gk_rep<WE>(ctx, f, GRP_FINISH, 0);
    gk_down<WE>(ctx, f);
    gk_prox<double>(ctx, f);
    ctx->launches += 2 + rep;
  }
  check_launch(ctx);
}

// The exchange on the device: sum of the ranks' buffers (in place) over NCCL.
void exchange_dev(wmpc_ctx* ctx) {
  NcclApi& api = nccl_api();
  const ncclResult_t r = api.all_reduce(ctx->xbuf, ctx->xbuf, (size_t)256 * ctx->n_rep_global, ncclDouble, ncclSum,
                                        ctx->nccl, ctx->stream);
  if (r != ncclSuccess) {
    ctx->err = std::string("NCCL all-reduce failed: ") + api.error_string(r);
    throw Fail{};
  }
}

// One sharded APG iteration with the exchange on the stream (graph-capturable).
void enqueue_shard_iteration(wmpc_ctx* ctx, const FastView& f) {
  if (ctx->ell_w == 4) shard_phase<4>(ctx, f, 0);
  else shard_phase<8>(ctx, f, 0);
  if (ctx->rep_group.second > 0) exchange_dev(ctx);
  if (ctx->ell_w == 4) shard_phase<4>(ctx, f, 1);
  else shard_phase<8>(ctx, f, 1);
}

}  // namespace

extern "C" {

const char* wmpc_global_error(void) { return g_global_err.c_str(); }

const char* wmpc_last_error(const wmpc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int wmpc_create(const wmpc_dims* dims, wmpc_ctx** out) {
  if (!dims || !out) {
    g_global_err = "null argument";
    return WMPC_E_ARG;
  }
  if (dims->n_nodes < 1 || dims->horizon < 1 || dims->n_tanks < 1 || dims->n_inputs < 1 ||
      dims->n_demands < 0 || dims->n_mixing < 0 || dims->n_mixing > 32 || dims->n_nodes > (1LL << 30)) {
    g_global_err = "invalid dimensions (need n>=1, H>=1, nt>=1, nu>=1, 0<=ns<=32)";
    return WMPC_E_ARG;
  }
  wmpc_ctx* ctx = new wmpc_ctx();
  try {
    ctx->dev = dims->device;
    CK(cudaSetDevice(ctx->dev));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    CK(cudaEventCreate(&ctx->ev2));
    CK(cudaEventCreate(&ctx->ev3));
    ctx->n = (int)dims->n_nodes; ctx->H = dims->horizon; ctx->nt = dims->n_tanks;
    ctx->nu = dims->n_inputs; ctx->nd = dims->n_demands; ctx->ns = dims->n_mixing;
    ctx->W = 2 * ctx->nt + ctx->nu; ctx->P = ctx->nu + ctx->nt;
    ctx->lx = ctx->nt + (ctx->nt & 1); ctx->ly = ctx->lx + ctx->nu;
    const size_t n = ctx->n, nt = ctx->nt, nu = ctx->nu, H = ctx->H, W = ctx->W, lx = ctx->lx;
    dalloc(ctx, &ctx->stage_of, n); dalloc(ctx, &ctx->anc, n); dalloc(ctx, &ctx->cptr, n + 1);
    dalloc(ctx, &ctx->cidx, n); dalloc(ctx, &ctx->prob, n);
    dalloc(ctx, &ctx->A, nt * nt); dalloc(ctx, &ctx->At, nt * nt); dalloc(ctx, &ctx->Bt, nu * nt);
    dalloc(ctx, &ctx->Wu, nu * nu); dalloc(ctx, &ctx->T, H * nu * nu); dalloc(ctx, &ctx->Lam, H * nu * nu);
    dalloc(ctx, &ctx->Mb, H * (nt + nu) * nu); dalloc(ctx, &ctx->Mf, H * 2 * nu * nu);
    dalloc(ctx, &ctx->E, (size_t)ctx->ns * nu); dalloc(ctx, &ctx->e_pinv, nu * ctx->ns);
    dalloc(ctx, &ctx->econ, n * nu); dalloc(ctx, &ctx->tmp, n * nu);
    dalloc(ctx, &ctx->demand, n * ctx->nd); dalloc(ctx, &ctx->Ed, (size_t)ctx->ns * ctx->nd);
    dalloc(ctx, &ctx->xmin, nt); dalloc(ctx, &ctx->xmax, nt); dalloc(ctx, &ctx->xsafe, nt);
    dalloc(ctx, &ctx->umin, nu); dalloc(ctx, &ctx->umax, nu); dalloc(ctx, &ctx->p, nt); dalloc(ctx, &ctx->q, nu);
    for (int k = 0; k < 3; ++k) dalloc(ctx, &ctx->Y[k], n * W);
    dalloc(ctx, &ctx->U, n * nu); dalloc(ctx, &ctx->X, n * lx); dalloc(ctx, &ctx->Ua, n * nu);
    dalloc(ctx, &ctx->Xa, n * lx); dalloc(ctx, &ctx->Uc, n * nu); dalloc(ctx, &ctx->Xc, n * lx);
    dalloc(ctx, &ctx->Uf, n * nu); dalloc(ctx, &ctx->Xf, n * lx); dalloc(ctx, &ctx->U0, n * nu);
    dalloc(ctx, &ctx->X0, n * lx); dalloc(ctx, &ctx->wbar, n * lx); dalloc(ctx, &ctx->lin, n * nu);
    dalloc(ctx, &ctx->Yc, n * ctx->ly);
    dalloc(ctx, &ctx->ys, n * W); dalloc(ctx, &ctx->gv, n * W); dalloc(ctx, &ctx->vv, n * W);
    dalloc(ctx, &ctx->zbuf, n * std::max(W, (size_t)ctx->P));
    dalloc(ctx, &ctx->iter, 1); dalloc(ctx, &ctx->bad_nu, 1); dalloc(ctx, &ctx->bad_row, 1);
    dalloc(ctx, &ctx->store_it, 1);
    dalloc(ctx, &ctx->d_np, 1);
    ctx->part_blocks = 1184;
    dalloc(ctx, &ctx->part, (size_t)ctx->part_blocks * 4);
    dalloc(ctx, &ctx->scal, 32);  // [0,8) general, [8] Dykstra tol, [16,26) certificate terms
    size_t smax = std::max(smem_fwd(ctx), smem_bwd(ctx, 0));
    if (smax > 48 * 1024) {
      CK(cudaFuncSetAttribute(k_fwd_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
      CK(cudaFuncSetAttribute(k_bwd_stage, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
    }
    sync(ctx);
  } catch (Fail&) {
    g_global_err = ctx->err;
    free_all(ctx);
    delete ctx;
    return WMPC_E_CUDA;
  }
  *out = ctx;
  return WMPC_OK;
}

void wmpc_destroy(wmpc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_all(ctx);
  delete ctx;
}

int wmpc_set_structure(wmpc_ctx* ctx, const double* A, const double* B, const double* Wu,
                       const double* T, const double* D, const double* Lam, const int64_t* anc_row,
                       const int64_t* stage_off, const double* prob, const double* E,
                       const double* e_pinv) {
  return run(ctx, [&]() -> int {
    ARG(A && B && Wu && T && D && Lam && anc_row && stage_off && prob, "null structure argument");
    const int n = ctx->n, H = ctx->H, nt = ctx->nt, nu = ctx->nu, ns = ctx->ns;
    ARG(stage_off[0] == 0 && stage_off[H] == n, "stage offsets must span all rows");
    ctx->off.assign(H + 1, 0);
    std::vector<int> stg(n), anc(n);
    for (int s = 0; s < H; ++s) {
      ARG(stage_off[s + 1] >= stage_off[s], "stage offsets must be nondecreasing");
      ctx->off[s + 1] = (int)stage_off[s + 1];
      for (int64_t r = stage_off[s]; r < stage_off[s + 1]; ++r) stg[r] = s;
    }
    for (int r = 0; r < n; ++r) {
      int64_t a = anc_row[r];
      if (stg[r] == 0) {
        ARG(a == -1, "stage-1 rows must have ancestor row -1");
      } else {
        ARG(a >= ctx->off[stg[r] - 1] && a < ctx->off[stg[r]], "ancestor must sit one stage up");
      }
      anc[r] = (int)a;
    }
    // CSR children, ascending child row (np.add.at order, solver.py:269-274).
    std::vector<int> cnt(n + 1, 0), cptr(n + 1, 0), cidx(n, 0);
    for (int r = 0; r < n; ++r)
      if (anc[r] >= 0) cnt[anc[r]]++;
    for (int r = 0; r < n; ++r) cptr[r + 1] = cptr[r] + cnt[r];
    std::vector<int> fill(cptr.begin(), cptr.end() - 1);
    for (int r = 0; r < n; ++r)
      if (anc[r] >= 0) cidx[fill[anc[r]]++] = r;
    // flags
    bool aid = true;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nt; ++j) aid &= A[i * nt + j] == (i == j ? 1.0 : 0.0);
    bool wsc = true;
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nu; ++j) wsc &= (i == j) ? Wu[i * nu + j] == Wu[0] : Wu[i * nu + j] == 0.0;
    ctx->a_identity = aid;
    ctx->w_scalar = wsc;
    ctx->w_c = Wu[0];
    std::vector<double> At(nt * nt), Bt((size_t)nu * nt);
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nt; ++j) At[j * nt + i] = A[i * nt + j];
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nu; ++j) Bt[(size_t)j * nt + i] = B[(size_t)i * nu + j];
    // Mb_s = [[B],[D_{s+1}]] ; Mf_s = [[D_s^T],[-T_s]]
    std::vector<double> Mb((size_t)H * (nt + nu) * nu, 0.0), Mf((size_t)H * 2 * nu * nu);
    for (int s = 0; s < H; ++s) {
      double* mb = Mb.data() + (size_t)s * (nt + nu) * nu;
      std::memcpy(mb, B, sizeof(double) * nt * nu);
      if (s + 1 < H) std::memcpy(mb + (size_t)nt * nu, D + (size_t)(s + 1) * nu * nu, sizeof(double) * nu * nu);
      double* mf = Mf.data() + (size_t)s * 2 * nu * nu;
      const double* Ds = D + (size_t)s * nu * nu;
      const double* Ts = T + (size_t)s * nu * nu;
      for (int k = 0; k < nu; ++k)
        for (int c = 0; c < nu; ++c) {
          mf[(size_t)k * nu + c] = Ds[(size_t)c * nu + k];
          mf[(size_t)(nu + k) * nu + c] = -Ts[(size_t)k * nu + c];
        }
    }
    h2d(ctx, ctx->stage_of, stg.data(), sizeof(int) * n);
    h2d(ctx, ctx->anc, anc.data(), sizeof(int) * n);
    h2d(ctx, ctx->cptr, cptr.data(), sizeof(int) * (n + 1));
    h2d(ctx, ctx->cidx, cidx.data(), sizeof(int) * n);
    h2d(ctx, ctx->prob, prob, sizeof(double) * n);
    ctx->prob_host.assign(prob, prob + n);
    h2d(ctx, ctx->A, A, sizeof(double) * nt * nt);
    h2d(ctx, ctx->At, At.data(), sizeof(double) * nt * nt);
    h2d(ctx, ctx->Bt, Bt.data(), sizeof(double) * nu * nt);
    h2d(ctx, ctx->Wu, Wu, sizeof(double) * nu * nu);
    h2d(ctx, ctx->T, T, sizeof(double) * H * nu * nu);
    h2d(ctx, ctx->Lam, Lam, sizeof(double) * H * nu * nu);
    h2d(ctx, ctx->Mb, Mb.data(), sizeof(double) * Mb.size());
    h2d(ctx, ctx->Mf, Mf.data(), sizeof(double) * Mf.size());
    if (ns > 0) {
      ARG(E && e_pinv, "E and e_pinv required when n_mixing > 0");
      h2d(ctx, ctx->E, E, sizeof(double) * ns * nu);
      h2d(ctx, ctx->e_pinv, e_pinv, sizeof(double) * nu * ns);
    }
    if (ns > 0) {  // sparse projector for the certificate's Dykstra (and the graph kernels)
      std::vector<int> kp(ns + 1, 0), kc, ecp(nu + 1, 0), ecr;
      std::vector<double> kv, ecv;
      double kmax = 0.0;
      for (size_t i = 0; i < (size_t)nu * ns; ++i) kmax = std::max(kmax, std::fabs(e_pinv[i]));
      for (int i = 0; i < ns; ++i) {
        for (int k = 0; k < nu; ++k) {
          const double v = e_pinv[(size_t)k * ns + i];
          if (std::fabs(v) > 1e-14 * kmax) {
            kc.push_back(k);
            kv.push_back(v);
          }
        }
        kp[i + 1] = (int)kc.size();
      }
      for (int k = 0; k < nu; ++k) {
        for (int i = 0; i < ns; ++i)
          if (E[(size_t)i * nu + k] != 0.0) {
            ecr.push_back(i);
            ecv.push_back(E[(size_t)i * nu + k]);
          }
        ecp[k + 1] = (int)ecr.size();
      }
      if (kc.empty()) { kc.push_back(0); kv.push_back(0.0); }
      if (ecr.empty()) { ecr.push_back(0); ecv.push_back(0.0); }
      upload_vec(ctx, &ctx->pj_kp, kp);
      upload_vec(ctx, &ctx->pj_kc, kc);
      upload_vec(ctx, &ctx->pj_kv, kv);
      upload_vec(ctx, &ctx->pj_ecp, ecp);
      upload_vec(ctx, &ctx->pj_ecr, ecr);
      upload_vec(ctx, &ctx->pj_ecv, ecv);
      if (!ctx->dk_mv) dalloc(ctx, &ctx->dk_mv, 512);
      if (!ctx->dk_sweeps) dalloc(ctx, &ctx->dk_sweeps, 1);
      if (!ctx->dk_fix) dalloc(ctx, &ctx->dk_fix, (size_t)n * std::max(ctx->ns, 1));  // per node or (node, row)
      if (!ctx->dk_list) dalloc(ctx, &ctx->dk_list, (size_t)n * std::max(ctx->ns, 1) + 1);  // [count | blocks]
      {
        std::vector<int> fr;
        for (int k = 0; k < nu; ++k)
          if (ecp[k + 1] == ecp[k]) fr.push_back(k);
        ctx->dk_nfree = (int)fr.size();
        if (fr.empty()) fr.push_back(0);
        upload_vec(ctx, &ctx->dk_free, fr);
      }
    }
    sync(ctx);
    configure_fast(ctx, B, E, e_pinv, T, D, cptr, cidx);
    ctx->graph_gamma = -1.0;
    sync(ctx);
    ctx->have_structure = true;
    return WMPC_OK;
  });
}

int wmpc_nodes_create(wmpc_ctx* ctx, wmpc_nodes** out) {
  return run(ctx, [&]() -> int {
    ARG(out, "null argument");
    wmpc_nodes* nd = new wmpc_nodes();
    nd->dev = ctx->dev;
    nd->n = ctx->n;
    const size_t n = ctx->n;
    try {
      dalloc(ctx, &nd->u_part, n * ctx->nu);
      dalloc(ctx, &nd->e_off, n * ctx->nu);
      dalloc(ctx, &nd->R, n * ctx->nu);
      dalloc(ctx, &nd->shift, n * ctx->ns);
      dalloc(ctx, &nd->g, n * ctx->lx);
      dalloc(ctx, &nd->ebar, n * ctx->nu);
    } catch (Fail&) {
      wmpc_nodes_destroy(nd);
      throw;
    }
    *out = nd;
    return WMPC_OK;
  });
}

void wmpc_nodes_destroy(wmpc_nodes* nd) {
  if (!nd) return;
  cudaSetDevice(nd->dev);
  void* ptrs[] = {nd->u_part, nd->e_off, nd->R, nd->shift, nd->g, nd->ebar};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete nd;
}

int wmpc_bind_nodes(wmpc_ctx* ctx, wmpc_nodes* nodes) {
  return run(ctx, [&]() -> int {
    ARG(nodes && nodes->n == (size_t)ctx->n, "node state does not match this context");
    if (!nodes->ready) {
      ctx->err = "node state has not been computed";
      return WMPC_E_STATE;
    }
    if (ctx->nodes != nodes) point_nodes(ctx, nodes);
    ctx->have_nodes = true;
    return WMPC_OK;
  });
}

int wmpc_set_node_data(wmpc_ctx* ctx, wmpc_nodes* nodes, const double* demand, const double* Ed,
                       const double* demand_gd, const double* econ, int64_t* bad_row) {
  return run(ctx, [&]() -> int {
    if (!ctx->have_structure) {
      ctx->err = "set_structure must precede set_node_data";
      return WMPC_E_STATE;
    }
    ARG(nodes && nodes->n == (size_t)ctx->n, "node state does not match this context");
    ARG(demand_gd && econ, "null node data");
    const size_t n = ctx->n;
    if (ctx->ns > 0) {
      ARG(demand && Ed, "demand and Ed required when n_mixing > 0");
      h2d(ctx, ctx->demand, demand, sizeof(double) * n * ctx->nd);
      h2d(ctx, ctx->Ed, Ed, sizeof(double) * ctx->ns * ctx->nd);
    }
    // demand_gd in one contiguous copy, padded to lx on the device (a pitched
    // host copy of 504-byte rows is several times slower)
    if (!ctx->gd_stage) dalloc(ctx, &ctx->gd_stage, n * ctx->nt);
    h2d(ctx, ctx->gd_stage, demand_gd, sizeof(double) * n * ctx->nt);
    ctx->launches++;
    k_pad_rows<<<grid_for(n * ctx->lx), 256, 0, ctx->stream>>>(ctx->gd_stage, ctx->nt, nodes->g, ctx->lx, (int)n,
                                                              ctx->bad_row);
    h2d(ctx, ctx->econ, econ, sizeof(double) * n * ctx->nu);
    point_nodes(ctx, nodes);
    DevView d = view(ctx);
    int blocks = (int)((n * 32 + 255) / 256);
    ctx->launches++;
    if (ctx->fast && ctx->ns > 0 && ctx->ns <= 32)  // projector structure verified (configure_fast)
      k_node_offsets_proj<<<(int)((n + 7) / 8), 256, 0, ctx->stream>>>(
          d, ctx->demand, ctx->Ed, ctx->pj_kp, ctx->pj_kc, ctx->pj_kv, ctx->pj_ecp, ctx->pj_ecr, ctx->pj_ecv,
          1.0 / (2.0 * ctx->w_c), nodes->shift, nodes->u_part, nodes->e_off, ctx->bad_row);
    else
      k_node_offsets<<<blocks, 256, 0, ctx->stream>>>(d, ctx->demand, ctx->Ed, nodes->shift, nodes->u_part,
                                                       nodes->e_off, ctx->tmp, ctx->bad_row);
    ctx->launches++;
    k_node_R<<<blocks, 256, 0, ctx->stream>>>(d, nodes->e_off, nodes->R);
    if (ctx->fast) {
      ctx->launches++;
      const int tot = ctx->nchain * ctx->nu;
      k_chain_ebar<<<(tot + 255) / 256, 256, 0, ctx->stream>>>(ctx->chain_node, ctx->nchain, ctx->H - ctx->kstar,
                                                               ctx->nu, nodes->e_off, nodes->ebar);
    }
    check_launch(ctx);
    int bad = INT_MAX;
    d2h(ctx, &bad, ctx->bad_row, sizeof(int));
    sync(ctx);
    if (bad != INT_MAX) {
      ctx->nodes = nullptr;
      ctx->have_nodes = false;
      if (bad_row) *bad_row = bad;
      ctx->err = "coupling E u = -Ed d is infeasible at tree node " + std::to_string(bad + 1);
      return WMPC_E_INFEASIBLE;
    }
    nodes->ready = true;
    ctx->have_nodes = true;
    return WMPC_OK;
  });
}

int wmpc_get_offsets(wmpc_ctx* ctx, wmpc_nodes* nodes, double* u_part, double* e_offset) {
  return run(ctx, [&]() -> int {
    ARG(nodes && nodes->n == (size_t)ctx->n, "node state does not match this context");
    const size_t bytes = sizeof(double) * (size_t)ctx->n * ctx->nu;
    if (u_part) d2h(ctx, u_part, nodes->u_part, bytes);
    if (e_offset) d2h(ctx, e_offset, nodes->e_off, bytes);
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_kernel_launches_per_iteration(const wmpc_ctx* ctx) {
  if (!ctx) return -1;
  if (ctx->fast && ctx->use_graphk) return graphk_kernels(ctx);
  return ctx->fast ? 0 : 2 * ctx->H + 1;  // fast: one persistent launch per chunk
}

int wmpc_path_info(const wmpc_ctx* ctx, int* out, int cap) {
  if (!ctx || !out) return WMPC_E_ARG;
  const bool g = ctx->fast && ctx->use_graphk;
  const int v[] = {wmpc_fast_path(ctx),
                   g && dp_on(ctx) ? 1 : 0,
                   g && ctx->chainw ? 1 : 0,
                   ctx->cw_pd,
                   (int)ctx->gk_groups.size(),
                   ctx->nchain,
                   ctx->kstar,
                   ctx->ell_vf,
                   ctx->fp32,
                   ctx->dp_wpc,
                   ctx->dp_grid,
                   ctx->dp_cpw,
                   wmpc_kernel_launches_per_iteration(ctx),
                   ctx->n_branch,
                   ctx->sms,
                   g && dp_on(ctx) ? ctx->dp_sib : 0,
                   g && dp_on(ctx) ? ctx->dp_segm : 0};
  const int nv = (int)(sizeof(v) / sizeof(v[0]));
  for (int i = 0; i < cap && i < nv; ++i) out[i] = v[i];
  return nv;
}

int wmpc_set_pdl(wmpc_ctx* ctx, int on) {
  if (!ctx) return WMPC_E_ARG;
  if (ctx->pdl != (on ? 1 : 0)) {
    ctx->pdl = on ? 1 : 0;
    ctx->gk_gamma = -1.0;  // recapture the iteration graphs
  }
  return WMPC_OK;
}

int wmpc_fast_path(const wmpc_ctx* ctx) {
  if (!ctx || !ctx->fast) return 0;
  if (ctx->use_graphk) return 300;
  if (ctx->use_scan) return 200 + ctx->fast_mc;
  return ctx->fast_mc;
}

int wmpc_set_bounds(wmpc_ctx* ctx, const double* x_min, const double* x_max, const double* x_safe,
                    const double* u_min, const double* u_max, double w_x, double w_s, const double* p,
                    const double* q, const double* econ) {
  return run(ctx, [&]() -> int {
    ARG(x_min && x_max && x_safe && u_min && u_max && p && q, "null bound argument");
    const size_t nt = ctx->nt, nu = ctx->nu;
    h2d(ctx, ctx->xmin, x_min, sizeof(double) * nt);
    h2d(ctx, ctx->xmax, x_max, sizeof(double) * nt);
    h2d(ctx, ctx->xsafe, x_safe, sizeof(double) * nt);
    h2d(ctx, ctx->umin, u_min, sizeof(double) * nu);
    h2d(ctx, ctx->umax, u_max, sizeof(double) * nu);
    h2d(ctx, ctx->p, p, sizeof(double) * nt);
    h2d(ctx, ctx->q, q, sizeof(double) * nu);
    if (econ) h2d(ctx, ctx->econ, econ, sizeof(double) * (size_t)ctx->n * nu);
    ctx->w_x = w_x;
    ctx->w_s = w_s;
    sync(ctx);
    ctx->have_bounds = true;
    return WMPC_OK;
  });
}

static int need_ready(wmpc_ctx* ctx) {
  if (!ctx->have_structure || !ctx->have_nodes || !ctx->have_bounds) {
    ctx->err = "structure, node data and bounds must be set first";
    return WMPC_E_STATE;
  }
  return WMPC_OK;
}

int wmpc_dual_gradient(wmpc_ctx* ctx, const double* y, double* z, double* value) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(y && z, "null argument");
    const size_t n = ctx->n;
    h2d(ctx, ctx->ys, y, sizeof(double) * n * ctx->W);
    DevView d = view(ctx);
    d.U = ctx->Uc;
    d.X = ctx->Xc;
    dual_gradient_dev(ctx, ctx->ys, ctx->Uc, ctx->Xc);
    ctx->launches++;
    k_join_primal<<<grid_for(n * ctx->P), 256, 0, ctx->stream>>>(ctx->n, ctx->nu, ctx->nt, ctx->lx, ctx->Uc, ctx->Xc,
                                                                   ctx->zbuf);
    check_launch(ctx);
    d2h(ctx, z, ctx->zbuf, sizeof(double) * n * ctx->P);
    if (value) {
      double t[4];
      cost_terms(ctx, d, ctx->Uc, ctx->Xc, ctx->ys, 0, t);
      *value = t[0] + t[1];
    }
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_prox(wmpc_ctx* ctx, const double* v, double gamma, int conjugate, double* out) {
  return run(ctx, [&]() -> int {
    if (!ctx->have_bounds) {
      ctx->err = "bounds must be set first";
      return WMPC_E_STATE;
    }
    ARG(v && out, "null argument");
    ARG(gamma > 0.0, "gamma must be positive");
    const size_t len = (size_t)ctx->n * ctx->W;
    h2d(ctx, ctx->ys, v, sizeof(double) * len);
    DevView d = view(ctx);
    int blocks = (int)(((size_t)ctx->n * 32 + 255) / 256);
    ctx->launches++;
    k_prox_rows<<<blocks, 256, 0, ctx->stream>>>(d, ctx->ys, ctx->zbuf, gamma, conjugate);
    check_launch(ctx);
    d2h(ctx, out, ctx->zbuf, sizeof(double) * len);
    sync(ctx);
    return WMPC_OK;
  });
}

// gv = Op(vsrc) = H(x*(0) - x*(v)); returns (v.gv, ||gv||^2).
static void apply_operator(wmpc_ctx* ctx, const double* vsrc, double out[2]) {
  DevView d = view(ctx);
  d.U = ctx->Uc;
  d.X = ctx->Xc;
  dual_gradient_dev(ctx, vsrc, ctx->Uc, ctx->Xc);
  size_t len = (size_t)ctx->n * ctx->W;
  int nb = std::min(ctx->part_blocks, grid_for(len));
  ctx->launches++;
  k_op_rows<<<nb, 256, 0, ctx->stream>>>(d, ctx->U0, ctx->X0, ctx->Uc, ctx->Xc, vsrc, ctx->gv, ctx->part);
  ctx->launches++;
  k_finish<0><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 2, 0, 2, ctx->scal);
  check_launch(ctx);
  d2h(ctx, out, ctx->scal, 2 * sizeof(double));
  sync(ctx);
}

static void zero_dual_solution(wmpc_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->ys, 0, sizeof(double) * (size_t)ctx->n * ctx->W, ctx->stream));
  dual_gradient_dev(ctx, ctx->ys, ctx->U0, ctx->X0);
}

int wmpc_power_iteration(wmpc_ctx* ctx, const double* v0, double rel_tol, int max_iter, double* lam,
                         int* settled, int* iters) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(v0 && lam && settled, "null argument");
    const size_t len = (size_t)ctx->n * ctx->W;
    zero_dual_solution(ctx);
    h2d(ctx, ctx->vv, v0, sizeof(double) * len);
    double l = 0.0, lprev = 0.0;
    int ok = 0, k = 0;
    for (k = 0; k < max_iter; ++k) {
      double r[2];
      apply_operator(ctx, ctx->vv, r);
      l = r[0];
      double nrm = std::sqrt(r[1]);
      if (nrm == 0.0) break;
      ctx->launches++;
      k_scale_into<<<grid_for(len), 256, 0, ctx->stream>>>(ctx->gv, len, ctx->scal + 1, ctx->vv);
      check_launch(ctx);
      if (std::fabs(l - lprev) <= rel_tol * std::max(std::fabs(l), 1e-300)) {
        ok = 1;
        break;
      }
      lprev = l;
    }
    sync(ctx);
    *lam = l;
    *settled = ok;
    if (iters) *iters = k;
    return WMPC_OK;
  });
}

int wmpc_operator_trace(wmpc_ctx* ctx, double* trace) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    const size_t len = (size_t)ctx->n * ctx->W;
    zero_dual_solution(ctx);
    double total = 0.0;
    const double one = 1.0, zero = 0.0;
    CK(cudaMemsetAsync(ctx->vv, 0, sizeof(double) * len, ctx->stream));
    for (size_t i = 0; i < len; ++i) {
      h2d(ctx, ctx->vv + i, &one, sizeof(double));
      double r[2];
      apply_operator(ctx, ctx->vv, r);
      double gi;
      d2h(ctx, &gi, ctx->gv + i, sizeof(double));
      h2d(ctx, ctx->vv + i, &zero, sizeof(double));
      sync(ctx);
      total += gi;
    }
    *trace = total;
    return WMPC_OK;
  });
}

int wmpc_apg_begin(wmpc_ctx* ctx, double gamma, int max_iter, const double* theta, const double* beta) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(gamma > 0.0 && max_iter >= 1 && theta && beta, "invalid APG parameters");
    if (max_iter > ctx->max_iter) {
      if (ctx->theta) cudaFree(ctx->theta);
      if (ctx->beta) cudaFree(ctx->beta);
      ctx->theta = ctx->beta = nullptr;
      ctx->graph_gamma = -1.0;  // table pointers change: recapture
      dalloc(ctx, &ctx->theta, max_iter);
      dalloc(ctx, &ctx->beta, max_iter);
      ctx->max_iter = max_iter;
    }
    h2d(ctx, ctx->theta, theta, sizeof(double) * max_iter);
    h2d(ctx, ctx->beta, beta, sizeof(double) * max_iter);
    const size_t len = (size_t)ctx->n * ctx->W;
    for (int k = 0; k < 3; ++k) CK(cudaMemsetAsync(ctx->Y[k], 0, sizeof(double) * len, ctx->stream));
    CK(cudaMemsetAsync(ctx->U, 0, sizeof(double) * (size_t)ctx->n * ctx->nu, ctx->stream));
    CK(cudaMemsetAsync(ctx->X, 0, sizeof(double) * (size_t)ctx->n * ctx->lx, ctx->stream));
    CK(cudaMemsetAsync(ctx->Yc, 0, sizeof(double) * (size_t)ctx->n * ctx->ly, ctx->stream));
    CK(cudaMemsetAsync(ctx->Ua, 0, sizeof(double) * (size_t)ctx->n * ctx->nu, ctx->stream));
    CK(cudaMemsetAsync(ctx->Xa, 0, sizeof(double) * (size_t)ctx->n * ctx->lx, ctx->stream));
    CK(cudaMemsetAsync(ctx->iter, 0, sizeof(int), ctx->stream));
    int big = INT_MAX;
    h2d(ctx, ctx->bad_nu, &big, sizeof(int));
    ctx->gamma = gamma;
    ctx->it_host = 0;
    sync(ctx);
    if (ctx->fast) {
      if (ctx->use_graphk && ctx->fp32) {  // node data in fp32, Yc32 = 0
        const size_t n = ctx->n;
        CK(cudaMemsetAsync(ctx->f32_Yc, 0, sizeof(float) * n * ctx->ly, ctx->stream));
        ctx->launches += 3;
        k_convert<<<grid_for(n * ctx->nu), 256, 0, ctx->stream>>>(ctx->nodes->e_off, ctx->f32_eoff, n * ctx->nu);
        k_convert<<<grid_for(n * ctx->nu), 256, 0, ctx->stream>>>(ctx->nodes->R, ctx->f32_R, n * ctx->nu);
        k_convert<<<grid_for(n * ctx->lx), 256, 0, ctx->stream>>>(ctx->nodes->g, ctx->f32_g, n * ctx->lx);
        check_launch(ctx);
      }
      if (ctx->use_graphk) {
        FastView f0 = make_fastview(ctx, 1);
        if (f0.rfree) {  // ut = u at Yc = 0 (Yc was just zeroed): one full up/branch/down pass
          f0.rfree = 0;
          f0.d.U = ctx->ut;
          f0.d.X = ctx->Xc;
          if (ctx->ell_w == 4) {
            gk_up<4>(ctx, f0);
            gk_grp<4>(ctx, f0, 0);
            gk_down<4>(ctx, f0);
          } else {
            gk_up<8>(ctx, f0);
            gk_grp<8>(ctx, f0, 0);
            gk_down<8>(ctx, f0);
          }
          ctx->launches += 2 + ctx->gk_groups.size();
          if (ctx->fp32) {
            ctx->launches++;
            k_convert<<<grid_for((size_t)ctx->n * ctx->nu), 256, 0, ctx->stream>>>(ctx->ut, ctx->ut32,
                                                                                    (size_t)ctx->n * ctx->nu);
          }
          check_launch(ctx);
        }
        if (dp_on(ctx)) {  // k_chain_dp state at Yc = 0: L = 0, chain totals 0, per-chain constants
          const size_t n = ctx->n, na = (size_t)(ctx->n_branch + ctx->nchain) * ctx->nu;
          CK(cudaMemsetAsync(ctx->Lb, 0, sizeof(double) * n * ctx->nu, ctx->stream));
          CK(cudaMemsetAsync(ctx->Asub, 0, sizeof(double) * na, ctx->stream));
          CK(cudaMemsetAsync(ctx->wbar, 0, sizeof(double) * n * ctx->lx, ctx->stream));
          FastView f1 = make_fastview(ctx, 1);
          const int nbk = ((ctx->nchain + ctx->n_branch) * 32 + 255) / 256;
          ctx->launches++;
          if (ctx->dp_segm > 0) {  // segmented chains: corrections 0, handshake flags reset
            CK(cudaMemsetAsync(ctx->dp_corr, 0, sizeof(double) * ctx->nchain * 2 * ctx->nu, ctx->stream));
            CK(cudaMemsetAsync(ctx->dp_flag, 0, sizeof(int) * ctx->nchain, ctx->stream));
          }
          k_dp_agg_init<<<nbk, 256, 0, ctx->stream>>>(f1, ctx->dp_agg, ctx->dp_putg, ctx->dp_aggu, ctx->dp_auxs,
                                                      ctx->dp_segm);
          check_launch(ctx);
        }
        capture_graphk(ctx);
      }
      return WMPC_OK;  // persistent kernel: no graph
    }
    if (ctx->gexec && ctx->graph_gamma == gamma) return WMPC_OK;  // captured iteration still valid
    if (ctx->gexec) {
      cudaGraphExecDestroy(ctx->gexec);
      ctx->gexec = nullptr;
    }
    if (ctx->graph) {
      cudaGraphDestroy(ctx->graph);
      ctx->graph = nullptr;
    }
    DevView d = view(ctx);
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    launch_dg(ctx, d, nullptr, 1);
    k_advance<<<1, 32, 0, ctx->stream>>>(ctx->iter);
    CK(cudaStreamEndCapture(ctx->stream, &ctx->graph));
    CK(cudaGraphInstantiate(&ctx->gexec, ctx->graph, 0));
    ctx->launches -= 2 * ctx->H;  // captured, not launched
    ctx->graph_gamma = gamma;
    return WMPC_OK;
  });
}

int wmpc_apg_run(wmpc_ctx* ctx, int count) {
  return run(ctx, [&]() -> int {
    if (ctx->shard_k > 0 && !ctx->nccl) {
      ctx->err = "a shard with replicated rows advances through wmpc_shard_step (or set up NCCL)";
      return WMPC_E_STATE;
    }
    if (ctx->fast && ctx->max_iter > 0) {
      ARG(count >= 0 && ctx->it_host + count <= ctx->max_iter, "iteration count exceeds the theta table");
      if (count > 0) launch_fast(ctx, count);
      check_launch(ctx);
      ctx->it_host += count;
      return WMPC_OK;
    }
    if (!ctx->gexec) {
      ctx->err = "wmpc_apg_begin must precede wmpc_apg_run";
      return WMPC_E_STATE;
    }
    ARG(count >= 0 && ctx->it_host + count <= ctx->max_iter, "iteration count exceeds the theta table");
    for (int i = 0; i < count; ++i) CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    ctx->it_host += count;
    ctx->launches += (int64_t)count * (2 * ctx->H + 1);
    return WMPC_OK;
  });
}

int wmpc_apg_run_timed(wmpc_ctx* ctx, int count, float* ms) {
  return run(ctx, [&]() -> int {
    if (ctx->shard_k > 0 && !ctx->nccl) {
      ctx->err = "a shard with replicated rows advances through wmpc_shard_step (or set up NCCL)";
      return WMPC_E_STATE;
    }
    if (ctx->fast && ctx->max_iter > 0) {
      ARG(count >= 0 && ctx->it_host + count <= ctx->max_iter, "iteration count exceeds the theta table");
      CK(cudaEventRecord(ctx->ev2, ctx->stream));
      if (count > 0) launch_fast(ctx, count);
      CK(cudaEventRecord(ctx->ev3, ctx->stream));
      CK(cudaEventSynchronize(ctx->ev3));
      CK(cudaEventElapsedTime(ms, ctx->ev2, ctx->ev3));
      ctx->it_host += count;
      return WMPC_OK;
    }
    if (!ctx->gexec) {
      ctx->err = "wmpc_apg_begin must precede wmpc_apg_run_timed";
      return WMPC_E_STATE;
    }
    ARG(count >= 0 && ctx->it_host + count <= ctx->max_iter, "iteration count exceeds the theta table");
    CK(cudaEventRecord(ctx->ev2, ctx->stream));
    for (int i = 0; i < count; ++i) CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    CK(cudaEventRecord(ctx->ev3, ctx->stream));
    CK(cudaEventSynchronize(ctx->ev3));
    CK(cudaEventElapsedTime(ms, ctx->ev2, ctx->ev3));
    ctx->it_host += count;
    ctx->launches += (int64_t)count * (2 * ctx->H + 1);
    return WMPC_OK;
  });
}

// Per-kernel device time of the iteration (bench.py roofline): `count` APG
// iterations launched eagerly (no graph, no programmatic overlap) with events
// between the kernel groups. out (ms per iteration): k_chain_dp path
// [branch groups, k_chain_dp]; graph path [up, branch groups, down, prox].
// Advances the APG state like wmpc_apg_run.
int wmpc_iteration_profile(wmpc_ctx* ctx, int count, double* out, int cap) {
  return run(ctx, [&]() -> int {
    if (!(ctx->fast && ctx->use_graphk && ctx->max_iter > 0 && ctx->shard_k < 0)) {
      ctx->err = "iteration profile needs the structured graph path after wmpc_apg_begin";
      return WMPC_E_STATE;
    }
    ARG(count >= 1 && ctx->it_host + count <= ctx->max_iter && out, "iteration count exceeds the theta table");
    const int pdl = ctx->pdl;
    ctx->pdl = 0;
    int never = -1;
    CK(cudaMemcpyAsync(ctx->store_it, &never, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    FastView f = make_fastview(ctx, 1);
    const bool dp = dp_on(ctx);
    const int nk = dp ? 2 : 4;
    std::vector<cudaEvent_t> ev(nk + 1);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    std::vector<double> acc(nk, 0.0);
    try {
      for (int i = 0; i < count; ++i) {
        if (ctx->gk_groups.empty()) k_advance<<<1, 32, 0, ctx->stream>>>(ctx->iter);
        CK(cudaEventRecord(ev[0], ctx->stream));
        if (dp) {
          gk_grp<4, double>(ctx, f, 1, GRP_LATE, ctx->dp_sib);
          CK(cudaEventRecord(ev[1], ctx->stream));
          launch_dp(ctx, f);
          CK(cudaEventRecord(ev[2], ctx->stream));
        } else {
          const int bump = ctx->gk_groups.empty() ? 0 : 1;
          if (ctx->ell_w == 4) {
            if (ctx->fp32) {
              gk_up<4, float>(ctx, f); CK(cudaEventRecord(ev[1], ctx->stream));
              gk_grp<4, float>(ctx, f, bump); CK(cudaEventRecord(ev[2], ctx->stream));
              gk_down<4, float>(ctx, f); CK(cudaEventRecord(ev[3], ctx->stream));
              gk_prox<float>(ctx, f);
            } else {
              gk_up<4, double>(ctx, f); CK(cudaEventRecord(ev[1], ctx->stream));
              gk_grp<4, double>(ctx, f, bump); CK(cudaEventRecord(ev[2], ctx->stream));
              gk_down<4, double>(ctx, f); CK(cudaEventRecord(ev[3], ctx->stream));
              gk_prox<double>(ctx, f);
            }
          } else {
            gk_up<8, double>(ctx, f); CK(cudaEventRecord(ev[1], ctx->stream));
            gk_grp<8, double>(ctx, f, bump); CK(cudaEventRecord(ev[2], ctx->stream));
            gk_down<8, double>(ctx, f); CK(cudaEventRecord(ev[3], ctx->stream));
            gk_prox<double>(ctx, f);
          }
          CK(cudaEventRecord(ev[4], ctx->stream));
        }
        CK(cudaEventSynchronize(ev[nk]));
        for (int k = 0; k < nk; ++k) {
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
          acc[k] += ms;
        }
        ctx->it_host++;
        ctx->launches += graphk_kernels(ctx);
      }
    } catch (Fail&) {
      ctx->pdl = pdl;
      for (auto& e : ev) cudaEventDestroy(e);
      throw;
    }
    ctx->pdl = pdl;
    for (auto& e : ev) cudaEventDestroy(e);
    for (int k = 0; k < nk && k < cap; ++k) out[k] = acc[k] / count;
    return WMPC_OK;
  });
}

int wmpc_apg_iterations(const wmpc_ctx* ctx) { return ctx ? ctx->it_host : -1; }

int wmpc_apg_check(wmpc_ctx* ctx, double* primal_residual, double* image_scale, double* dual_change,
                   int* first_nonfinite_nu) {
  return run(ctx, [&]() -> int {
    if (ctx->it_host < 1) {
      ctx->err = "no APG iteration has run";
      return WMPC_E_STATE;
    }
    DevView d = view(ctx);
    const int it = ctx->it_host;
    size_t len = (size_t)ctx->n * ctx->W;
    int nb = std::min(ctx->part_blocks, grid_for(len));
    ctx->launches++;
    k_check_partial<<<nb, 256, 0, ctx->stream>>>(d, ctx->Y[it % 3], ctx->Y[(it + 2) % 3], ctx->part);
    ctx->launches++;
    k_finish<1><<<1, 256, 0, ctx->stream>>>(ctx->part, nb, 3, 0, 3, ctx->scal);
    check_launch(ctx);
    double h[3];
    int bad = INT_MAX;
    d2h(ctx, h, ctx->scal, 3 * sizeof(double));
    d2h(ctx, &bad, ctx->bad_nu, sizeof(int));
    sync(ctx);
    if (primal_residual) *primal_residual = h[0];
    if (image_scale) *image_scale = h[1];
    if (dual_change) *dual_change = h[2];
    if (first_nonfinite_nu) *first_nonfinite_nu = bad == INT_MAX ? -1 : bad;
    return WMPC_OK;
  });
}

int wmpc_certificate(wmpc_ctx* ctx, double* gap, double* objective) {
  return run(ctx, [&]() -> int {
    if (ctx->shard_k > 0) {
      ctx->err = "a shard with replicated rows certifies through wmpc_cert_* and the exchange";
      return WMPC_E_STATE;
    }
    int st = need_ready(ctx);
    if (st) return st;
    DevView d = view(ctx);
    const size_t nU = (size_t)ctx->n * ctx->nu;
    // 1. feasibility restoration of the averaged inputs (problem.py:221-250)
    if (ctx->ns == 0) {
      ctx->launches++;
      k_clip_inputs<<<grid_for(nU), 256, 0, ctx->stream>>>(d, ctx->Ua, ctx->Uf);
    } else {
      int nb0 = grid_for(nU);
      ctx->launches++;
      k_absmax_partial<<<nb0, 256, 0, ctx->stream>>>(ctx->Ua, nU, ctx->part);
      ctx->launches++;
      k_dyk_tol<<<1, 256, 0, ctx->stream>>>(ctx->part, nb0, ctx->scal + 8);
      DykOps po = dyk_ops(ctx);
      CK(cudaMemsetAsync(ctx->dk_mv, 0, sizeof(unsigned long long) * 512, ctx->stream));
      const int nbw = (ctx->n + 7) / 8;
      ctx->launches += 3;
      unsigned* bad = reinterpret_cast<unsigned*>(ctx->dk_mv);
      if (po.eidx) {  // block-diagonal coupling: one thread per (node, coupling row)
        const long long nthr = (long long)((ctx->n + 31) / 32) * 32 * ctx->ns;
        const int gb = (int)((nthr + 255) / 256);
        k_dyk_block<3><<<gb, 256, 0, ctx->stream>>>(d, po, ctx->Ua, ctx->Uf, bad, ctx->dk_sweeps, 500, ctx->dk_fix,
                                                   (const double*)(ctx->scal + 8));
        k_dyk_count_bits<<<1, 512, 0, ctx->stream>>>(bad, 500, ctx->dk_sweeps);
        // pass 2 over the blocks not settled by the global count, compacted
        const long long nblk = (long long)ctx->n * ctx->ns;
        CK(cudaMemsetAsync(ctx->dk_list, 0, sizeof(int), ctx->stream));
        k_dyk_compact<<<(int)((nblk + 255) / 256), 256, 0, ctx->stream>>>(ctx->dk_fix, nblk, ctx->dk_sweeps,
                                                                         ctx->dk_list + 1, ctx->dk_list);
        k_dyk_redo<<<std::min((int)((nblk + 255) / 256), ctx->sms * 8), 256, 0, ctx->stream>>>(
            d, po, ctx->Ua, ctx->Uf, ctx->dk_sweeps, ctx->dk_list + 1, ctx->dk_list);
        ctx->launches += 2;
      } else {
        launch_dyk(ctx, nbw, po, d, po, ctx->Ua, ctx->Uf, ctx->dk_mv, ctx->dk_sweeps, 500, 3, ctx->dk_fix,
                   (const double*)(ctx->scal + 8));
        k_dyk_count_bits<<<1, 512, 0, ctx->stream>>>(bad, 500, ctx->dk_sweeps);
        launch_dyk(ctx, nbw, po, d, po, ctx->Ua, ctx->Uf, ctx->dk_mv, ctx->dk_sweeps, 500, 2, ctx->dk_fix,
                   (const double*)(ctx->scal + 8));
      }
    }
    // 2. rollout (problem.py:207-218)
    rollout(ctx, d, ctx->Uf, ctx->Xf);
    check_launch(ctx);
    // 3. primal value (solver.py:453): terms into scal[16..20)
    cost_terms_dev(ctx, d, ctx->Uf, ctx->Xf, nullptr, 1, ctx->scal + 16);
    // 4. dual value at the current iterate (solver.py:454-456)
    const double* y = ctx->Y[ctx->it_host % 3];
    DevView dc = d;
    dc.U = ctx->Uc;
    dc.X = ctx->Xc;
    if (ctx->fast && ctx->use_graphk) {
      if (ctx->ell_w == 4) dual_eval_graph<4>(ctx, y, -1);
      else dual_eval_graph<8>(ctx, y, -1);
    } else {
      launch_dg(ctx, dc, y, 0);
    }
    cost_terms_dev(ctx, dc, ctx->Uc, ctx->Xc, y, 0, ctx->scal + 20);
    gconj_dev(ctx, d, y, ctx->scal + 24);
    check_launch(ctx);
    double h[10];  // the certificate's only host round trip
    d2h(ctx, h, ctx->scal + 16, sizeof(h));
    sync(ctx);
    const double* tp = h;
    const double* td = h + 4;
    double primal = tp[0] + (ctx->w_x * tp[2] + ctx->w_s * tp[3]);
    double inner = td[0] + td[1];
    double gc = h[9] > 0.0 ? INFINITY : h[8];
    double dual = inner - gc;
    if (gap) *gap = primal - dual;
    if (objective) *objective = primal;
    return WMPC_OK;
  });
}

int wmpc_apg_read(wmpc_ctx* ctx, int averaged, double* u0, double* primal, double* primal_avg, double* dual) {
  return run(ctx, [&]() -> int {
    DevView d = view(ctx);
    const size_t n = ctx->n;
    if (ctx->fp32 && ctx->it_host > 0) {  // the last iterate lives in the fp32 arrays
      ctx->launches += 2;
      k_convert<<<grid_for(n * ctx->nu), 256, 0, ctx->stream>>>(ctx->f32_U, ctx->U, n * ctx->nu);
      k_convert<<<grid_for(n * ctx->lx), 256, 0, ctx->stream>>>(ctx->f32_X, ctx->X, n * ctx->lx);
    }
    if (u0) {
      ctx->launches++;
      k_u0<<<1, 128, 0, ctx->stream>>>(d, averaged ? ctx->Ua : ctx->U, ctx->off[1], ctx->zbuf);
      check_launch(ctx);
      d2h(ctx, u0, ctx->zbuf, sizeof(double) * ctx->nu);
      sync(ctx);
    }
    if (primal) {
      ctx->launches++;
      k_join_primal<<<grid_for(n * ctx->P), 256, 0, ctx->stream>>>(ctx->n, ctx->nu, ctx->nt, ctx->lx, ctx->U, ctx->X,
                                                                     ctx->zbuf);
      d2h(ctx, primal, ctx->zbuf, sizeof(double) * n * ctx->P);
      sync(ctx);
    }
    if (primal_avg) {
      ctx->launches++;
      k_join_primal<<<grid_for(n * ctx->P), 256, 0, ctx->stream>>>(ctx->n, ctx->nu, ctx->nt, ctx->lx, ctx->Ua, ctx->Xa,
                                                                     ctx->zbuf);
      d2h(ctx, primal_avg, ctx->zbuf, sizeof(double) * n * ctx->P);
      sync(ctx);
    }
    if (dual) d2h(ctx, dual, ctx->Y[ctx->it_host % 3], sizeof(double) * n * ctx->W);
    check_launch(ctx);
    sync(ctx);
    return WMPC_OK;
  });
}

// Result readout on a second stream: the join kernels and device-to-host
// copies run while the caller goes on (the certificate reads Ua and y and
// writes only its own scratch, so it can run concurrently). Copies into
// page-locked destinations are truly asynchronous; wmpc_apg_read_wait joins.
int wmpc_apg_read_async(wmpc_ctx* ctx, int averaged, double* u0, double* primal, double* primal_avg,
                        double* dual) {
  return run(ctx, [&]() -> int {
    DevView d = view(ctx);
    const size_t n = ctx->n, np_ = n * ctx->P;
    if (!ctx->stream_rd) {
      CK(cudaStreamCreateWithFlags(&ctx->stream_rd, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->ev_rd, cudaEventDisableTiming));
      dalloc(ctx, &ctx->rb_u0, (size_t)ctx->nu);
      dalloc(ctx, &ctx->rb_p, np_);
      dalloc(ctx, &ctx->rb_a, np_);
    }
    if (ctx->fp32 && ctx->it_host > 0) {  // the last iterate lives in the fp32 arrays
      ctx->launches += 2;
      k_convert<<<grid_for(n * ctx->nu), 256, 0, ctx->stream>>>(ctx->f32_U, ctx->U, n * ctx->nu);
      k_convert<<<grid_for(n * ctx->lx), 256, 0, ctx->stream>>>(ctx->f32_X, ctx->X, n * ctx->lx);
    }
    CK(cudaEventRecord(ctx->ev_rd, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->stream_rd, ctx->ev_rd, 0));
    cudaStream_t s = ctx->stream_rd;
    if (u0) {
      ctx->launches++;
      k_u0<<<1, 128, 0, s>>>(d, averaged ? ctx->Ua : ctx->U, ctx->off[1], ctx->rb_u0);
      CK(cudaMemcpyAsync(u0, ctx->rb_u0, sizeof(double) * ctx->nu, cudaMemcpyDeviceToHost, s));
    }
    if (primal) {
      ctx->launches++;
      k_join_primal<<<grid_for(np_), 256, 0, s>>>(ctx->n, ctx->nu, ctx->nt, ctx->lx, ctx->U, ctx->X, ctx->rb_p);
      CK(cudaMemcpyAsync(primal, ctx->rb_p, sizeof(double) * np_, cudaMemcpyDeviceToHost, s));
    }
    if (primal_avg) {
      ctx->launches++;
      k_join_primal<<<grid_for(np_), 256, 0, s>>>(ctx->n, ctx->nu, ctx->nt, ctx->lx, ctx->Ua, ctx->Xa, ctx->rb_a);
      CK(cudaMemcpyAsync(primal_avg, ctx->rb_a, sizeof(double) * np_, cudaMemcpyDeviceToHost, s));
    }
    if (dual)
      CK(cudaMemcpyAsync(dual, ctx->Y[ctx->it_host % 3], sizeof(double) * n * ctx->W, cudaMemcpyDeviceToHost, s));
    check_launch(ctx);
    return WMPC_OK;
  });
}

int wmpc_apg_read_wait(wmpc_ctx* ctx) {
  return run(ctx, [&]() -> int {
    if (ctx->stream_rd) CK(cudaStreamSynchronize(ctx->stream_rd));
    return WMPC_OK;
  });
}

int wmpc_timer_start(wmpc_ctx* ctx) {
  return run(ctx, [&]() -> int {
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    return WMPC_OK;
  });
}

int wmpc_timer_stop(wmpc_ctx* ctx, float* ms) {
  return run(ctx, [&]() -> int {
    CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaEventSynchronize(ctx->ev1));
    CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
    return WMPC_OK;
  });
}

int64_t wmpc_launch_count(const wmpc_ctx* ctx) { return ctx ? ctx->launches : -1; }

int wmpc_host_alloc(uint64_t bytes, void** out) {
  if (!out) return WMPC_E_ARG;
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    g_global_err = std::string("cudaHostAlloc: ") + cudaGetErrorString(e);
    return WMPC_E_CUDA;
  }
  return WMPC_OK;
}

void wmpc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int wmpc_debug_div(const double* v, const double* g64, int n, uint64_t* mismatches) {
  double *dv = nullptr, *dg = nullptr;
  unsigned long long* dbad = nullptr;
  if (cudaMalloc(&dv, sizeof(double) * n) || cudaMalloc(&dg, sizeof(double) * 64) ||
      cudaMalloc(&dbad, sizeof(unsigned long long))) {
    g_global_err = "cudaMalloc failed";
    return WMPC_E_CUDA;
  }
  cudaMemcpy(dv, v, sizeof(double) * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dg, g64, sizeof(double) * 64, cudaMemcpyHostToDevice);
  cudaMemset(dbad, 0, sizeof(unsigned long long));
  k_debug_div<<<1184, 256>>>(dv, dg, n, dbad);
  unsigned long long bad = 0;
  cudaError_t e = cudaMemcpy(&bad, dbad, sizeof(bad), cudaMemcpyDeviceToHost);
  cudaFree(dv);
  cudaFree(dg);
  cudaFree(dbad);
  if (e != cudaSuccess) {
    g_global_err = cudaGetErrorString(e);
    return WMPC_E_CUDA;
  }
  *mismatches = bad;
  return WMPC_OK;
}

float wmpc_last_debug_ms(const wmpc_ctx* ctx) { return ctx ? ctx->last_debug_ms : -1.f; }

int wmpc_profile_fast(wmpc_ctx* ctx, int count, uint64_t* counters, int cap) {
  return run(ctx, [&]() -> int {
    if (!ctx->fast || !ctx->max_iter) {
      ctx->err = "fast path not configured or no APG begun";
      return WMPC_E_STATE;
    }
    ARG(count >= 1 && ctx->it_host + count <= ctx->max_iter, "bad count");
    const size_t slots = (size_t)std::max(ctx->fast_grid, ctx->nchain) * P_N;
    if (!ctx->prof) dalloc(ctx, &ctx->prof, slots);
    CK(cudaMemsetAsync(ctx->prof, 0, sizeof(uint64_t) * slots, ctx->stream));
    ctx->prof_on = 1;
    if (ctx->use_graphk) {  // direct launches with the clock counters on
      ctx->store_it_host = ctx->it_host + count - 1;
      CK(cudaMemcpyAsync(ctx->store_it, &ctx->store_it_host, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
      FastView f = make_fastview(ctx, 1);
      for (int i = 0; i < count; ++i) enqueue_graphk_iteration(ctx, f);
    } else {
      launch_fast(ctx, count);
    }
    ctx->prof_on = 0;
    ctx->it_host += count;
    check_launch(ctx);
    size_t nvals = std::min((size_t)cap, slots);
    d2h(ctx, counters, ctx->prof, sizeof(uint64_t) * nvals);
    sync(ctx);
    return WMPC_OK;
  });
}

// ---------------------------------------------------------------- sharding
int wmpc_shard_setup(wmpc_ctx* ctx, int k_stage, int n_rep_global, const int64_t* rep_gidx, const int64_t* acct) {
  return run(ctx, [&]() -> int {
    if (!ctx->have_structure || !ctx->fast || !ctx->use_graphk) {
      ctx->err = "subtree sharding needs the structured graph path (A = I, W = cI) and a set structure";
      return WMPC_E_STATE;
    }
    ARG(k_stage >= 0 && k_stage <= ctx->kstar, "shard stage must lie in the branching region");
    ARG(rep_gidx && acct && n_rep_global >= 0, "null shard argument");
    ARG(k_stage == 0 || n_rep_global >= 1, "replicated rows need an exchange buffer");
    const int n = ctx->n;
    std::vector<int> ac(n), rg(n);
    for (int r = 0; r < n; ++r) {
      ac[r] = acct[r] ? 1 : 0;
      rg[r] = (int)rep_gidx[r];
      ARG(rg[r] < n_rep_global, "replicated index out of range");
      ARG((r < ctx->off[k_stage]) == (rg[r] >= 0), "rows above the shard stage (and only those) are replicated");
    }
    upload_vec(ctx, &ctx->acct, ac);
    upload_vec(ctx, &ctx->rep_gidx, rg);
    ctx->n_rep_global = n_rep_global;
    ctx->shard_k = k_stage;
    build_groups(ctx, k_stage, ac.data());
    ctx->gk_gamma = -1.0;  // groups changed: recapture the iteration graphs
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_set_min_branch_stage(wmpc_ctx* ctx, int stage) {
  return run(ctx, [&]() -> int {
    ARG(stage >= 0 && stage < ctx->H, "stage out of range");
    ctx->kstar_min = stage;
    return WMPC_OK;
  });
}

int wmpc_set_precision(wmpc_ctx* ctx, int fp32) {
  return run(ctx, [&]() -> int {
    if (!fp32) {
      if (ctx->fp32) ctx->gk_gamma = -1.0;
      ctx->fp32 = 0;
      return WMPC_OK;
    }
    if (!ctx->fast || !ctx->use_graphk || ctx->shard_k >= 0) {
      ctx->err = "fp32 mode needs the structured graph path (A = I, W = cI), unsharded";
      return WMPC_E_STATE;
    }
    const size_t n = ctx->n, nu = ctx->nu, lx = ctx->lx, ly = ctx->ly;
    const size_t na = (size_t)(ctx->n_branch + ctx->nchain) * nu;
    if (!ctx->f32_Yc) {
      dalloc(ctx, &ctx->f32_Yc, n * ly); dalloc(ctx, &ctx->f32_Lb, n * nu); dalloc(ctx, &ctx->f32_Asub, na);
      dalloc(ctx, &ctx->f32_wbar, n * lx); dalloc(ctx, &ctx->f32_U, n * nu); dalloc(ctx, &ctx->f32_X, n * lx);
      dalloc(ctx, &ctx->f32_eoff, n * nu); dalloc(ctx, &ctx->f32_R, n * nu); dalloc(ctx, &ctx->f32_g, n * lx);
      dalloc(ctx, &ctx->f32_aux, n * 2); dalloc(ctx, &ctx->f32_ell, ctx->ell_len);
      dalloc(ctx, &ctx->ut32, n * nu);
    }
    ctx->launches += 2;
    k_convert<<<grid_for(n * 2), 256, 0, ctx->stream>>>(ctx->aux, ctx->f32_aux, n * 2);
    k_convert<<<grid_for(ctx->ell_len), 256, 0, ctx->stream>>>(ctx->ell_val, ctx->f32_ell, ctx->ell_len);
    check_launch(ctx);
    sync(ctx);
    if (!ctx->fp32) ctx->gk_gamma = -1.0;  // recapture the iteration graphs
    ctx->fp32 = 1;
    return WMPC_OK;
  });
}

int wmpc_apg_warm(wmpc_ctx* ctx, const double* y0) {
  return run(ctx, [&]() -> int {
    ARG(y0, "null argument");
    if (ctx->max_iter <= 0 || ctx->it_host != 0) {
      ctx->err = "wmpc_apg_warm must directly follow wmpc_apg_begin";
      return WMPC_E_STATE;
    }
    const size_t len = (size_t)ctx->n * ctx->W;
    h2d(ctx, ctx->Y[0], y0, sizeof(double) * len);
    CK(cudaMemcpyAsync(ctx->Y[2], ctx->Y[0], sizeof(double) * len, cudaMemcpyDeviceToDevice, ctx->stream));
    DevView d = view(ctx);
    ctx->launches++;
    k_collapse<<<grid_for((size_t)ctx->n * ctx->ly), 256, 0, ctx->stream>>>(d, ctx->Y[0], ctx->Yc);
    if (ctx->fp32) {
      ctx->launches++;
      k_convert<<<grid_for((size_t)ctx->n * ctx->ly), 256, 0, ctx->stream>>>(ctx->Yc, ctx->f32_Yc,
                                                                             (size_t)ctx->n * ctx->ly);
    }
    if (ctx->fast && ctx->use_graphk && dp_on(ctx)) {  // L, aggregates and chain totals of iteration 0
      FastView f = make_fastview(ctx, 1);  // the up pass of Yc(0) (R-free), then the L aggregates
      const int nbk = (ctx->nchain * 32 + 255) / 256;
      gk_up<4, double>(ctx, f);
      if (ctx->dp_sib) gk_grp<4, double>(ctx, f, 0, 0, 0, 1);  // the stage k_chain_dp finishes itself
      k_dp_agg_L<<<nbk, 256, 0, ctx->stream>>>(f, ctx->dp_agg, ctx->dp_aggu, ctx->dp_segm);
      ctx->launches += 2 + ctx->dp_sib;
    }
    check_launch(ctx);
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_nccl_unique_id(void* out) {
  ncclUniqueId id;
  NcclApi& api = nccl_api();
  if (!out || !api.ok) {
    g_global_err = "libnccl.so.2 not available";
    return WMPC_E_CUDA;
  }
  if (api.get_unique_id(&id) != ncclSuccess) return WMPC_E_CUDA;
  std::memcpy(out, &id, sizeof(id));
  return WMPC_OK;
}

int wmpc_shard_nccl_init(wmpc_ctx* ctx, const void* id, int nranks, int rank) {
  return run(ctx, [&]() -> int {
    ARG(id && nranks >= 1 && rank >= 0 && rank < nranks, "bad NCCL arguments");
    CK(cudaSetDevice(ctx->dev));
    NcclApi& api = nccl_api();
    if (!api.ok) {
      ctx->err = "libnccl.so.2 not available";
      return WMPC_E_CUDA;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    if (ctx->nccl) api.destroy(ctx->nccl);
    ctx->nccl = nullptr;
    const ncclResult_t r = api.init_rank(&ctx->nccl, nranks, uid, rank);
    if (r != ncclSuccess) {
      ctx->nccl = nullptr;
      ctx->err = std::string("ncclCommInitRank failed: ") + api.error_string(r);
      return WMPC_E_CUDA;
    }
    ctx->gk_gamma = -1.0;  // iteration graphs now carry the exchange
    return WMPC_OK;
  });
}

int wmpc_shard_exchange(wmpc_ctx* ctx) {
  return run(ctx, [&]() -> int {
    if (!ctx->nccl || !ctx->xbuf) {
      ctx->err = "NCCL communicator and exchange buffer must be set";
      return WMPC_E_STATE;
    }
    if (ctx->n_rep_global > 0) exchange_dev(ctx);
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_sync(wmpc_ctx* ctx) {
  return run(ctx, [&]() -> int {
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_shard_set_exchange(wmpc_ctx* ctx, void* device_buffer) {
  return run(ctx, [&]() -> int {
    ctx->xbuf = static_cast<double*>(device_buffer);
    return WMPC_OK;
  });
}

int wmpc_shard_step(wmpc_ctx* ctx, int phase) {
  return run(ctx, [&]() -> int {
    if (ctx->shard_k < 0 || ctx->max_iter <= 0) {
      ctx->err = "wmpc_shard_setup and wmpc_apg_begin must precede wmpc_shard_step";
      return WMPC_E_STATE;
    }
    ARG(phase == 0 || phase == 1, "phase must be 0 or 1");
    ARG(ctx->it_host < ctx->max_iter, "iteration count exceeds the theta table");
    ARG(ctx->rep_group.second == 0 || ctx->xbuf, "exchange buffer not set");
    FastView f = make_fastview(ctx, 1);
    if (ctx->ell_w == 4) shard_phase<4>(ctx, f, phase);
    else shard_phase<8>(ctx, f, phase);
    if (phase == 1) ctx->it_host += 1;
    return WMPC_OK;
  });
}

int wmpc_shard_fix_R(wmpc_ctx* ctx, int phase) {
  return run(ctx, [&]() -> int {
    if (ctx->shard_k < 0 || !ctx->nodes || !ctx->xbuf) {
      ctx->err = "wmpc_shard_setup, node data and the exchange buffer must precede wmpc_shard_fix_R";
      return WMPC_E_STATE;
    }
    ARG(phase == 0 || phase == 1, "phase must be 0 or 1");
    if (ctx->n_rep_global == 0) return WMPC_OK;
    if (phase == 0) CK(cudaMemsetAsync(ctx->xbuf, 0, sizeof(double) * 256 * (size_t)ctx->n_rep_global, ctx->stream));
    DevView d = view(ctx);
    ctx->launches++;
    k_shard_R<<<(int)(((size_t)ctx->n * 32 + 255) / 256), 256, 0, ctx->stream>>>(d, ctx->nodes->e_off, ctx->rep_gidx,
                                                                              ctx->xbuf, phase, ctx->nodes->R);
    check_launch(ctx);
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_cert_absmax(wmpc_ctx* ctx, double* absmax) {
  return run(ctx, [&]() -> int {
    ARG(absmax, "null argument");
    const size_t nU = (size_t)ctx->n * ctx->nu;
    const int nb0 = grid_for(nU);
    ctx->launches += 2;
    k_absmax_partial<<<nb0, 256, 0, ctx->stream>>>(ctx->Ua, nU, ctx->part);
    k_finish<1><<<1, 256, 0, ctx->stream>>>(ctx->part, nb0, 1, 0, 1, ctx->scal);
    check_launch(ctx);
    d2h(ctx, absmax, ctx->scal, sizeof(double));
    sync(ctx);
    return WMPC_OK;
  });
}

int wmpc_cert_dykstra(wmpc_ctx* ctx, int max_sweeps, double* mv) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(mv && max_sweeps >= 1 && max_sweeps <= 512, "bad Dykstra arguments");
    std::vector<unsigned long long> bits(max_sweeps, 0ull);
    if (ctx->ns > 0) {
      DevView d = view(ctx);
      DykOps po = dyk_ops(ctx);
      CK(cudaMemsetAsync(ctx->dk_mv, 0, sizeof(unsigned long long) * 512, ctx->stream));
      ctx->launches++;
      launch_dyk(ctx, (ctx->n + 7) / 8, po, d, po, ctx->Ua, nullptr, ctx->dk_mv, ctx->dk_sweeps,
                 max_sweeps, 1, nullptr, (const double*)nullptr);
      check_launch(ctx);
      d2h(ctx, bits.data(), ctx->dk_mv, sizeof(unsigned long long) * max_sweeps);
      sync(ctx);
    }
    for (int i = 0; i < max_sweeps; ++i) std::memcpy(mv + i, &bits[i], sizeof(double));
    return WMPC_OK;
  });
}

int wmpc_shard_dual_eval(wmpc_ctx* ctx, int phase) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(phase == 0 || phase == 1, "phase must be 0 or 1");
    if (!ctx->fast || !ctx->use_graphk) {
      ctx->err = "sharded certificate needs the structured graph path";
      return WMPC_E_STATE;
    }
    const double* y = ctx->Y[ctx->it_host % 3];
    if (ctx->ell_w == 4) dual_eval_graph<4>(ctx, y, phase);
    else dual_eval_graph<8>(ctx, y, phase);
    return WMPC_OK;
  });
}

int wmpc_cert_terms(wmpc_ctx* ctx, int sweeps, double* terms) {
  return run(ctx, [&]() -> int {
    int st = need_ready(ctx);
    if (st) return st;
    ARG(terms && sweeps >= 1 && sweeps <= 512, "bad certificate arguments");
    DevView d = view(ctx);
    const size_t nU = (size_t)ctx->n * ctx->nu;
    if (ctx->ns == 0) {
      ctx->launches++;
      k_clip_inputs<<<grid_for(nU), 256, 0, ctx->stream>>>(d, ctx->Ua, ctx->Uf);
    } else {
      h2d(ctx, ctx->dk_sweeps, &sweeps, sizeof(int));
      DykOps po = dyk_ops(ctx);
      ctx->launches++;
      launch_dyk(ctx, (ctx->n + 7) / 8, po, d, po, ctx->Ua, ctx->Uf, ctx->dk_mv, ctx->dk_sweeps, sweeps,
                 2, nullptr, (const double*)nullptr);
    }
    rollout(ctx, d, ctx->Uf, ctx->Xf);
    check_launch(ctx);
    double tp[4], td[4], g[2];
    cost_terms(ctx, d, ctx->Uf, ctx->Xf, nullptr, 1, tp);
    const double* y = ctx->Y[ctx->it_host % 3];
    DevView dc = d;
    dc.U = ctx->Uc;
    dc.X = ctx->Xc;
    cost_terms(ctx, dc, ctx->Uc, ctx->Xc, y, 0, td);
    gconj_raw(ctx, d, y, g);
    for (int i = 0; i < 4; ++i) {
      terms[i] = tp[i];
      terms[4 + i] = td[i];
    }
    terms[8] = g[0];
    terms[9] = g[1];
    return WMPC_OK;
  });
}

void wmpc_u0_rows(int nu, int mu1, const double* prob, const double* rows, const double* u_min, const double* u_max,
                  double* u0) {
  for (int j = 0; j < nu; ++j) {
    double s = 0.0;
    for (int r = 0; r < mu1; ++r) s = std::fma(prob[r], rows[(size_t)r * nu + j], s);
    const double lo = u_min[j], hi = u_max[j];
    const double m = std::isnan(s) ? s : (s > lo ? s : lo);  // np.clip (k_u0)
    u0[j] = std::isnan(m) ? m : (m < hi ? m : hi);
  }
}

}  // extern "C"
