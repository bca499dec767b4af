/*
 * wmpc.h — C ABI of the B200 scenario-tree dual-APG solver (libwmpc.so).
 *
 * The reference (watermpc, /root/reference/pkg/src/watermpc) has no FFI: its
 * boundary is the Python API of watermpc.solver / watermpc.problem. Each entry
 * point below replaces one piece of that API; the Python facade
 * (paper_1904_10548_b200/solver.py) binds them with ctypes.
 *
 * Conventions: host pointers are C-contiguous float64 (or int64 for indices),
 * node-major in breadth-first row order (row r = tree node r+1). Every call
 * returns 0 on success, a negative WMPC_E_* code otherwise; the message is in
 * wmpc_last_error(). A context is bound to one CUDA device and one tree
 * structure and is not thread-safe (one solve per context at a time).
 */
#ifndef WMPC_H
#define WMPC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WMPC_OK 0
#define WMPC_E_ARG -1        /* bad argument / shape            -> ValueError   */
#define WMPC_E_CUDA -2       /* CUDA runtime failure            -> RuntimeError */
#define WMPC_E_INFEASIBLE -3 /* coupling infeasible at a node   -> ValueError   */
#define WMPC_E_NONFINITE -4  /* non-finite iterate              -> RuntimeError */
#define WMPC_E_STATE -5      /* call order violated             -> RuntimeError */

typedef struct wmpc_ctx wmpc_ctx;

typedef struct wmpc_dims {
  int64_t n_nodes;   /* non-root nodes n                           */
  int32_t horizon;   /* H (stages 1..H)                            */
  int32_t n_tanks;   /* n_t                                        */
  int32_t n_inputs;  /* n_u                                        */
  int32_t n_demands; /* n_d                                        */
  int32_t n_mixing;  /* n_s (rows of E; may be 0)                  */
  int32_t device;    /* CUDA ordinal                               */
} wmpc_dims;

/* Create a context; allocates every device buffer for n_nodes.
 * Replaces the allocation part of solver.py:427-436. */
int wmpc_create(const wmpc_dims* dims, wmpc_ctx** out);
void wmpc_destroy(wmpc_ctx* ctx);
const char* wmpc_last_error(const wmpc_ctx* ctx);
/* Errors raised before a context exists. */
const char* wmpc_global_error(void);

/* Tree + stage factors (FactorCache structural members, solver.py:150-205).
 * A (nt*nt), B (nt*nu), Wu (nu*nu), T/D/Lam (H*nu*nu, stage-major),
 * anc_row (n; -1 = stage 1), stage_off (H+1), prob (n), E (ns*nu),
 * e_pinv (nu*ns). */
int wmpc_set_structure(wmpc_ctx* ctx, const double* A, const double* B, const double* Wu,
                       const double* T, const double* D, const double* Lam,
                       const int64_t* anc_row, const int64_t* stage_off, const double* prob,
                       const double* E, const double* e_pinv);

/* Per-node factor state (u_part, e_offset, child-aggregated offsets, coupling
 * shift, demand_gd) lives in its own device object so FactorCaches sharing one
 * tree structure (solver.py:163-170 reuse) share one context without copies. */
typedef struct wmpc_nodes wmpc_nodes;
int wmpc_nodes_create(wmpc_ctx* ctx, wmpc_nodes** out);
void wmpc_nodes_destroy(wmpc_nodes* nodes);
/* Make `nodes` the node state used by subsequent calls on ctx. */
int wmpc_bind_nodes(wmpc_ctx* ctx, wmpc_nodes* nodes);

/* Factor step per-node part on the GPU (solver.py:206-225) into `nodes`
 * (and bind it): demand (n*nd), Ed (ns*nd), demand_gd (n*nt), econ (n*nu).
 * Returns WMPC_E_INFEASIBLE with *bad_row = first infeasible row (node-1). */
int wmpc_set_node_data(wmpc_ctx* ctx, wmpc_nodes* nodes, const double* demand, const double* Ed,
                       const double* demand_gd, const double* econ, int64_t* bad_row);
/* Read back u_part / e_offset of `nodes` (n*nu each; FactorCache fields). */
int wmpc_get_offsets(wmpc_ctx* ctx, wmpc_nodes* nodes, double* u_part, double* e_offset);

/* Mutable per-solve data (tests mutate these after factor_step): state box,
 * safety level, input box, penalty weights, measured state p, previous input q,
 * economic rows econ (n*nu, nullable = keep). */
int wmpc_set_bounds(wmpc_ctx* ctx, const double* x_min, const double* x_max,
                    const double* x_safe, const double* u_min, const double* u_max,
                    double w_x, double w_s, const double* p, const double* q,
                    const double* econ);

/* Dual gradient (solver.py:242-306): y (n*(2nt+nu)) -> z (n*(nu+nt)) and the
 * attained value f(z) + <H'y, z>. value may be NULL. */
int wmpc_dual_gradient(wmpc_ctx* ctx, const double* y, double* z, double* value);

/* Row-wise prox (problem.py:313-327): conjugate=0 -> prox_{gamma g}(v);
 * conjugate=1 -> prox_{gamma g*}(v) via Moreau, the solver's expression order
 * (solver.py:563-575). Bit-exact with numpy on identical inputs. */
int wmpc_prox(wmpc_ctx* ctx, const double* v, double gamma, int conjugate, double* out);

/* Power iteration for the dual Lipschitz constant (solver.py:326-387).
 * v0 (n_dual) is the normalised start vector; returns the raw Rayleigh
 * quotient in *lam (no safety factor) and whether it settled. */
int wmpc_power_iteration(wmpc_ctx* ctx, const double* v0, double rel_tol, int max_iter,
                         double* lam, int* settled, int* iters);
/* Trace-bound fallback: sum_i <e_i, Op e_i> (solver.py:376-382). */
int wmpc_operator_trace(wmpc_ctx* ctx, double* trace);

/* APG loop (solver.py:398-543). begin: step gamma, theta/beta tables of
 * length max_iter (theta_nu and beta_nu = theta_nu (1/theta_{nu-1} - 1)),
 * y0 = 0. run: iterations [it, it + count) on the device, CUDA-graph replayed.
 * check: scalars of the last completed iteration. */
int wmpc_apg_begin(wmpc_ctx* ctx, double gamma, int max_iter, const double* theta,
                   const double* beta);
int wmpc_apg_run(wmpc_ctx* ctx, int count);
/* fp32 mode: the dual-gradient kernels (chain/branch passes,
 * Yc, L, U, X, node data) run in fp32; y, the prox, the ergodic averages, the
 * checks and the certificate stay fp64. Needs the structured graph path;
 * before wmpc_apg_begin. Own tolerance (tests: 1e-4 relative). */
int wmpc_set_precision(wmpc_ctx* ctx, int fp32);
/* Warm start (closed loop; the reference always starts at y = 0,
 * solver.py:430-431): right after wmpc_apg_begin, y0 = y_prev = the given dual. */
int wmpc_apg_warm(wmpc_ctx* ctx, const double* y0);
int wmpc_apg_check(wmpc_ctx* ctx, double* primal_residual, double* image_scale,
                   double* dual_change, int* first_nonfinite_nu);
/* Duality-gap certificate at the current dual iterate (solver.py:449-457):
 * Dykstra restoration of the averaged inputs, rollout, primal value, dual value. */
int wmpc_certificate(wmpc_ctx* ctx, double* gap, double* objective);
/* Results: u0 (nu), primal/primal_avg (n*(nu+nt)), dual (n*(2nt+nu)); any may
 * be NULL. averaged selects the ergodic average for u0. */
int wmpc_apg_read(wmpc_ctx* ctx, int averaged, double* u0, double* primal,
                  double* primal_avg, double* dual);
/* wmpc_apg_read on a second stream: returns once the join kernels and copies
 * are queued (they start when the work queued so far on the solver stream,
 * i.e. the APG loop, is done) so the caller can run the certificate
 * meanwhile; destinations must stay valid until wmpc_apg_read_wait. With
 * page-locked destinations (wmpc_host_alloc) the copies are asynchronous.
 * Replaces the tail of solver.py:520-543 (result assembly) with an overlapped readout. */
int wmpc_apg_read_async(wmpc_ctx* ctx, int averaged, double* u0, double* primal, double* primal_avg,
                        double* dual);
int wmpc_apg_read_wait(wmpc_ctx* ctx);
/* Per-kernel device time of the APG iteration (bench.py roofline): runs
 * `count` iterations eagerly with CUDA events between the kernel groups
 * (no graph, no programmatic overlap); out[] in ms per iteration:
 * [branch groups, k_chain_dp] on the fused path, [up, branch groups, down,
 * prox] on the graph path (path_info field 1 says which). Diagnostics; no
 * reference counterpart. */
int wmpc_iteration_profile(wmpc_ctx* ctx, int count, double* out, int cap);
/* Iterations completed since wmpc_apg_begin. */
int wmpc_apg_iterations(const wmpc_ctx* ctx);

/* Kernels launched per APG iteration (bench accounting; 0 = one persistent
 * launch per wmpc_apg_run call). */
int wmpc_kernel_launches_per_iteration(const wmpc_ctx* ctx);
/* Structured persistent kernel in use (A = I, W = cI): 200 + tile size for the
 * scan-form kernel (default), 100 + row slots for the warp-per-chain kernel,
 * the row-tile size for the step-recursive CTA kernel, 0 when the general
 * per-stage kernels run. */
int wmpc_fast_path(const wmpc_ctx* ctx);
/* Kernel selection of the bound structure, for tests and bench provenance:
 * out[0] wmpc_fast_path, [1] fused one-kernel iteration (k_chain_dp) in use,
 * [2] warp-per-chain up/down kernels, [3] their ring depth, [4] branch stage
 * groups, [5] chains, [6] first chain stage, [7] B/E values as float, [8] fp32
 * mode, [9] k_chain_dp warps per CTA, [10] its grid, [11] chains per warp,
 * [12] kernels per iteration, [13] branching rows, [14] SMs, [15] k_chain_dp
 * runs the lowest branching stage's up pass itself, [16] k_chain_dp's
 * upper-segment rows per chain (0: one warp per whole chain). Returns the
 * number of fields (writes at most cap). No reference counterpart. */
int wmpc_path_info(const wmpc_ctx* ctx, int* out, int cap);
/* Programmatic dependent launch between the iteration kernels on (default) or
 * off (plain stream order). Test hook: results must be bit-identical either
 * way (tests/test_gpu_hazards.py). No reference counterpart. */
int wmpc_set_pdl(wmpc_ctx* ctx, int on);

/* Timing helpers for bench.py: run `count` iterations between CUDA events on
 * the context's stream; *ms = elapsed device time. */
int wmpc_apg_run_timed(wmpc_ctx* ctx, int count, float* ms);

/* Test hook: number of v[i] / g64[i % 64] (n samples) where the kernels'
 * reciprocal-based exact division differs from IEEE division. */
int wmpc_debug_div(const double* v, const double* g64, int n, uint64_t* mismatches);

/* Diagnostics: run `count` APG iterations of the persistent kernel with
 * per-CTA clock64 counters (grid*12 values: total, phases A-D, projector,
 * prox, row wait, grid sync, chain steps) copied to `counters`. */
int wmpc_profile_fast(wmpc_ctx* ctx, int count, uint64_t* counters, int cap);

/* Device time (ms) of the last debug/test-hook launch. */
float wmpc_last_debug_ms(const wmpc_ctx* ctx);

/* Device-time bracket on the context's stream (bench.py): start records an
 * event; stop records a second one, waits for it and returns the elapsed ms. */
int wmpc_timer_start(wmpc_ctx* ctx);
int wmpc_timer_stop(wmpc_ctx* ctx, float* ms);
/* Kernels this context has launched so far (graph replays counted per node). */
int64_t wmpc_launch_count(const wmpc_ctx* ctx);

/* Page-locked host buffers for end-to-end transfers (bench.py e2e leg). */
int wmpc_host_alloc(uint64_t bytes, void** out);
void wmpc_host_free(void* p);

/* ---- Subtree sharding across GPUs (host side in shard.py).
 * The context holds one rank's rows: its own stage-k subtrees plus their
 * ancestors (stages < k), which are replicated on every rank sharing them.
 * Per APG iteration the replicated rows need the item sums of all ranks'
 * subtrees: phase 0 writes this rank's partial sums into the exchange buffer
 * (n_rep_global x 256 doubles, caller-owned device memory, zero except this
 * rank's rows), the caller all-reduces (sum) it across ranks, phase 1
 * finishes the replicated rows identically on every rank and runs the down
 * pass and the prox. With k = 0 there is nothing to exchange.
 * rep_gidx[r]: global index of local row r among the replicated rows, or -1;
 * acct[r]: 1 if this rank accounts for row r in global sums (its own rows and
 * the replicated rows whose lowest holder it is). Replaces the single-process
 * loop of solve() (solver.py:460-506) for one rank. */
int wmpc_shard_setup(wmpc_ctx* ctx, int k_stage, int n_rep_global, const int64_t* rep_gidx,
                     const int64_t* acct);
/* Before wmpc_set_structure of a shard: rows at stages < stage are treated as
 * branching rows even where this rank holds a single child (the replicated
 * rows must go through the exchange, not the chain scans). */
int wmpc_set_min_branch_stage(wmpc_ctx* ctx, int stage);
int wmpc_shard_set_exchange(wmpc_ctx* ctx, void* device_buffer);
int wmpc_shard_step(wmpc_ctx* ctx, int phase);
/* R of a replicated row (sum over its children, solver.py:269-274) spans
 * ranks: phase 0 writes this rank's accounted children, the caller sums the
 * exchange buffer across ranks, phase 1 stores the totals. Once per factor. */
int wmpc_shard_fix_R(wmpc_ctx* ctx, int phase);
/* Device-side exchange over NCCL (one communicator per context, ranks =
 * shards): with it, wmpc_apg_run replays CUDA graphs that contain the
 * all-reduce between the two phases of every iteration, and
 * wmpc_shard_exchange performs one (fix_R, certificate) on the stream.
 * wmpc_nccl_unique_id fills 128 bytes (ncclUniqueId) on rank 0. */
int wmpc_nccl_unique_id(void* out128);
int wmpc_shard_nccl_init(wmpc_ctx* ctx, const void* id128, int nranks, int rank);
int wmpc_shard_exchange(wmpc_ctx* ctx);
/* Wait for the context's stream (before the caller touches the exchange buffer). */
int wmpc_sync(wmpc_ctx* ctx);
/* Certificate pieces for a sharded solve (solver.py:449-457, problem.py:221-250):
 * local max|Ua| (the Dykstra tolerance is global), local per-sweep Dykstra
 * movement maxima (mv[max_sweeps]; the global stop sweep is the first whose
 * all-rank max is <= tol), the dual minimiser in two phases around the same
 * exchange as wmpc_shard_step, and the raw accounted sums
 * terms = [primal cost, <y,Hz> (0), box^2, safe^2 | dual cost, <y,Hz>, -, - |
 *          g* support sum, g* domain violation]. */
int wmpc_cert_absmax(wmpc_ctx* ctx, double* absmax);
int wmpc_cert_dykstra(wmpc_ctx* ctx, int max_sweeps, double* mv);
int wmpc_shard_dual_eval(wmpc_ctx* ctx, int phase);
int wmpc_cert_terms(wmpc_ctx* ctx, int sweeps, double* terms);
/* u0 from the stage-1 rows gathered in global order (k_u0 on the host:
 * clip(sum_r fma(p_r, u_r)), bit-identical to the device kernel). */
void wmpc_u0_rows(int nu, int mu1, const double* prob, const double* rows, const double* u_min,
                  const double* u_max, double* u0);

#ifdef __cplusplus
}
#endif
#endif /* WMPC_H */
