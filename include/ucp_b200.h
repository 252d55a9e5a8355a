/* ucp_b200 -- C ABI of the B200 (sm_100a) marginal-cost evaluator for the
 * arXiv 1908.04489 UCP solver (`ucpsolve`), Witsenhausen counterexample.
 *
 * This is the drop-in boundary: the reference's hot path is the Python
 * plugin API `Problem.marginal_cost_segmented` / the solver phases / the
 * `kernels` module (numba); each entry point below replaces one of them and
 * cites it (paths relative to /root/reference/pkg/src/ucpsolve).  The host
 * side that binds them (ctypes) is paper_1908_04489_b200/_lib.py; the
 * binding a maintainer would add to the reference is in INTEGRATION.md.
 *
 * Conventions
 *  - every array argument is a DEVICE pointer (float64 / int64, C
 *    contiguous) owned by the caller (PyTorch tensors in the Python host);
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); every call
 *    is asynchronous on it unless documented otherwise;
 *  - results are bitwise the reference's ("ref-order" arithmetic: glibc-exact
 *    exp/erf, no FMA contraction, the reference's summation order);
 *  - return value: UCP_OK or an error status (ucp_status_string());
 *    non-finite numerics are NOT return codes: sweeps atomicMin the first
 *    offending grid point into a caller-owned device `err` array so the host
 *    can raise the reference's NumericError lazily.
 */
#ifndef UCP_B200_H
#define UCP_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UCP_ABI_VERSION 3

enum ucp_status {
  UCP_OK = 0,
  UCP_ERR_ARG = 1,     /* bad argument (shape, stage index, null pointer) -> ValueError */
  UCP_ERR_CUDA = 3,    /* CUDA runtime error */
};

/* Sentinel stored in `err` slots that saw no failure. */
#define UCP_NO_ERROR INT64_MAX

/* Witsenhausen problem (problems/witsenhausen.py:36-57).  Grid spacing
 * h = (b-a)/(d-1) (grids.py:55-56); y0/y1 are the np.linspace points
 * (grids.py:50), f0 = numerics.pdf(N(0, sigma), y0) and fw0 = trapezoid
 * weights * f0 (witsenhausen.py:47-53), all computed by the host with NumPy
 * and uploaded (NumPy's SIMD exp is not glibc's). */
typedef struct ucp_wc_problem {
  double k;
  double a0, h0;
  int64_t d0;
  double a1, h1;
  int64_t d1;
  const double* y0;  /* [d0] */
  const double* y1;  /* [d1] */
  const double* f0;  /* [d0] */
  const double* fw0; /* [d0] */
  int64_t flags;     /* UCP_WC_FAST or 0 (the reference's arithmetic, bitwise) */
} ucp_wc_problem;

/* ucp_wc_problem.flags: stage-0 walks in the tolerance-stated fast mode --
 * h folded into the pdf recurrence and FMA in the v-weighted sums (6 FP64
 * instructions per node instead of 8).  NOT bitwise the reference: moments
 * agree to rounding (~1e-15 relative), costs within 1e-10 relative (the
 * quadratic in s cancels), argmin picks may differ on near-ties only, J of a
 * snapshot within 1e-13 relative; a full solve may branch at a near-tie (the
 * d=2000 solve converges 4.9e-7 relative below the reference's J) -- stated
 * and tested in tests/test_gpu_fast_mode.py. */
#define UCP_WC_FAST 1
/* ucp_wc_problem.flags (opt-in, tolerance-stated; with UCP_WC_FAST): window
 * sums from expansions instead of per-candidate walks/sums, on grids with
 * h1 <= 2e-3.  Stage 0 (both phases; the objective through
 * ucp_wc_objective_terms_ws): per-cell Taylor expansions, 12 terms, cells of
 * width 0.016 over [a1 - 12, b1 + 12] built once per call, the reference
 * walk's first-order rounding bias reproduced, exact cdf tails added -- O(1)
 * per candidate instead of O(24/h1).  Stage 1 (both phases): Taylor
 * expansions of the moments per tile of floor(0.016/h1) queries, grid ends
 * completed with the cdf tails.  J of a snapshot within 1e-9 of the
 * reference arithmetic's; exhaustion picks differ on near-ties only;
 * local-update decisions at near-zero curvature may differ; converged J
 * within 1e-9 (tests/test_gpu_fast_mode.py). */
#define UCP_WC_TABLE 2

/* Local-update parameters (solver.py:47-97, SolverConfig), already resolved
 * per stage (newton_cap = cfg.cap_for(grid)). */
typedef struct ucp_local_params {
  double fd_step;
  double curvature_min;
  double grad_step;
  double newton_cap;
} ucp_local_params;

typedef struct ucp_workspace ucp_workspace;

/* ---- library / workspace ------------------------------------------------ */
int ucp_abi_version(void);
const char* ucp_status_string(int status);
const char* ucp_last_error(void);
/* Number of kernel launches issued by this library so far (instrumentation). */
int64_t ucp_launch_count(void);
/* Scratch memory for the sweeps; grows on first use, reused afterwards. */
int ucp_workspace_create(ucp_workspace** ws);
int ucp_workspace_destroy(ucp_workspace* ws);
/* Hand a workspace to a new owner (the Python side pools them across
 * problems): synchronises the device (the next owner may use another stream),
 * drops the content-keyed Inventory caches and marks the captured block graphs
 * stale -- never replayed as they are, only reused through
 * cudaGraphExecUpdate by a capture of the same shape. */
int ucp_workspace_recycle(ucp_workspace* ws);
/* Pre-size scratch for grids of d0/d1 points and up to max_cand exhaustion
 * candidates so later calls never allocate. */
int ucp_workspace_reserve(ucp_workspace* ws, int64_t d0, int64_t d1, int64_t max_cand);

/* ---- kernels.py surface ---------------------------------------------------
 * kernels.gauss_moments_grid (kernels.py:406-445): T_k(s_t) for t < n. */
int ucp_gauss_moments_grid(const double* s, int64_t n, const double* v, double a, double h,
                           int64_t d, double* t0, double* t1, double* t2, void* stream);
/* kernels.gauss_moments_points (kernels.py:447-486). */
int ucp_gauss_moments_points(const double* y, int64_t n, const double* x, const double* w,
                             int64_t m, double a, double h, int64_t d, double* o0, double* o1,
                             double* o2, ucp_workspace* ws, void* stream);
/* kernels.trapezoid_sum (kernels.py:136-144): serial ascending sum, written
 * to *out (device).  If err != NULL, err[0] receives the first index with a
 * non-finite sample (problem.py:117-127 diagnostics). */
int ucp_trapezoid_sum(const double* samples, int64_t n, double spacing, double* out,
                      int64_t* err, void* stream);
/* kernels.segmented_argmin (kernels.py:147-160). */
int ucp_segmented_argmin(const double* costs, const int64_t* offsets, int64_t nseg,
                         int64_t* out, void* stream);
/* kernels.flatten_windows, numba variant (kernels.py:163-187, dedup of later
 * duplicates within each window, window order kept).  Point i's window is
 * values[lo[i]..hi[i]] (0 <= lo[i] <= hi[i] < d).  offsets: n+1 entries (its
 * last one is the kept total); flat: capacity sum(hi-lo+1) doubles, or NULL
 * to compute only the offsets.  Asynchronous: read offsets[n] to size the
 * result. */
int ucp_flatten_windows(const double* values, int64_t d, const int64_t* lo, const int64_t* hi, int64_t n,
                        double* flat, int64_t* offsets, ucp_workspace* ws, void* stream);
/* Device libm port, exposed for parity tests: out[i] = exp(x[i]) (which=0),
 * erf(x[i]) (which=1) or the reference's phi_cdf(x[i]) (which=2). */
int ucp_device_libm(int which, const double* x, int64_t n, double* out, void* stream);

/* ---- Witsenhausen plugin: Problem.marginal_cost_segmented -----------------
 * witsenhausen.py:62-70 (m=0).  Candidate u_flat[c] for c in
 * [offsets[s], offsets[s+1]) is scored at observation y_seg[s] with stage-0
 * density f0_seg[s]; v1 = U.values(1); n_cand = offsets[nseg] (host copy). */
int ucp_wc_stage0_cost(const ucp_wc_problem* P, const double* v1, const double* u_flat,
                       int64_t n_cand, const int64_t* offsets, const double* y_seg,
                       const double* f0_seg, int64_t nseg, double* out, void* stream);
/* The same with a workspace: the walks stop at their provably no-op tail
 * (same bits), and under UCP_WC_TABLE the costs come from the expansion
 * cells, as in the problem's phases. */
int ucp_wc_stage0_cost_ws(const ucp_wc_problem* P, const double* v1, const double* u_flat,
                          int64_t n_cand, const int64_t* offsets, const double* y_seg,
                          const double* f0_seg, int64_t nseg, double* out, ucp_workspace* ws,
                          void* stream);
/* witsenhausen.py:71-78 (m=1); u0 = U.values(0). */
int ucp_wc_stage1_cost(const ucp_wc_problem* P, const double* u0, const double* u_flat,
                       int64_t n_cand, const int64_t* offsets, const double* y_seg, int64_t nseg,
                       double* out, ucp_workspace* ws, void* stream);

/* ---- solver phases (sharded over grid points [begin, end)) ----------------
 * solver.py:179-203 local_update_phase for stage `stage`; out[i] written for
 * i in [begin, end).  err[0] <- first point with non-finite c1/c2,
 * err[1] <- first point with non-finite cost_old/cost_new,
 * err[2] <- first point whose new value is non-finite (grids.py:80-84). */
int ucp_wc_local_update(const ucp_wc_problem* P, int stage, const double* u0, const double* u1,
                        const ucp_local_params* lp, int64_t begin, int64_t end, double* out,
                        int64_t* err, ucp_workspace* ws, void* stream);
/* solver.py:206-223 partial_exhaustion_phase; win_lo/win_hi from
 * grids.node_window_bounds (grids.py:180-195).  err[0] <- first point with a
 * non-finite candidate cost.  cand_bound = sum of window widths over the
 * shard (host-known): when given (> 0) and within budget the call never
 * synchronises; with 0 it reads the candidate count back (one stream sync). */
int ucp_wc_exhaustion(const ucp_wc_problem* P, int stage, const double* u0, const double* u1,
                      const int64_t* win_lo, const int64_t* win_hi, int64_t cand_bound,
                      int64_t begin, int64_t end, double* out, int64_t* err, ucp_workspace* ws,
                      void* stream);
/* solver.py:226-231 _run_block, unsharded: `iters` iterations over both
 * stages of one phase kind (0 = local update with lp[0..1], 1 = partial
 * exhaustion with the two stages' windows), each phase reading the latest
 * controllers.  u0/u1 are updated IN PLACE (scratch0/1: d0/d1 doubles);
 * err holds 3 slots per phase, phase p = 2*iteration + stage.  One host call
 * per block: no per-phase host round trip beyond the exhaustion count. */
int ucp_wc_run_block(const ucp_wc_problem* P, int kind, int iters, double* u0, double* u1,
                     const ucp_local_params* lp, const int64_t* win_lo0, const int64_t* win_hi0,
                     const int64_t* win_lo1, const int64_t* win_hi1, int64_t cand_bound0,
                     double* scratch0, double* scratch1, int64_t* err, ucp_workspace* ws,
                     void* stream);
/* Same block as ucp_wc_run_block, with the iterations after the first
 * replayed from a CUDA graph (captured once per block signature on a private
 * stream, launched on `stream`).  err6 = 3 slots per stage, the minimum over
 * all iterations (the host re-runs the block eagerly to name the first
 * failing phase).  Exhaustion blocks need cand_bound0 > 0 to be graphed. */
int ucp_wc_run_block_graph(const ucp_wc_problem* P, int kind, int iters, double* u0, double* u1,
                           const ucp_local_params* lp, const int64_t* win_lo0,
                           const int64_t* win_hi0, const int64_t* win_lo1,
                           const int64_t* win_hi1, int64_t cand_bound0, double* scratch0,
                           double* scratch1, int64_t* err6, ucp_workspace* ws, void* stream);
/* problem.py:110-127 objective, per-point part: terms[i] = C0(u0[i], y0[i])
 * for i in [begin, end); err[0] <- first non-finite term.  The serial
 * trapezoid over all terms is ucp_trapezoid_sum. */
int ucp_wc_objective_terms(const ucp_wc_problem* P, const double* u0, const double* u1,
                           int64_t begin, int64_t end, double* terms, int64_t* err,
                           void* stream);
/* The same with a workspace: the walks stop at their provably no-op tail
 * (range-max table built in ws; bitwise the same terms, ~17% fewer nodes at
 * 2^20), and under UCP_WC_TABLE the integrand's window sums come from the
 * expansion cells instead of the FMA walk -- J within ~1e-10 relative of the
 * walk's (tests/test_gpu_fast_mode.py). */
int ucp_wc_objective_terms_ws(const ucp_wc_problem* P, const double* u0, const double* u1,
                              int64_t begin, int64_t end, double* terms, int64_t* err,
                              ucp_workspace* ws, void* stream);

/* ---- config 5: uniform-noise kernels and the other UCP examples -----------
 * kernels.py:488-615 (numba bodies); rad = noise half-width. */
int ucp_unif_moments_grid(const double* x, int64_t n, const double* v, double a, double h, int64_t d,
                          double rad, double* s0, double* s1, double* s2, void* stream);
int ucp_unif_ball_sum(const double* x, int64_t n, const double* g, double a, double h, int64_t d,
                      double rad, double* out, void* stream);
/* out has d entries */
int ucp_unif_propagate(const double* masses, const double* centers, int64_t n, double a, double h,
                       int64_t d, double rad, double* out, void* stream);
int ucp_unif_moments_points(const double* y, int64_t n, const double* centers, const double* w,
                            const double* vals, int64_t m, double a, double h, int64_t d, double rad,
                            double* m0, double* m1, double* m2, void* stream);

/* Zero-delay source-channel coding (problems/zero_delay.py:36-86): encoder
 * grid 0, decoder grid 1, f0 = pdf(N(0,1), y0) and fw0 from host NumPy. */
typedef struct ucp_zd_problem {
  double power_weight;
  double a0, h0;
  int64_t d0;
  double a1, h1;
  int64_t d1;
  const double* y0;
  const double* y1;
  const double* f0;
  const double* fw0;
} ucp_zd_problem;
/* marginal_cost_segmented (zero_delay.py:66-86): y_seg/f0_seg per segment */
int ucp_zd_cost(const ucp_zd_problem* P, int stage, const double* u0, const double* u1,
                const double* u_flat, int64_t n_cand, const int64_t* offsets, const double* y_seg,
                const double* f0_seg, int64_t nseg, double* out, ucp_workspace* ws, void* stream);
/* local update with the widened probe h = max(h, h1) (zero_delay.py:56-65) */
int ucp_zd_local_update(const ucp_zd_problem* P, int stage, const double* u0, const double* u1,
                        const ucp_local_params* lp, int64_t begin, int64_t end, double* out,
                        int64_t* err, ucp_workspace* ws, void* stream);
/* wmax = max window width (hi - lo + 1) over the sweep */
int ucp_zd_exhaustion(const ucp_zd_problem* P, int stage, const double* u0, const double* u1,
                      const int64_t* win_lo, const int64_t* win_hi, int64_t wmax, int64_t begin,
                      int64_t end,
                      double* out, int64_t* err, ucp_workspace* ws, void* stream);
int ucp_zd_objective_terms(const ucp_zd_problem* P, const double* u0, const double* u1,
                           int64_t begin, int64_t end, double* terms, int64_t* err, void* stream);

/* Multi-stage inventory control (problems/inventory.py:31-150), M <= 16
 * stages, grid m = (a[m], h[m], d[m]) with device points pts[m]; controllers
 * are passed as a host array of M device pointers.  Projection u >= 0. */
#define UCP_INV_MAX_STAGES 16
typedef struct ucp_inv_problem {
  int32_t stages;
  int32_t quadratic; /* stage_cost: 0 piecewise_linear, 1 quadratic */
  double order_cost, holding_rate, backlog_rate;
  double a[UCP_INV_MAX_STAGES];
  double h[UCP_INV_MAX_STAGES];
  int64_t d[UCP_INV_MAX_STAGES];
  const double* pts[UCP_INV_MAX_STAGES];
  /* Optional (NULL: none): host array of M caller-assigned content keys, one
   * per controller u[m], nonzero and never reused for different contents.
   * With keys, the stock densities f_k (keyed by u[0..k-1]) and costs-to-go
   * g_k (keyed by u[k..M-1]) of earlier calls on the same workspace and
   * problem are reused instead of re-propagated: the same kernels on the same
   * inputs, so results are unchanged.  Zero-initialise this field. */
  const uint64_t* ukey;
} ucp_inv_problem;
int ucp_inv_cost(const ucp_inv_problem* P, int stage, const double* const* u, const double* u_flat,
                 int64_t n_cand, const int64_t* offsets, const double* y_seg, int64_t nseg,
                 double* out, ucp_workspace* ws, void* stream);
int ucp_inv_local_update(const ucp_inv_problem* P, int stage, const double* const* u,
                         const ucp_local_params* lp, int64_t begin, int64_t end, double* out,
                         int64_t* err, ucp_workspace* ws, void* stream);
int ucp_inv_exhaustion(const ucp_inv_problem* P, int stage, const double* const* u,
                       const int64_t* win_lo, const int64_t* win_hi, int64_t wmax, int64_t begin,
                       int64_t end,
                       double* out, int64_t* err, ucp_workspace* ws, void* stream);
int ucp_inv_objective_terms(const ucp_inv_problem* P, const double* const* u, int64_t begin,
                            int64_t end, double* terms, int64_t* err, ucp_workspace* ws,
                            void* stream);
/* stock density at stage m (inventory.py:96-110), out[d[m]] */
int ucp_inv_forward_density(const ucp_inv_problem* P, int stage, const double* const* u, double* out,
                            ucp_workspace* ws, void* stream);

/* ---- Monte-Carlo objective ------------------------------
 * Replaces oracle.monte_carlo_objective (oracle.py:98-105) over the problems'
 * simulate_cost (witsenhausen.py:81-89, zero_delay.py:88-94,
 * inventory.py:152-166).  Draw streams, in the order simulate_cost consumes
 * the generator: witsenhausen (x0 ~ N(0, sigma), w ~ N(0, 1)); zero_delay
 * (x0 ~ N(0, 1), w ~ U(-1, 1)); inventory (x ~ U(-1, 1), then w_m ~ U(-1, 1)
 * for m < stages). */
#define UCP_MC_WITSENHAUSEN 0
#define UCP_MC_ZERO_DELAY 1
#define UCP_MC_INVENTORY 2
#define UCP_MC_CHUNK 4096 /* samples per partial sum (fixes the reduction order) */
typedef struct ucp_mc_problem {
  int32_t kind;   /* UCP_MC_* */
  int32_t stages; /* inventory stage count (2 otherwise) */
  double k, sigma;      /* witsenhausen */
  double power_weight;  /* zero_delay */
  int32_t quadratic;    /* inventory stage_cost: 0 piecewise_linear, 1 quadratic */
  int32_t reserved;
  double order_cost, holding_rate, backlog_rate;
  double a[UCP_INV_MAX_STAGES]; /* stage grids: a, spacing, d */
  double h[UCP_INV_MAX_STAGES];
  int64_t d[UCP_INV_MAX_STAGES];
  const double* pts[UCP_INV_MAX_STAGES]; /* device grid points (inventory state snapping) */
  const double* u[UCP_INV_MAX_STAGES];   /* device controller values */
} ucp_mc_problem;
/* number of draw streams S per sample (or -1 on a bad problem) */
int ucp_mc_streams(const ucp_mc_problem* P);
/* per-sample costs from caller-supplied draws laid out [S][n] (e.g. drawn on
 * the host by the reference's NumPy generator): bitwise simulate_cost */
int ucp_mc_costs(const ucp_mc_problem* P, const double* draws, int64_t n, double* costs, void* stream);
/* the device generator's draws for samples [begin, end), laid out [S][end-begin]
 * (Philox4x32-10, key = seed: counter (i, c) gives uniforms U[i][2c], U[i][2c+1];
 * normals by Box-Muller on (U[i][0], U[i][1]), cosine then sine) */
int ucp_mc_philox_draws(const ucp_mc_problem* P, uint64_t seed, int64_t begin, int64_t end, double* draws,
                        void* stream);
/* fixed-order partial sums over chunks [chunk_begin, chunk_end) of n samples:
 * total == NULL -> sum of costs; else sum of (cost - *total / n)^2.
 * partials[c - chunk_begin] per chunk. */
int ucp_mc_partials(const ucp_mc_problem* P, uint64_t seed, int64_t n, int64_t chunk_begin, int64_t chunk_end,
                    const double* total, double* partials, void* stream);
/* fixed-order sum of n partials into *out (device) */
int ucp_mc_reduce(const double* partials, int64_t n, double* out, void* stream);

/* ---- batched multi-instance engine (config 4) -----------
 * B Witsenhausen instances on the SAME grids (k, sigma free) advanced
 * together: each call runs every kernel once over (instance, point).  Rows:
 * u0[B][ld0], u1[B][ld1] (updated in place), f0/fw0[B][ld0] (host NumPy
 * densities, witsenhausen.py:47-53), k[B].  Each instance's results are
 * bitwise its single-instance solve's.  Replaces one solver.solve() per
 * instance (solver.py:234-290) for k/sigma sweeps and multi-start. */
typedef struct ucp_wc_batch_desc {
  int64_t instances; /* B, 1..1024 */
  double a0, h0;
  int64_t d0;
  double a1, h1;
  int64_t d1;
  const double* y0; /* shared grid points */
  const double* y1;
  double* u0; /* [B][ld0] */
  double* u1; /* [B][ld1], 16-byte aligned rows */
  int64_t ld0, ld1; /* even row strides */
  const double* f0;  /* [B][ld0] */
  const double* fw0; /* [B][ld0] */
  const double* k;   /* [B] */
  ucp_local_params lp0, lp1; /* per stage (shared) */
  const int64_t* win_lo0; /* shared exhaustion windows (grids.py:180-195) */
  const int64_t* win_hi0;
  const int64_t* win_lo1;
  const int64_t* win_hi1;
  int64_t cand_bound0; /* sum of stage-0 window widths */
} ucp_wc_batch_desc;
typedef struct ucp_wc_batch ucp_wc_batch;
int ucp_wc_batch_create(const ucp_wc_batch_desc* desc, ucp_wc_batch** out);
int ucp_wc_batch_destroy(ucp_wc_batch* b);
/* `iters` block iterations (kind 0 local update, 1 partial exhaustion; both
 * stages each, solver.py:226-231) for instances ids[0..nslots) (host array).
 * lane: scratch set (exhaustion needs lane 1); two lanes may run concurrently
 * on two streams for disjoint instance sets.  err[b*6 + 3*m + e]: first bad
 * point (atomicMin; initialise to UCP_NO_ERROR) of stage m, as err6 of
 * ucp_wc_run_block_graph. */
int ucp_wc_batch_iterate(ucp_wc_batch* b, int lane, int kind, const int32_t* ids, int32_t nslots, int iters,
                         int64_t* err, void* stream);
/* J[b] = objective of each listed instance (problem.py:110-127); err_obj[b]
 * first non-finite integrand point. */
int ucp_wc_batch_objective(ucp_wc_batch* b, int lane, const int32_t* ids, int32_t nslots, double* J,
                           int64_t* err_obj, void* stream);

/* ---- NCCL plumbing for non-Python hosts ----------------------
 * One communicator per rank (one process per GPU, the current device).  Rank
 * 0 creates the id and the host ships it to the other ranks out of band.
 * A phase's controller shard is exchanged with ucp_allgather_f64 (in place
 * when send == recv + rank * count), error slots with ucp_allreduce_min_i64.
 * The Python host does the same through torch.distributed (distributed.py). */
#define UCP_COMM_ID_BYTES 128
typedef struct ucp_comm ucp_comm;
int ucp_comm_unique_id(unsigned char* id /* [UCP_COMM_ID_BYTES] */);
int ucp_comm_init(int nranks, int rank, const unsigned char* id, ucp_comm** comm);
int ucp_comm_destroy(ucp_comm* comm);
int ucp_allgather_f64(ucp_comm* comm, const double* send, double* recv, int64_t count, void* stream);
/* Uneven in-place all-gather of a phase's output in the natural layout: rank r
 * owns buf[bounds[r] .. bounds[r+1]) (bounds: nranks+1 ascending entries, the
 * work-balanced plan) and every rank ends with the whole vector.  Grouped
 * ncclBroadcast, one per non-empty shard. */
int ucp_allgatherv_f64(ucp_comm* comm, double* buf, const int64_t* bounds, void* stream);
int ucp_allreduce_min_i64(ucp_comm* comm, int64_t* buf, int64_t count, void* stream);

/* ---- instrumentation ------------------------------------------------------
 * FP64 pipe throughput probe (no FMA: DMUL/DADD only, 8 independent chains
 * per thread).  Performs iters*16 DP ops per thread; sink must hold
 * blocks*threads doubles. */
int ucp_fp64_probe(int blocks, int threads, int iters, double* sink, void* stream);

/* Throughput-mode stage-0 walks launched while `counter` (a device pointer,
 * nullptr = off) is set add the number of walk nodes they actually visited to
 * it (the no-op tail exit makes this fewer than the reference's window).  For
 * the roofline's executed-work count only; not thread-safe across host threads. */
int ucp_walk_node_counter(unsigned long long* counter);

#ifdef __cplusplus
}
#endif
#endif /* UCP_B200_H */
