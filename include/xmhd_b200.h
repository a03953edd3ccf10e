/*
 * xmhd_b200.h — C-ABI of the B200 (sm_100a) Leja / FD-JVP / MHD-RHS hot path.
 *
 * Drop-in boundary for the reference's operator interface (arxiv/paper_2108_13622,
 * Python package xmhd).  The reference binds its hot path through Python
 * duck-typing; each entry point below replaces one reference callable and is
 * bound from the Python host mirror (paper_2108_13622_b200/_lib.py) with ctypes.
 *
 * Conventions
 *   - All vector pointers are DEVICE pointers to fp64 data in the reference's
 *     flat field-major layout (8, ny, nx): index f*ny*nx + j*nx + i
 *     (mhd.py:51-70).  Buffers are owned by the caller (PyTorch allocations);
 *     the context owns only scratch (reductions, Leja ping-pong, control block).
 *   - All work is enqueued on the context's CUDA stream (xmhd_set_stream).
 *   - Return value: XMHD_OK, XMHD_NONFINITE (a non-finite RHS cell: the caller
 *     raises RhsBlowupError, mhd.py:225-231), XMHD_BADARG, XMHD_CUDA_ERROR.
 *     xmhd_last_error() describes the last failure of the calling thread.
 *   - Numerics: element-wise results reproduce the reference's NumPy IEEE
 *     operation sequence bit for bit; norms are deterministic device
 *     reductions (same value on every run, not OpenBLAS's summation order).
 */
#ifndef XMHD_B200_H
#define XMHD_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define XMHD_OK 0
#define XMHD_NONFINITE 1
#define XMHD_BADARG 2
#define XMHD_CUDA_ERROR 3

/* Boundary kinds: mhd.py:34-36 (XMHD_BC_HALO = y-strip rows from neighbour ranks). */
#define XMHD_BC_PERIODIC 0
#define XMHD_BC_REFLECTING 1
#define XMHD_BC_HALO 2

/* Leja status (leja.py:103-150). */
#define XMHD_LEJA_RUNNING 0
#define XMHD_LEJA_CONVERGED 1
#define XMHD_LEJA_BLOWUP 2        /* non-converged result, residual = inf (leja.py:135-139) */
#define XMHD_LEJA_RHS_NONFINITE 3 /* matvec hit a non-finite RHS: caller raises            */
#define XMHD_LEJA_NEED_COEFFS 4   /* grow the coefficient chunk (leja.py:128-130)           */
#define XMHD_LEJA_EXHAUSTED 5     /* 499 terms, not converged (leja.py:149-150)            */
#define XMHD_LEJA_PEER_TIMEOUT 6  /* y-strips over peer memory: a rank never posted its sums */

typedef struct xmhd_ctx xmhd_ctx;

typedef struct xmhd_leja_state {
  int status;      /* XMHD_LEJA_* */
  int iterations;  /* matvecs performed = PhiApplyResult.iterations        */
  int rhs_calls;   /* RHS evaluations (advance RhsOperator.calls by this)   */
  int m;           /* next Newton index                                     */
  double residual; /* PhiApplyResult.residual                              */
  double eps;      /* FD step of the last matvec (diagnostics, blow-up repro) */
  double ynorm;    /* ||y|| of the current Newton basis vector              */
} xmhd_leja_state;

/* Record of one asynchronous step (xmhd_async_*), read back once at its end. */
#define XMHD_ASYNC_LEJA_MAX 32
typedef struct xmhd_step_record {
  int rhs_nonfinite;   /* an asynchronous RHS / JVP evaluation produced non-finite cells */
  int jvp_calls;       /* RHS evaluations made by the asynchronous JVPs (zero w: none)   */
  int nleja;           /* phi-actions recorded (xmhd_leja_finish_async calls)          */
  int lin_nonfinite;   /* F(u) of the last xmhd_linearize_async had non-finite cells    */
  double err_diff;     /* ||a - b|| of xmhd_diff_norms_async                          */
  double err_ref;      /* ||b||                                                        */
  double lc_norm;      /* ||out|| of the last xmhd_lincomb_async                       */
  double lc_nonfinite; /* 1.0 when that combination has non-finite entries             */
  xmhd_leja_state leja[XMHD_ASYNC_LEJA_MAX];
} xmhd_step_record;

/* Context for one (local) grid: the geometry + MHDParams captured by
 * RhsOperator(lambda flat: mhd_rhs(geometry.with_flat(flat), params))
 * (harness.py:129; mhd.py:39-48, 51-70).  `stream` is a cudaStream_t (0 = legacy). */
int xmhd_create(xmhd_ctx** out, int nx, int ny, double dx, double dy, double mu, double eta,
                double kappa, double gamma, double mu0, int bc_x, int bc_y, void* stream);
int xmhd_destroy(xmhd_ctx* ctx);
int xmhd_set_stream(xmhd_ctx* ctx, void* stream);
const char* xmhd_last_error(void);
/* Launch geometry chosen for the stencil (units, grid) — diagnostics/benchmarks. */
int xmhd_plan_info(xmhd_ctx* ctx, int* out4);
/* Kernels launched by this context since creation (bench "gpu_launches"). */
long long xmhd_launch_count(xmhd_ctx* ctx);

/* y-strip decomposition: halo rows (2 rows above / below, layout [field][2][nx])
 * for the base state and for the current JVP direction.  Only with bc_y == XMHD_BC_HALO. */
int xmhd_set_halo(xmhd_ctx* ctx, const double* lo, const double* hi, const double* lo_dir,
                  const double* hi_dir);

/* Non-finite cells of a failed RHS evaluation, the payload of the reference's
 * RhsBlowupError (mhd.py:225-231: message from the first cell, `cells` = the
 * first 8 in C order): bad_cells[0] = number of non-finite entries,
 * bad_cells[1 + 3k .. 3 + 3k] = (field, i, j) of the k-th (k < 8), -1 when
 * unused.  j is the row of THIS context's grid (a y-strip adds its y0). */
#define XMHD_BAD_CELLS_LEN 25

/* mhd_rhs (mhd.py:127-232): f = F(u).  Replaces the RHS callback
 * `lambda flat: mhd_rhs(geometry.with_flat(flat), params)` (harness.py:129).
 * On XMHD_NONFINITE, bad_cells (int[XMHD_BAD_CELLS_LEN], may be NULL) receives
 * the cells. */
int xmhd_rhs(xmhd_ctx* ctx, const double* u, double* f, int* bad_cells);

/* jvp (linearize.py:56-67): out = (F(u + eps*w) - fu) / eps with
 * eps = sqrt(eps_mach)*max(1,unorm)/max(||w||,1e-300); zero w -> zeros, no RHS call.
 * *called = number of RHS evaluations (0 or 1); *out_norm = ||out|| (may be NULL).
 * On XMHD_NONFINITE, bad_cells (may be NULL) receives the cells of
 * F(u + eps*w), the evaluation the reference raises from (single domain). */
int xmhd_jvp(xmhd_ctx* ctx, const double* u, const double* fu, double unorm, const double* w,
             double* out, int* called, double* out_norm, int* bad_cells);

/* The tail of _stage_difference (integrators.py:146-153) in one stencil pass:
 * out = (fstage - fu) - jvp(d) with d = stage - u and dnorm = ||d|| as reduced by
 * xmhd_lincomb_diff (same bits as xmhd_norm(d)); fstage = F(stage) from xmhd_rhs.
 * Counters and the non-finite contract are xmhd_jvp's. */
int xmhd_stage_difference(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                          const double* d, double dnorm, const double* fstage, double* out,
                          int* called, int* bad_cells);

/* apply_phi_leja (leja.py:103-150) for the frozen MHD Jacobian in ONE call:
 * p_out = phi_l(dt J(u)) v by Newton interpolation at the Leja points xi[500]
 * on [q - 2 theta, q + 2 theta], the whole loop on the device.  `coeffs` holds
 * ncoef entries of the table the reference indexes (xmhd_leja_schedule builds
 * the uncached one; a caller with a coefficient cache passes its cached chunk
 * where leja.py:90-99 would return it).  Outputs = PhiApplyResult: iterations
 * (= RHS evaluations, *rhs_calls), converged (0/1), residual (inf after a
 * blow-up).  Non-convergence is a result, not an error (XMHD_OK); a
 * non-finite RHS returns XMHD_NONFINITE with bad_cells filled (the reference
 * raises RhsBlowupError from the matvec); a table shorter than the degree
 * reached returns XMHD_BADARG.  Single-domain contexts only. */
int xmhd_leja(xmhd_ctx* ctx, int l, const double* u, const double* fu, double unorm,
              const double* v, double dt, double q, double theta, double tol,
              const double* xi, const double* coeffs, int ncoef, double* p_out,
              int* iterations, int* converged, double* residual, int* rhs_calls,
              int* bad_cells);

/* Asynchronous single-domain steps: every call below only enqueues work on the
 * context's stream; xmhd_async_fetch synchronises once and returns the step's
 * record.  The host driver (integrators.step) replays the step through the
 * synchronous entry points whenever the record shows an event the reference
 * reacts to mid-step (a non-finite RHS raising RhsBlowupError, a phi-action
 * needing more coefficients), so counters and results stay the reference's.
 *   xmhd_async_begin        reset the record
 *   xmhd_rhs_async          f = F(u) (mhd.py:127-232), non-finite cells -> record
 *   xmhd_jvp_async          jvp (linearize.py:56-67) with ||w|| and eps on the device
 *   xmhd_leja_loop          the whole Leja loop of the started phi-action in one
 *                           cooperative launch (after xmhd_leja_start_async)
 *   xmhd_leja_finish_async  p_out = the interpolant; its final state -> record
 *   xmhd_lincomb_async      xmhd_lincomb with ||out|| and the non-finite flag -> record
 *   xmhd_diff_norms_async   error_norm inputs (integrators.py:88-96) -> record */
int xmhd_async_begin(xmhd_ctx* ctx);
int xmhd_rhs_async(xmhd_ctx* ctx, const double* u, double* f);
int xmhd_jvp_async(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                   const double* w, double* out);
int xmhd_leja_loop(xmhd_ctx* ctx);
int xmhd_leja_loop_available(xmhd_ctx* ctx);
/* Loop kernel of xmhd_leja_loop: 0 = 2D tiles (default; XMHD_TILE=0 in the
 * environment selects 1), 1 = the sliding-window iteration kernel in a loop,
 * 2 = none (xmhd_leja_loop_available reports 0: xmhd_leja runs per-term
 * launches, the large-grid path, on any grid). */
int xmhd_set_loop_kind(xmhd_ctx* ctx, int kind);
/* Deferred interpolant stores of the fused Leja kernels (default on; XMHD_PDEFER=0
 * in the environment turns them off): an odd Newton term neither reads nor
 * stores p, the even term after it forms p + c*y (and its norm, resolving the
 * odd term's residual first) before its own update and stores, in the
 * reference's order (same bits): 320 instead of 384 B/cell per term.  A call
 * that converged on the odd term discards the even one (not counted). */
int xmhd_set_leja_defer(xmhd_ctx* ctx, int on);
/* Adaptive lookahead for the started single-domain call run by xmhd_leja_launch:
 * from term m0 on (0: never; xmhd_leja / xmhd_leja_start pick m0 from
 * xmhd_leja_hint) every term is enqueued as the pair {scheduled variant,
 * store variant}.  An odd term that may be the last one (the residual before
 * it was already <= tol) then resolves its own residual instead of leaving it
 * to one more full launch; exactly one kernel of a pair runs, the other exits.
 * Same terms, same bits, same counters.  XMHD_ADAPTIVE=0 disables it. */
int xmhd_leja_set_dual_from(xmhd_ctx* ctx, int m0);
/* xmhd_leja_start_async with an in-place start, for calls run by per-term
 * launches (xmhd_leja_launch; not xmhd_leja_loop): nothing is copied -- the
 * first term reads v where it lies (leja.py:121 `y = v`) and the interpolant
 * c0*v (leja.py:123) is formed by the first term that reads it; v must stay
 * untouched until the call's result has been taken.  Same bits, two vector
 * passes less per call.  (xmhd_leja and xmhd_leja_start start in place
 * themselves when they run per-term launches.) */
int xmhd_leja_start_inplace(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                            const double* v, double dt, double q, double theta, double tol,
                            const double* xi, const double* coeffs, int ncoef);
/* Caller-owned interpolant buffers (two distinct vectors, or two NULLs to return
 * to the context's own) for the following single-domain calls; with them
 * xmhd_leja_result_inplace hands the result back in buffer *which (0 / 1)
 * without a copy when the last term stored it, else after one p + c*y pass. */
int xmhd_leja_set_pbuf(xmhd_ctx* ctx, double* p0, double* p1);
int xmhd_leja_result_inplace(xmhd_ctx* ctx, int* which);
int xmhd_leja_finish_async(xmhd_ctx* ctx, double* p_out);
int xmhd_lincomb_async(xmhd_ctx* ctx, double* out, long long n, const double* const* v,
                       const double* coeffs, int nterms);
int xmhd_diff_norms_async(xmhd_ctx* ctx, const double* a, const double* b, long long n);
int xmhd_async_fetch(xmhd_ctx* ctx, xmhd_step_record* out);

/* One exponential Rosenbrock step enqueued natively with the operations and
 * order of the asynchronous Python step (integrators.py:156-199): scheme
 * XMHD_SCHEME_EXPRB43 (5 phi-actions) or XMHD_SCHEME_EXPRB54S4 (10).
 * phi_param: per phi-action, in call order, [dt_eff, q, theta] as the host
 * computed them (shift_and_scale); tables: per phi-action the first 64 Newton
 * coefficients (the host's _newton_coeffs, keeping the reference's cache);
 * tiny_alpha: alpha < 1e-14, phi_l(0) v = v / l! without Leja.  work:
 * XMHD_STEP_WORK * n doubles of scratch; u_new: the higher-order solution.
 * Starts a step record (xmhd_async_begin); read it with xmhd_async_fetch. */
#define XMHD_SCHEME_EXPRB43 0
#define XMHD_SCHEME_EXPRB54S4 1
#define XMHD_STEP_WORK 20
int xmhd_step_async(xmhd_ctx* ctx, int scheme, const double* u, const double* fu, double unorm,
                    long long n, double dt, const double* phi_param, const double* tables,
                    int tiny_alpha, double tol, const double* xi, double* work, double* u_new);

/* Power iteration of estimate_alpha (linearize.py:113-135; replaces the loop at
 * linearize.py:118-133 that the reference runs over jvp and np.linalg.norm).
 * w0: start vector (read only; a zero w0 starts from ones as linearize.py:115-116).
 * w: out, the last normalised iterate (SpectralEstimate.vector).  work: n-double
 * scratch.  Stops when |mag - mags[-2]| or |mag - mags[-3]| <= tol*mag, or after
 * maxit (<= 100) iterations.  mags[0..*nit): the magnitudes ||J w||;
 * *rhs_calls: RHS evaluations; *status: 0 = alpha from max(mags[-3:]),
 * 1 = magnitude < 1e-300 or non-finite (alpha 0, no vector).  Returns
 * XMHD_NONFINITE when an RHS evaluation produced non-finite cells (the
 * reference raises RhsBlowupError from inside jvp).  Single-domain contexts. */
int xmhd_power(xmhd_ctx* ctx, const double* u, const double* fu, double unorm, const double* w0,
               double* w, double* work, int maxit, double tol, double* mags, int* nit,
               int* rhs_calls, int* status);

/* FrozenLinearization (linearize.py:46-53): fu = F(u) and *unorm = ||u|| with one
 * host synchronisation; XMHD_NONFINITE when F(u) has non-finite cells.
 * Single-domain contexts. */
int xmhd_linearize(xmhd_ctx* ctx, const double* u, double* fu, double* unorm);

/* The same without a host wait, for a caller that knows ||u|| (the harness:
 * the previous step's flagged combination already reduced it, bit for bit):
 * fu = F(u); its non-finite flag is read by xmhd_linearize_check (one sync)
 * or arrives with the next step record (lin_nonfinite). */
int xmhd_linearize_async(xmhd_ctx* ctx, const double* u, double* fu);
int xmhd_linearize_check(xmhd_ctx* ctx, int* nonfinite);

/* max |div B| (mhd.py:235-240) into a device double, no host wait. */
int xmhd_divb_async(xmhd_ctx* ctx, const double* u, double* out_dev);

/* np.linalg.norm(x) (deterministic device reduction). */
int xmhd_norm(xmhd_ctx* ctx, const double* x, long long n, double* out);

/* out = ((c0*v0 + c1*v1) + c2*v2) + c3*v3, the stage algebra of integrators.py:139-199.
 * norm_out / nonfinite_out may be NULL (then no reduction is performed). */
int xmhd_lincomb(xmhd_ctx* ctx, double* out, long long n, const double* const* v,
                 const double* c, int nterms, double* norm_out, int* nonfinite_out);
/* A stage vector and its offset from the base state in one pass
 * (integrators.py:139-153): out = the combination above with v[0] = u, c[0] = 1;
 * diff = out - v[0]; *diff_norm = ||diff||. */
int xmhd_lincomb_diff(xmhd_ctx* ctx, double* out, double* diff, long long n,
                      const double* const* v, const double* c, int nterms, double* diff_norm);
/* nout (2..4) combinations of the same three vectors in one pass (the w_k of
 * integrators.py:166-167, 186-189): out[j] = sum_k coef[3j+k]*v[k], k in order,
 * zero coefficients skipped (a term the reference's expression does not have). */
int xmhd_lincomb_multi(xmhd_ctx* ctx, double* const* out, int nout, long long n,
                       const double* const* v, const double* coef);
/* The two embedded solutions of an exponential Rosenbrock step and their
 * distance in one pass (integrators.py:168-171 / 190-199 with error_norm,
 * 88-96): the lower-order solution is formed on the fly, the higher-order one
 * goes to out_hi; err_out[0] = ||lo - hi||, err_out[1] = ||hi||, *nonfinite = hi
 * has a non-finite entry.  Same operations, order and reductions as the
 * separate xmhd_lincomb calls followed by xmhd_diff_norms.
 *   XMHD_SCHEME_EXPRB43:   v = {u, phi1, p3, p4},            c = {1, dt, dt, dt}:
 *     lo = (c0*v0 + c1*v1) + c2*v2;  hi = 1.0*lo + c3*v3
 *   XMHD_SCHEME_EXPRB54S4: v = {u, phi1, p3, p4, p3', p4'},  c = {1, dt, dt, dt, dt, dt}:
 *     s = c0*v0 + c1*v1;  lo = (s + c2*v2) + c3*v3;  hi = (s + c4*v4) + c5*v5 */
int xmhd_final_pair(xmhd_ctx* ctx, int scheme, double* out_hi, long long n,
                    const double* const* v, const double* c, double* err_out, int* nonfinite);

/* out = x / d elementwise (IEEE), optionally ||out|| (w/||w||, jw/mag, v/l!). */
int xmhd_divide(xmhd_ctx* ctx, double* out, const double* x, double d, long long n,
                double* norm_out);

/* error_norm pieces (integrators.py:88-96): out[0] = ||a-b||, out[1] = ||b||. */
int xmhd_diff_norms(xmhd_ctx* ctx, const double* a, const double* b, long long n, double* out);

/* Diagnostics: max|discrete_div_b| (mhd.py:235-240), per-field sums
 * (conserved_totals before the area factor, mhd.py:243-247), and the two
 * CFL speed maxima of harness.py:105-116. */
int xmhd_divb(xmhd_ctx* ctx, const double* u, double* field, double* out_max);
int xmhd_field_sums(xmhd_ctx* ctx, const double* u, double* out8);
int xmhd_cfl_speeds(xmhd_ctx* ctx, const double* u, double* out2);

/* apply_phi_leja with matvec = jvp(lin, .) fused into the stencil (leja.py:103-150;
 * integrators.py:117-136).  xi: 500 Leja points (host), coeffs: ncoef Newton
 * coefficients (host).  Runs device-side until the status leaves RUNNING. */
int xmhd_leja_start(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                    const double* v, double dt, double q, double theta, double tol,
                    const double* xi, const double* coeffs, int ncoef, xmhd_leja_state* st);
/* Expected number of Newton terms of the next xmhd_leja_start (host-side
 * launch batching only; results do not depend on it). */
int xmhd_leja_hint(xmhd_ctx* ctx, int expected_iterations);
/* Host-paced form of the same loop (what the Python mirror uses): start
 * without running (xmhd_leja_start_async, or xmhd_leja_p2p_start), enqueue n
 * iteration kernels without waiting (peer != 0: the y-strip peer-memory
 * kernel); extend the device coefficient table to `to` entries with
 * coeffs[from..to) ahead of the terms that need them (the values the reference
 * would fetch when the chunk grows, leja.py:128-130), so the loop never stops
 * at a chunk boundary; sync and read the state.  Kernels enqueued after the
 * status left RUNNING exit immediately. */
int xmhd_leja_start_async(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                          const double* v, double dt, double q, double theta, double tol,
                          const double* xi, const double* coeffs, int ncoef);
int xmhd_leja_launch(xmhd_ctx* ctx, int n, int peer);
int xmhd_leja_extend(xmhd_ctx* ctx, const double* coeffs, int from, int to);
int xmhd_leja_sync(xmhd_ctx* ctx, xmhd_leja_state* st);
/* After XMHD_LEJA_NEED_COEFFS: upload the grown chunk and continue. */
int xmhd_leja_resume(xmhd_ctx* ctx, const double* coeffs, int ncoef, xmhd_leja_state* st);
/* Copy the interpolant p of the finished call into p_out (device, 8*nx*ny). */
int xmhd_leja_result(xmhd_ctx* ctx, double* p_out);
/* Copy the current Newton basis vector y into dst (generic matvec input, RHS blow-up replay). */
int xmhd_leja_current_y(xmhd_ctx* ctx, double* dst);

/* apply_phi_leja for an arbitrary caller-supplied matvec (leja.py:103-150):
 * start -> loop { current_y; w = matvec(y) on the caller side; step } -> result. */
int xmhd_leja_generic_start(xmhd_ctx* ctx, const double* v, long long n, double dt, double q,
                            double theta, double tol, const double* xi, const double* coeffs,
                            int ncoef, xmhd_leja_state* st);
int xmhd_leja_generic_step(xmhd_ctx* ctx, const double* w, xmhd_leja_state* st);
int xmhd_leja_generic_resume(xmhd_ctx* ctx, const double* coeffs, int ncoef,
                             xmhd_leja_state* st);
int xmhd_leja_generic_result(xmhd_ctx* ctx, double* p_out);

/* ---- y-strip decomposition (bc_y == XMHD_BC_HALO) ----------------
 * Each rank owns rows [y0, y0+ny) of every field.  Every norm is a cross-rank
 * sum, so these entry points expose local partial sums and the control updates
 * that run after the caller's allreduce; all ranks then take identical
 * decisions.  Sequence per Leja term (stream-ordered, no host sync):
 *   strip_pack -> halo exchange of y (caller, NCCL P2P) -> strip_iterate(sums)
 *   -> allreduce(sums[0..2], SUM) (caller) -> strip_finalize(sums). */
int xmhd_sumsq(xmhd_ctx* ctx, const double* x, long long n, double* out);
/* jvp with the FD step eps given by the caller (from the global ||w||);
 * *out_sumsq = local sum of squares of the result (may be NULL). */
int xmhd_jvp_eps(xmhd_ctx* ctx, const double* u, const double* fu, const double* w, double eps,
                 double* out, double* out_sumsq);
/* y = v, p = c0*v; sums[0] (device) = local sum of v^2; then strip_start_finalize. */
int xmhd_leja_strip_start(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                          const double* v, double dt, double q, double theta, double tol,
                          const double* xi, const double* coeffs, int ncoef, double* sums);
int xmhd_leja_strip_start_finalize(xmhd_ctx* ctx, const double* sums);
/* Boundary rows of the current y into send buffers / mirrored ghost rows ([field][2][nx]). */
int xmhd_leja_strip_pack(xmhd_ctx* ctx, double* send_lo, double* send_hi, double* halo_lo_dir,
                         double* halo_hi_dir, int mirror_lo, int mirror_hi);
/* One fused Newton term on the strip; sums[0..2] (device) = local [sum y'^2, sum p'^2, bad]. */
int xmhd_leja_strip_iterate(xmhd_ctx* ctx, double* sums);
/* Control update from the allreduced sums (no-op once the call has finished). */
int xmhd_leja_strip_finalize(xmhd_ctx* ctx, const double* sums);
int xmhd_leja_query(xmhd_ctx* ctx, xmhd_leja_state* st);
/* Upload a grown coefficient chunk and clear NEED_COEFFS without running. */
int xmhd_leja_set_coeffs(xmhd_ctx* ctx, const double* coeffs, int ncoef);

/* Benchmark hook: average duration (CUDA events on the context stream) of
 * n_iter back-to-back stencil launches, mode 0 = F(u) into out (as xmhd_rhs),
 * mode 1 = the FD Jacobian-vector product of w into out (as xmhd_jvp; fu, unorm
 * and w required).  Returns XMHD_NONFINITE like those calls. */
int xmhd_time_stencil(xmhd_ctx* ctx, int mode, const double* u, const double* fu, double unorm,
                      const double* w, double* out, int n_iter, double* ms_per_launch);

/* Benchmark hook: average duration (CUDA events on the context stream) of
 * n_iter back-to-back fused Leja iteration kernels with the convergence test
 * disabled (tol = 0); coeffs500 holds 500 Newton coefficients.  With
 * ms_by_kind (may be NULL) an event separates every launch and
 * ms_by_kind[0] / [1] receive the average of the odd (PM_SKIP, 256 B/cell)
 * and even (PM_LOOK, 384 B/cell) terms of the lookahead schedule. */
int xmhd_time_leja_iterations(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                              const double* v, double dt, double q, double theta,
                              const double* xi, const double* coeffs500, int n_iter,
                              double* ms_per_iter, double* ms_by_kind);

/* ---- y-strips over peer memory (one NVLink / NVSwitch node, CUDA IPC) ----
 * Replaces the per-term halo exchange + allreduce of the strip driver (the
 * NCCL path above) inside the fused iteration kernel: it stores the boundary
 * rows of y' into the neighbours' ghost-row buffers and all-reduces its
 * [sum y'^2, sum p'^2, bad] through per-rank boards in peer memory, so a
 * Newton term is one kernel launch on every rank and no host call.
 *
 * Setup (once per strip context): xmhd_p2p_alloc returns this rank's 64-byte
 * CUDA IPC handle; the caller all-gathers the handles (any transport) and
 * calls xmhd_p2p_connect with all of them.  periodic: the strips form a ring
 * in y; otherwise the end ranks build mirrored ghost rows (reflecting walls).
 * The state's ghost rows are still set with xmhd_set_halo (once per call). */
int xmhd_p2p_alloc(xmhd_ctx* ctx, void* ipc_handle_out);
int xmhd_p2p_connect(xmhd_ctx* ctx, int rank, int nranks, const void* ipc_handles,
                     int periodic);
/* Connectivity probe: write `value` into every rank's board (no waiting) /
 * read this rank's board: out[4*q] = value written by rank q, out[4*q+1] = q. */
int xmhd_p2p_probe(xmhd_ctx* ctx, double value);
int xmhd_p2p_read_board(xmhd_ctx* ctx, double* out /* 32 doubles */);
/* One phi-action on the strips: start (y0 = v, p0 = c0*v, global ||v||, ghost
 * rows of y0), then run until the status leaves RUNNING; NEED_COEFFS:
 * xmhd_leja_set_coeffs + xmhd_leja_p2p_run again.  Results: xmhd_leja_result. */
int xmhd_leja_p2p_start(xmhd_ctx* ctx, const double* u, const double* fu, double unorm,
                        const double* v, double dt, double q, double theta, double tol,
                        const double* xi, const double* coeffs, int ncoef);
int xmhd_leja_p2p_run(xmhd_ctx* ctx, xmhd_leja_state* st);
/* Test driver: nranks strip contexts on ONE GPU sharing one stream, wired to
 * each other's regions directly, every Newton term ONE cooperative launch
 * over all ranks' blocks (ranks that wait on each other must be co-resident). */
int xmhd_p2p_connect_local(xmhd_ctx* const* ctxs, int nranks, int periodic);
int xmhd_leja_p2p_emul_start(xmhd_ctx* const* ctxs, int nranks, const double* const* u,
                             const double* const* fu, double unorm, const double* const* v,
                             double dt, double q, double theta, double tol, const double* xi,
                             const double* coeffs, int ncoef);
int xmhd_leja_p2p_emul_run(xmhd_ctx* const* ctxs, int nranks, xmhd_leja_state* st);

/* ---- Krylov baseline (replaces the NumPy Arnoldi loop of krylov.py:34-84) ----
 * The paper's Leja-vs-Krylov comparison arm; the Hessenberg matrix and its
 * phi_l(H)e1 stay on the host (at most 200 x 200).
 *
 * xmhd_krylov_mgs: both modified Gram-Schmidt passes of Arnoldi step j
 * (krylov.py:60-67) against basis[0..nb-1] (device vectors of n doubles), w
 * updated in place.  Stream-ordered: each update reads the previous launch's
 * reduced dot from device memory; one host sync at the end.
 * coef_out[0..nb) = pass-1 coefficients, coef_out[nb..2nb) = pass-2;
 * *wsumsq_out = sum(w^2) after both passes (||w||^2 of krylov.py:68). */
int xmhd_krylov_mgs(xmhd_ctx* ctx, const double* const* basis, int nb, double* w, long long n,
                    double* coef_out, double* wsumsq_out);
/* One MGS update for y-strip callers (coefficients are global, reduced by the
 * caller between updates): w -= coef*v (v may be NULL: no update), then
 * *sum_out = local sum(next * w) (sum(w * w) when next is NULL). */
int xmhd_mgs_update(xmhd_ctx* ctx, double* w, long long n, const double* v, double coef,
                    const double* next, double* sum_out);
/* out = scale * sum_k coef[k] * basis[k], k = 0..m-1 (m <= 200; krylov.py:79-80). */
int xmhd_krylov_combine(xmhd_ctx* ctx, const double* const* basis, const double* coef, int m,
                        double scale, long long n, double* out);

/* Host C++ port of _phi_divided_diffs (phi.py:99-144): first column of
 * phi_l of the bidiagonal node matrix, bitwise equal to the NumPy routine.
 * out has n entries. */
int xmhd_phi_divided_diffs(int l, const double* nodes, int n, double subdiag, double* out);
/* _newton_coeffs without the cache (leja.py:94-96): the first `count` Newton
 * coefficients of phi_l(q + theta*xi) / theta**l (host, bitwise NumPy). */
int xmhd_newton_coeffs(int l, double q, double theta, const double* xi, int count, double* out);
/* The 500-entry table an uncached apply_phi_leja call indexes with the chunk
 * schedule of leja.py:119-130 (64 -> 128 -> 256 -> 500, each chunk recomputed):
 * entries [0,64) of the 64-chunk, [64,128) of the 128-chunk, ... (host). */
int xmhd_leja_schedule(int l, double q, double theta, const double* xi, double* out500);

/* Pageable host memory -> device, the H2D of a reference caller's NumPy array
 * (the reference's API takes host arrays: leja.py:103, linearize.py:46-53).
 * A persistent pool of host threads (xmhd_h2d_threads; env XMHD_H2D_THREADS)
 * fills page-locked slots while the copy engine drains the ones filled before,
 * in `stream` order.  Returns once src_host is no longer read; the device copy
 * completes in stream order.  No context: one staging area per process. */
int xmhd_h2d_staged(void* dst_dev, const void* src_host, long long bytes, void* stream);
int xmhd_h2d_threads(void);

/* Measurement aid (bench.py's roofline): device time of the fused Leja terms
 * inside a timed region.  While enabled, every batch of term launches of this
 * context (xmhd_leja, xmhd_leja_launch) is bracketed by two CUDA events on the
 * context's stream; the pairs are read at the call's next host synchronisation.
 * enable = 1 / 0: synchronise, write the milliseconds accumulated so far to
 * *total_ms (may be NULL), reset the sum and switch the brackets on / off;
 * enable < 0: read the sum only.  Launches that exit at once (past a stop, the
 * idle variant of a pair) are inside the brackets. */
int xmhd_term_timing(xmhd_ctx* ctx, int enable, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* XMHD_B200_H */
