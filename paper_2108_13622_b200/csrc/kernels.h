// Internal (C++) interface between the C-ABI layer and the CUDA kernels.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include "common.cuh"

namespace xb {

// Device-resident control block of one Leja phi-action (leja.py:103-150).
// Written only by the last block of each fused iteration kernel.
struct LejaCtl {
  int m;            // next Newton index to compute (1 .. 499)
  int status;       // LejaStatus
  int small_prev;   // previous residual <= tol
  int ncoef;        // valid coefficients on the device
  int cur;          // index of the current y / p buffer
  int rhs_calls;    // RHS evaluations performed (zero directions excluded)
  int iters;        // matvecs performed
  int zero_dir;     // current y has norm 0 (jvp short-circuit, linearize.py:63-64)
  int fbad;         // an RHS evaluation produced non-finite cells
  int pad_;
  double eps;       // FD step for the next JVP (linearize.py:65)
  double ynorm;     // ||y|| of the current y
  double pnorm;
  double residual;
  double blowup;    // 1e120 * max(1, ||v||)   (leja.py:122)
  double unorm;     // ||u|| of the frozen linearization
  double dt, q, theta, tol;
  Divisor epsd;     // eps with its RN reciprocal (exact division in the epilogue)
  Divisor thetad;   // theta, likewise (host-computed)
  int force_ieee;   // testing: plain IEEE division for eps as well
  int pad2_;
  unsigned long long epoch;   // y-strips over peer memory: last exchange epoch
  // Deferred interpolant update: with `defer` set, every other term leaves
  // p' = p + c_m*y_m in registers (for ||p'||) without storing it; the next
  // term adds c_m*y_m (its own direction) before its own update and stores.
  // Same two roundings per element as the reference's p = p + c*y per term
  // (bitwise-identical p and norms), 352 instead of 384 B per cell per term.
  // defer == 2 (single domain, "lookahead"): an odd term neither reads nor
  // stores p (y' and ||y'|| only, 256 B/cell); the even term after it reads
  // p, forms p_m = p + c_m*y_m and ||p_m|| (resolving the odd term's
  // residual first, in the reference's order) and then its own update, and
  // stores (384 B/cell): 320 B per term.  A call that converged on the odd
  // term discards the even one (no iteration, no RHS call counted).
  int pcur;         // buffer holding the last stored interpolant
  int ppend;        // 1: the interpolant is pbuf[pcur] + pend_coef * ybuf[cur]
  int defer;        // 0: store every term; 1: every other term; 2: with lookahead
  int pmode;        // LejaPMode of the next term (= leja_pmode(m, defer))
  double pend_coef; // coefficient of the pending term
  double pend_ynorm;// ||y|| of a term whose residual is not resolved yet
  // In-place start (single domain, host-paced terms): the caller's v is read
  // as the first direction and the interpolant is c0 * v, formed on the fly by
  // whoever reads it, until the first term that stores p (StencilArgs::v0).
  int pvirt;        // 1: the stored interpolant is still c0 * v (nothing in pbuf)
  int pad3_;
  double c0;        // coeffs[0]
};

// What a term does with the interpolant.
enum LejaPMode {
  PM_ANY = -1,    // (kernel template) read the mode from the control block
  PM_STORE = 0,   // read p (+ pending term), add c*y', store
  PM_KEEP = 1,    // read p, add c*y' in registers for ||p'||, no store (defer 1)
  PM_SKIP = 2,    // neither read nor store p: y' and ||y'|| only (defer 2)
  PM_LOOK = 3,    // read p, add the pending term (||.|| of it), add c*y', store
};

// The scheduled mode of term m: a pure function of m, so the host launches the
// kernel variant compiled for it (and the kernel checks it against the device's).
__host__ __device__ __forceinline__ int leja_pmode(int m, int defer) {
  if (defer == 2) return m >= 499 ? PM_STORE : ((m & 1) ? PM_SKIP : PM_LOOK);
  if (defer == 1) return (m & 1) ? PM_KEEP : PM_STORE;
  return PM_STORE;
}

// The mode the device picks for the next term m.  With the lookahead schedule
// a call that converges on an odd (PM_SKIP) term only finds out in the next
// launch, which then was a full term computed for nothing.  When the host
// enqueues term m as a {scheduled variant, PM_STORE} pair (`dual`), an odd term
// that could be the last one (the residual before it was already small) runs
// as PM_STORE instead: it reads and stores p and resolves its own residual.
// The even term after such a term has no pending term to resolve: PM_STORE.
__host__ __device__ __forceinline__ int leja_next_pmode(int m, int defer, int dual, int small_prev,
                                                        int ppend) {
  if (defer != 2 || m >= 499) return leja_pmode(m, defer);
  if (m & 1) return (dual && small_prev) ? PM_STORE : PM_SKIP;
  return ppend ? PM_LOOK : PM_STORE;
}

enum LejaStatus {
  LJ_RUNNING = 0,
  LJ_CONVERGED = 1,
  LJ_BLOWUP = 2,       // Newton basis blew up: non-converged result (leja.py:135-139)
  LJ_RHS_BAD = 3,      // non-finite RHS: the reference raises RhsBlowupError
  LJ_NEED_COEFFS = 4,  // m reached the coefficient chunk size (leja.py:128-130)
  LJ_EXHAUSTED = 5,    // 499 terms without convergence (leja.py:149-150)
  LJ_PEER_TIMEOUT = 6, // y-strips over peer memory: a peer never posted its sums
  LJ_MODE_ERROR = 7,   // a kernel variant launched for another interpolant mode
};

// Device-resident power iteration of estimate_alpha (linearize.py:113-135):
// one fused JVP (J w, ||J w||) and one division kernel (w = J w / mag, ||w||,
// next FD step) per iteration; both last blocks update this block, so the
// host only enqueues kernels and reads the block back once per batch.
constexpr int POWER_MAXIT = 100;   // linearize.py _POWER_MAXIT
struct PowerCtl {
  int status;       // PowerStatus
  int k;            // magnitudes recorded
  int maxit;
  int rhs_calls;    // JVPs evaluated (zero directions excluded)
  int stop;         // converged (or maxit): the next division is the last kernel
  int jvp_only;     // plain asynchronous jvp: the JVP only counts its RHS call
  double unorm;     // ||u|| of the frozen linearization
  double tol;       // relative change accepted against mags[-2] or mags[-3]
  double div;       // divisor of the next division (||w0||, then mag)
  double wn;        // ||w|| of the current iterate
  double eps;       // FD step of the next JVP
  Divisor epsd;
  int force_ieee;
  int pad2_;
  double mags[POWER_MAXIT];
};

enum PowerStatus {
  PW_RUNNING = 0,
  PW_DONE = 1,      // converged or maxit: alpha = safety * max(mags[-3:])
  PW_ZERO = 2,      // magnitude < 1e-300 or non-finite: alpha = 0, no vector
  PW_RHS_BAD = 3,   // non-finite RHS inside the JVP: the reference raises
};

constexpr int P2P_MAX = 8;   // ranks of one NVLink / NVSwitch node

// Peer-memory transport of the y-strip Leja loop.  The fused iteration kernel
// stores the boundary rows of y' straight into the neighbours' ghost-row
// buffers and all-reduces [sum y'^2, sum p'^2, bad] through per-rank boards
// whose flags carry a monotonically increasing epoch, so a Newton term needs
// no host call and no collective library.  Pointers are this process's CUDA
// IPC mappings of the peers' regions (or plain device pointers when the ranks
// are emulated in one launch on one GPU).  Ghost-row buffers are
// double-buffered by the parity of the current y (LejaCtl::cur).
struct P2PArgs {
  double* dst_lo[2];                 // per parity: destination of my rows 0, 1 ([f][2][nx])
  double* dst_hi[2];                 // destination of my rows ny-2, ny-1
  int mirror_lo, mirror_hi;          // the destination is my own ghost rows (reflecting wall)
  const double* halo_lo_dir[2];      // my ghost rows -2, -1 of the direction, per parity
  const double* halo_hi_dir[2];      // my ghost rows ny, ny+1
  double* board[P2P_MAX];            // rank q's board: [2 slots][P2P_MAX][4] doubles
  unsigned long long* flag[P2P_MAX]; // rank q's flags: [2 slots][P2P_MAX]
  int rank, nranks;
};

enum StencilMode { MODE_RHS = 0, MODE_JVP = 1, MODE_LEJA = 2 };

struct StencilArgs {
  Geom g;
  const double* u;     // base state, 8 planes of nx*ny
  const double* dir;   // JVP direction (MODE_JVP)
  const double* fu;    // cached F(u)
  double* out;         // MODE_RHS: F(u); MODE_JVP: J w
  double eps;          // MODE_JVP
  Divisor epsd;        // MODE_JVP: eps with its reciprocal
  // MODE_LEJA
  double* ybuf[2];
  double* pbuf[2];
  const double* coeffs;
  const double* xi;
  LejaCtl* ctl;
  const double* v0;    // in-place start: the call's v (direction of term 1, c0*v = p0)
  const double* stage_f; // MODE_JVP: F(stage); out = (F(stage) - F(u)) - J w (null: out = J w)
  // Adaptive lookahead (single domain, per-term launches): near the expected
  // end of a call every term is enqueued as a pair of variants -- the one the
  // parity schedule names and PM_STORE -- carrying the term index they are
  // meant for; the variant whose mode the control block does not name exits.
  int term;            // > 0: run only if the control block is at this term, silently
  int dual_next;       // the next term is enqueued as such a pair (mode rule below)
  // reductions / flags
  double* partials;    // [grid][2]
  unsigned* ticket;
  double* result;      // MODE_JVP: ||J w||
  int* bad;            // |= 1 when a non-finite F cell is produced
  double* ext_sums;    // MODE_LEJA y-strips: [sum y'^2, sum p'^2, bad] of this rank
  int units_x, nunits, seg_rows;
  // warp-specialized TMA kernel (stencil.cu, stencil_ws_kernel): its own
  // unit plan (1 CTA of 384 threads per SM); ws_grid == 0 selects the
  // one-role sliding-window kernel
  int ws_units_x, ws_nunits, ws_seg_rows, ws_grid;
  P2PArgs p2p;         // MODE_LEJA y-strips over peer memory
  PowerCtl* pctl;      // MODE_JVP inside the device power iteration (eps from here)
};

#ifndef XB_SW
#define XB_SW 128
#endif
constexpr int SW = XB_SW;        // threads per block = ghost-extended columns per strip
constexpr int SW_MINB = 256 / SW;   // resident blocks per SM the register budget targets
constexpr int SOUT = SW - 4;     // output columns per strip
size_t stencil_smem_bytes();
void stencil_plan(const Geom& g, int nsm, int& units_x, int& nunits, int& seg_rows, int& grid);
// Plan of the warp-specialized kernel; grid = 0 when it does not apply
// (odd nx: rows are not 16-byte aligned for the bulk copies; narrow grids).
void stencil_ws_plan(const Geom& g, int nsm, int& units_x, int& nunits, int& seg_rows,
                     int& grid);
cudaError_t launch_stencil(int mode, const StencilArgs& a, int grid, cudaStream_t s);
// One Newton term with the variant compiled for its interpolant mode (LejaPMode).
cudaError_t launch_leja_term(const StencilArgs& a, int grid, int pmode, cudaStream_t s);

// Vector kernels (vec.cu).
struct RedBuf {
  double* partials;    // [max_grid][4]
  unsigned* ticket;
  double* result;      // [8]
  int grid;
};
// result[0] = ||x||
cudaError_t launch_norm(const double* x, long long n, RedBuf rb, cudaStream_t s);
// out = c0*v0 + c1*v1 + c2*v2 + c3*v3 (left to right; null v ends the sum);
// result[0] = ||out|| when want_norm, result[1] = 1 if any non-finite entry.
cudaError_t launch_lincomb(double* out, long long n, const double* const* v,
                           const double* c, int nterms, int want_norm, RedBuf rb,
                           cudaStream_t s);
// out = the combination above and diff = out - v[0] in one pass; result[0] = ||diff||
// (a stage vector and the direction of its stage difference, integrators.py:139-153).
cudaError_t launch_lincomb_diff(double* out, double* diff, long long n, const double* const* v,
                                const double* c, int nterms, RedBuf rb, cudaStream_t s);
// out[j] = sum_k coef12[3j+k] * v[k] (k = 0..2 in order, zero coefficients skipped),
// j < nout <= 4: several combinations of the same three vectors in one pass.
cudaError_t launch_lincomb_multi(double* const* out, int nout, long long n,
                                 const double* const* v, const double* coef12, RedBuf rb,
                                 cudaStream_t s);
// The two embedded solutions of a step in one pass (vec.cu, FinalPairOp): the
// higher-order one into out_hi; result[0] = ||lo - hi||, result[1] = ||hi||,
// result[2] = 1 if hi has a non-finite entry.  kind 43: v[0..3], c[0..3];
// kind 54: v[0..5], c[0..5].
cudaError_t launch_final_pair(int kind, double* out_hi, long long n, const double* const* v,
                              const double* c, RedBuf rb, cudaStream_t s);
// out = x / d (IEEE), result[0] = ||out|| when want_norm.
cudaError_t launch_divide(double* out, const double* x, double d, long long n,
                          int want_norm, RedBuf rb, cudaStream_t s);
// result[0] = ||a - b||, result[1] = ||b||.
cudaError_t launch_diffnorm(const double* a, const double* b, long long n, RedBuf rb,
                            cudaStream_t s);
// result[0] = max |div B| (mhd.py:235-240 with the geometry's boundaries);
// the div B field itself is written to `field` when non-null.
cudaError_t launch_divb_max(const Geom& g, const double* u, double* field, RedBuf rb,
                            cudaStream_t s);
// result[0..7] = per-field plain sums (conserved_totals before the area factor).
cudaError_t launch_field_sums(const double* u, long long plane, RedBuf rb, cudaStream_t s);
// result[0] = max over cells of |vx| + cf, result[1] of |vy| + cf (harness.py:105-116).
cudaError_t launch_cfl(const double* u, long long plane, double gamma, double mu0,
                       RedBuf rb, cudaStream_t s);
// Leja start: y0 = v, p0 = c0*v, ctl init (norm of v, blowup, eps).  With
// ext_sums the local sum of squares goes there instead (y-strips: allreduce,
// then launch_leja_init_finalize).
cudaError_t launch_leja_init(const double* v, long long n, double* y0, double* p0,
                             LejaCtl* ctl, const double* coeffs, RedBuf rb, cudaStream_t s,
                             double* ext_sums = nullptr);
cudaError_t launch_leja_init_finalize(LejaCtl* ctl, const double* sums, cudaStream_t s);
// Control update from globally reduced [sum y'^2, sum p'^2, bad] (y-strips).
cudaError_t launch_leja_finalize(LejaCtl* ctl, const double* sums, const double* coeffs,
                                 cudaStream_t s);
// Halo rows of the current y (send buffers and/or mirrored ghost rows).
cudaError_t launch_leja_pack_halo(const LejaCtl* ctl, const double* y0, const double* y1, int nx,
                                  int ny, double* send_lo, double* send_hi, double* halo_lo,
                                  double* halo_hi, int mirror_lo, int mirror_hi, cudaStream_t s);
// Power iteration: out = x / pctl->div (IEEE) and the control update from
// ||out|| (next FD step, or the end of the iteration).  No-op unless RUNNING.
cudaError_t launch_power_divide(double* out, const double* x, long long n, PowerCtl* pctl,
                                RedBuf rb, cudaStream_t s);
// x[i] = v.
cudaError_t launch_fill(double* x, long long n, double v, cudaStream_t s);
// result[0] = sum of squares (no sqrt; y-strip partial norms).
cudaError_t launch_sumsq(const double* x, long long n, RedBuf rb, cudaStream_t s);
// Generic Leja update for an arbitrary (host-supplied) matvec result w.
cudaError_t launch_leja_update(const double* w, long long n, LejaCtl* ctl, double* const* ybuf,
                               double* const* pbuf, const double* coeffs, const double* xi,
                               RedBuf rb, cudaStream_t s);

// Krylov baseline (krylov.py:34-84).
constexpr int KRYLOV_MAX = 200;   // krylov.py:16 (M_CAP)
struct KrylovBasis {
  const double* v[KRYLOV_MAX];
  double c[KRYLOV_MAX];
};
// w -= c*v (v non-null; c = *cin, or c_host when cin is null), then
// *cout = sum(next * w) (sum(w * w) when next is null).
cudaError_t launch_mgs(double* w, long long n, const double* v, const double* cin,
                       double c_host, const double* next, double* cout, RedBuf rb,
                       cudaStream_t s);
// out = scale * sum_k c_k v_k (k = 0..m-1, left to right).
cudaError_t launch_krylov_combine(double* out, long long n, const KrylovBasis& B, int m,
                                  double scale, RedBuf rb, cudaStream_t s);

// The whole single-domain Leja loop in one cooperative launch (grid must be
// co-resident: grid <= leja_loop_max_blocks).
cudaError_t launch_leja_loop(const StencilArgs& a, int grid, cudaStream_t s);
int leja_loop_max_blocks(int nsm);
// Small grids: the same loop over 2D tiles (grid = leja_tile_loop_grid; the
// stencil partials buffer needs 6 doubles per block).
cudaError_t launch_leja_tile_loop(const StencilArgs& a, int grid, int minb, cudaStream_t s);
int leja_tile_loop_grid(const Geom& g, int nsm, int* minb);
// p_out = the interpolant of a finished call: pbuf[pcur], plus pend_coef *
// ybuf[cur] when a term is pending (no host read of the control block).
cudaError_t launch_leja_copy_result(double* p_out, const double* const* pbuf,
                                    const double* const* ybuf, const double* v0,
                                    const LejaCtl* ctl, long long n, cudaStream_t s);
// jvp prologue on the device: sum(w^2) -> ||w||, eps and its divisor in jc
// (status PW_RUNNING), or status PW_ZERO for a zero vector (linearize.py:62-65).
cudaError_t launch_jvp_prep(const double* w, long long n, double unorm, PowerCtl* jc, RedBuf rb,
                            cudaStream_t s);

// Record of one asynchronous step (read back once, at its end).
constexpr int ASYNC_LEJA_MAX = 32;
struct AsyncRec {
  int bad;          // an RHS / JVP evaluation produced non-finite cells
  int jvp_calls;    // RHS evaluations of the asynchronous JVPs
  int pad_[2];
  double err[2];    // ||a - b||, ||b|| of the error norm
  double lc[2];     // ||out||, non-finite flag of the flagged linear combination
  LejaCtl leja[ASYNC_LEJA_MAX];   // final control block of each phi-action
};

// Kernels of the peer-memory strip driver (stencil.cu / vec.cu).
cudaError_t launch_leja_peer(const StencilArgs& a, int grid, int pmode, cudaStream_t s);
// Emulation of P ranks on one GPU: ONE cooperative launch over all ranks'
// blocks (args: device array of P StencilArgs; nblk blocks per rank).
cudaError_t launch_leja_emul(const StencilArgs* args_dev, const StencilArgs& a0, int nranks,
                             int nblk, int pmode, cudaStream_t s);
int leja_emul_max_blocks(int nsm);
// Start of a peer-memory strip Leja call: exchange of sum(v^2) (ext_sums[0])
// and leja_init_ctl on the global sum.  Real ranks: one block; emulation: one
// block per rank over args_dev (cooperative).
cudaError_t launch_leja_p2p_init(const StencilArgs& a, cudaStream_t s);
cudaError_t launch_leja_p2p_init_emul(const StencilArgs* args_dev, int nranks, cudaStream_t s);
// Coefficient table grown to `to` entries (clears NEED_COEFFS when it applies).
cudaError_t launch_leja_extend(LejaCtl* ctl, int to, cudaStream_t s);
// Connectivity probe: write `value` into every peer board (slot 0, my row).
cudaError_t launch_p2p_probe(const P2PArgs& x, double value, cudaStream_t s);
// Non-finite scan (vec.cu): count of non-finite entries and the smallest flat
// index > after (atomicMin into *minidx, preset by the caller to ~0).
cudaError_t launch_nonfinite_scan(const double* f, long long n, long long after,
                                  unsigned long long* minidx, unsigned long long* count,
                                  cudaStream_t s);

#ifdef __CUDACC__
// All-reduce of 4 doubles over the ranks through peer memory (one thread).
// Every rank adds the same P entries in rank order, so all ranks obtain the
// same bits.  Slot = epoch parity: a rank can only reuse a slot after every
// rank has consumed it (it must first pass the exchange of epoch+1).
__device__ __forceinline__ bool p2p_allreduce4(const P2PArgs& x, unsigned long long epoch,
                                               const double v[4], double out[4]) {
  const int P = x.nranks, me = x.rank, slot = (int)(epoch & 1ull);
  for (int q = 0; q < P; ++q) {
    volatile double* b = x.board[q] + (slot * P2P_MAX + me) * 4;
    b[0] = v[0];
    b[1] = v[1];
    b[2] = v[2];
    b[3] = v[3];
  }
  __threadfence_system();
  for (int q = 0; q < P; ++q) {
    volatile unsigned long long* f = x.flag[q] + slot * P2P_MAX + me;
    *f = epoch;
  }
  volatile unsigned long long* mine = x.flag[me] + slot * P2P_MAX;
  for (int q = 0; q < P; ++q) {
    long long spins = 0;
    while (mine[q] < epoch) {
      __nanosleep(128);
      if (++spins > (1ll << 26)) return false;   // seconds: a peer is gone
    }
  }
  __threadfence_system();
  volatile const double* mb = x.board[me] + slot * P2P_MAX * 4;
  for (int k = 0; k < 4; ++k) out[k] = mb[k];
  for (int q = 1; q < P; ++q)
    for (int k = 0; k < 4; ++k) out[k] = __dadd_rn(out[k], mb[q * 4 + k]);
  return true;
}

// Next FD step and zero-direction flag from ||y|| (linearize.py:62-65).
__device__ __forceinline__ void leja_next_eps(LejaCtl* ctl, double ny) {
  const double kSqrtEps = 1.4901161193847656e-08;  // linearize.py:15
  ctl->zero_dir = (ny == 0.0);
  ctl->eps = __ddiv_rn(__dmul_rn(kSqrtEps, ctl->unorm > 1.0 ? ctl->unorm : 1.0),
                       ny < 1e-300 ? 1e-300 : ny);
  ctl->epsd = make_divisor_dev(ctl->eps);
  if (ctl->force_ieee) ctl->epsd.kind = DIV_IEEE;
}

// Control update after one Newton term (leja.py:134-148); run by one thread
// of the last CTA of the iteration kernel, after the deterministic reduction.
// sy = sum y'^2, sp = sum p'^2 of this term; sp_prev = sum p_{m-1}^2 of the
// pending term a PM_LOOK term resolves first.
__device__ __forceinline__ void leja_finalize(LejaCtl* ctl, double sy, double sp, double sp_prev,
                                              int bad, int counted, double cm,
                                              int dual_next = 0) {
  const int mode = ctl->pmode;
  if (mode == PM_LOOK) {
    // the previous (odd) term's residual (leja.py:141-145), in the reference's order
    const double np_prev = sqrt(sp_prev);
    const double res_prev = __ddiv_rn(__dmul_rn(fabs(ctl->pend_coef), ctl->pend_ynorm),
                                      fmax(1.0, np_prev));
    ctl->residual = res_prev;
    ctl->pnorm = np_prev;
    if (res_prev <= ctl->tol) {
      if (ctl->small_prev) {
        // converged on the odd term: this term never happened (no iteration,
        // no RHS call); the interpolant is pbuf[pcur] + pend_coef * ybuf[cur]
        ctl->m -= 1;
        ctl->status = LJ_CONVERGED;
        return;
      }
      ctl->small_prev = 1;
    } else {
      ctl->small_prev = 0;
    }
  }
  ctl->iters += 1;
  if (counted) ctl->rhs_calls += 1;
  if (bad) {  // mhd.py:225-231 raised inside the matvec
    ctl->fbad = 1;
    ctl->status = LJ_RHS_BAD;
    return;
  }
  const double ny = sqrt(sy);
  if (!isfinite(ny) || ny > ctl->blowup) {
    // the reference returns the interpolant before this term: pbuf[pcur]
    // (+ the pending term, whose y is still ybuf[cur])
    ctl->residual = CUDART_INF;
    ctl->status = LJ_BLOWUP;
    return;
  }
  if (mode == PM_SKIP) {
    // residual unresolved until the next term has ||p_m||
    ctl->cur ^= 1;
    ctl->ppend = 1;
    ctl->pend_coef = cm;
    ctl->pend_ynorm = ny;
    ctl->ynorm = ny;
    ctl->m += 1;   // <= 498
    ctl->pmode = leja_next_pmode(ctl->m, ctl->defer, dual_next, 0, 1);
    if (ctl->m >= ctl->ncoef) ctl->status = LJ_NEED_COEFFS;
    leja_next_eps(ctl, ny);
    return;
  }
  const double np = sqrt(sp);
  const double res = __ddiv_rn(__dmul_rn(fabs(cm), ny), fmax(1.0, np));
  ctl->cur ^= 1;
  if (mode == PM_KEEP) {   // this term kept p' in registers
    ctl->ppend = 1;
    ctl->pend_coef = cm;
  } else {                 // this term stored p'
    ctl->pcur ^= 1;
    ctl->pvirt = 0;        // a virtual interpolant (c0 * v) has now materialised
    ctl->ppend = 0;
  }
  ctl->residual = res;
  ctl->ynorm = ny;
  ctl->pnorm = np;
  if (res <= ctl->tol) {
    if (ctl->small_prev) {
      ctl->status = LJ_CONVERGED;
      return;
    }
    ctl->small_prev = 1;
  } else {
    ctl->small_prev = 0;
  }
  ctl->m += 1;
  if (ctl->m >= 500) {
    ctl->status = LJ_EXHAUSTED;
    return;
  }
  if (ctl->m >= ctl->ncoef) ctl->status = LJ_NEED_COEFFS;
  ctl->pmode = leja_next_pmode(ctl->m, ctl->defer, dual_next, ctl->small_prev, ctl->ppend);
  leja_next_eps(ctl, ny);
}

// Power iteration, after the fused JVP reduced sum((J w)^2) (linearize.py:121-133).
__device__ __forceinline__ void power_after_jvp(PowerCtl* pc, double sum, int bad) {
  pc->rhs_calls += 1;
  if (pc->jvp_only) return;   // non-finite cells are recorded in the caller's flag
  if (bad) {
    pc->status = PW_RHS_BAD;
    return;
  }
  const double mag = sqrt(sum);
  if (mag < 1e-300 || !isfinite(mag)) {
    pc->status = PW_ZERO;
    return;
  }
  const int k = pc->k;
  pc->mags[k] = mag;
  pc->k = k + 1;
  pc->div = mag;
  const double lim = __dmul_rn(pc->tol, mag);
  if ((k + 1 >= 3 && (fabs(__dsub_rn(mag, pc->mags[k - 1])) <= lim ||
                      fabs(__dsub_rn(mag, pc->mags[k - 2])) <= lim)) ||
      k + 1 >= pc->maxit)
    pc->stop = 1;
}

// Power iteration, after w = x / div and its norm (linearize.py:115-116, 124;
// the next jvp's eps, linearize.py:62-65).
__device__ __forceinline__ void power_after_divide(PowerCtl* pc, double sum) {
  const double kSqrtEps = 1.4901161193847656e-08;
  const double wn = sqrt(sum);
  pc->wn = wn;
  if (pc->stop) {
    pc->status = PW_DONE;
    return;
  }
  if (wn == 0.0) {   // jvp of a zero vector is zero (no RHS call): magnitude 0
    pc->status = PW_ZERO;
    return;
  }
  pc->eps = __ddiv_rn(__dmul_rn(kSqrtEps, pc->unorm > 1.0 ? pc->unorm : 1.0),
                      wn < 1e-300 ? 1e-300 : wn);
  pc->epsd = make_divisor_dev(pc->eps);
  if (pc->force_ieee) pc->epsd.kind = DIV_IEEE;
}

// Control-block start from sum(v^2) (leja.py:121-123): y = v, p = c0*v done by the caller.
__device__ __forceinline__ void leja_init_ctl(LejaCtl* ctl, double sumsq) {
  const double kSqrtEps = 1.4901161193847656e-08;
  const double ny = sqrt(sumsq);
  ctl->ynorm = ny;
  ctl->blowup = __dmul_rn(1e120, fmax(1.0, ny));
  ctl->zero_dir = (ny == 0.0);
  ctl->eps = __ddiv_rn(__dmul_rn(kSqrtEps, ctl->unorm > 1.0 ? ctl->unorm : 1.0),
                       ny < 1e-300 ? 1e-300 : ny);
  ctl->epsd = make_divisor_dev(ctl->eps);
  if (ctl->force_ieee) ctl->epsd.kind = DIV_IEEE;
  ctl->m = 1;
  ctl->cur = 0;
  ctl->pcur = 0;
  ctl->ppend = 0;
  ctl->pmode = leja_pmode(1, ctl->defer);
  ctl->iters = 0;
  ctl->rhs_calls = 0;
  ctl->small_prev = 0;
  ctl->fbad = 0;
  ctl->residual = CUDART_INF;
  ctl->status = (ctl->ncoef <= 1) ? LJ_NEED_COEFFS : LJ_RUNNING;
}
#endif

}  // namespace xb
