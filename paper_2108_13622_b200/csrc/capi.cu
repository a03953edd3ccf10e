// C-ABI of the B200 hot path (declared in include/xmhd_b200.h).
//
// Host-side control: context lifetime, scratch ownership, the device-resident
// Leja loop driver (leja.py:103-150) and the scalar glue of jvp
// (linearize.py:56-67).  Python (paper_2108_13622_b200/_lib.py) binds these with
// ctypes; no torch types cross this boundary.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "xmhd_b200.h"

using namespace xb;

struct xmhd_ctx {
  Geom g;
  cudaStream_t stream = 0;
  int device = 0;
  int nsm = 148;
  int units_x = 0, nunits = 0, seg_rows = 0, grid = 0;
  int ws_units_x = 0, ws_nunits = 0, ws_seg_rows = 0, ws_grid = 0;   // warp-specialized plan
  int red_grid = 0;
  double* partials = nullptr;  // [red_grid*8]  (also the stencil's [grid][2])
  unsigned* tickets = nullptr; // [8]
  double* result = nullptr;    // [16]
  int* bad = nullptr;          // [1]
  LejaCtl* ctl = nullptr;
  LejaCtl* ctl_h = nullptr;    // pinned mirror
  double* h_dbl = nullptr;     // pinned [16]
  int* h_int = nullptr;        // pinned [4]
  double* coeffs_d = nullptr;  // [512]
  double* xi_d = nullptr;      // [512]
  double* ybuf[2] = {nullptr, nullptr};
  double* pbuf[2] = {nullptr, nullptr};
  long long ws_n = 0;          // elements per Leja workspace vector
  long long gen_n = 0;         // vector length of the current generic Leja call
  const double* leja_u = nullptr;
  const double* leja_fu = nullptr;
  // in-place start of the host-paced per-term path (xmhd_leja_start_inplace):
  // the call's v is read where it lies, nothing is copied at the start
  const double* leja_v0 = nullptr;   // v of the current in-place call
  // caller-owned interpolant buffers (xmhd_leja_set_pbuf): the result is handed
  // back in one of them (xmhd_leja_result_inplace) instead of being copied out
  double* pbuf_ext[2] = {nullptr, nullptr};
  // y-strips over peer memory (P2PArgs): own region [ghost rows x 2 parities,
  // board, flags], the peers' regions mapped through CUDA IPC
  char* p2p_base = nullptr;
  char* p2p_peer[P2P_MAX] = {};
  P2PArgs p2p;
  bool p2p_ready = false;
  unsigned long long p2p_epoch = 0;   // last exchange epoch (continues across calls)
  StencilArgs* emul_args = nullptr;   // device [P2P_MAX] (one-GPU emulation driver)
  double* coef_h = nullptr;    // pinned [512]: staging of coefficient extensions
  double* kry_d = nullptr;     // [512] MGS coefficient slots (Krylov baseline)
  double* kry_h = nullptr;     // pinned [512]
  PowerCtl* pctl = nullptr;    // device power iteration (allocated on first use)
  PowerCtl* pctl_h = nullptr;  // pinned mirror
  // asynchronous steps (xmhd_async_*): device record + its pinned mirror, the
  // control block of the device-side jvp prologue, phi-actions recorded so far
  AsyncRec* arec = nullptr;
  AsyncRec* arec_h = nullptr;
  PowerCtl* jctl = nullptr;
  int nleja_async = 0;
  int loop_blocks = -1;        // co-resident blocks of the Leja loop kernel (-1: unknown)
  int tile_grid = -1;          // grid of the 2D-tile Leja loop (0: unavailable, -1: unknown)
  int tile_minb = 2;           // its occupancy variant
  bool loop_off = false;       // xmhd_set_loop_kind(2): phi-actions run per-term launches
  int partial_slots = 0;       // doubles in `partials`
  double xi_h[500];            // host copy of the Leja points on the device
  bool xi_valid = false;
  bool leja_defer = true;      // deferred interpolant stores (XMHD_PDEFER=0: off)
  bool leja_adaptive = true;   // variant pairs near the expected end (XMHD_ADAPTIVE=0: off)
  int leja_next_term = 1;      // Newton term index of the next iteration launch
  long long launches = 0;
  // xmhd_term_timing: CUDA-event brackets around the batches of fused-term launches
  int tt_on = 0;
  double tt_ms = 0.0;
  std::vector<cudaEvent_t> tt_free, tt_open;   // idle events; recorded (begin, end) pairs
  int batch_max = 64;
  int hint_iters = 2;          // expected degree of the next fused Leja call (batch sizing)
  int dual_from = 0;           // first term enqueued as a variant pair (0: parity schedule only)
  bool force_ieee = false;
  unsigned long long* scan_d = nullptr;   // [2] non-finite scan (min index, count)
  unsigned long long* scan_h = nullptr;   // pinned [2]
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (expr);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(XMHD_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// How a constant divisor is applied in exact_div (common.cuh).
Divisor make_divisor(double d, bool force_ieee) {
  Divisor v;
  v.d = d;
  v.r = 1.0 / d;  // RN(1/d): host IEEE division
  int ex = 0;
  const double m = std::frexp(d, &ex);
  if (force_ieee) {
    v.kind = DIV_IEEE;
  } else if (m == 0.5 || m == -0.5) {
    v.kind = DIV_MUL;  // power of two: a*r is a/d exactly
  } else {
    const double e = std::fma(-d, v.r, 1.0);  // exact: 1 - d*r
    v.kind = (std::fabs(e) <= std::ldexp(1.0, -54)) ? DIV_MK1 : DIV_MK2;
  }
  return v;
}

RedBuf redbuf(xmhd_ctx* c) {
  RedBuf rb;
  rb.partials = c->partials;
  rb.ticket = c->tickets;
  rb.result = c->result;
  rb.grid = c->red_grid;
  return rb;
}

// Leja workspace: the y ping-pong pair, and the p pair unless the caller
// supplied its own interpolant buffers for this call.
int ensure_ws(xmhd_ctx* c, long long n, bool need_p = true) {
  if (c->ws_n < n) {
    for (int k = 0; k < 2; ++k) {
      if (c->ybuf[k]) cudaFree(c->ybuf[k]);
      if (c->pbuf[k]) cudaFree(c->pbuf[k]);
      c->ybuf[k] = c->pbuf[k] = nullptr;
    }
    c->ws_n = 0;
    for (int k = 0; k < 2; ++k) CK(cudaMalloc(&c->ybuf[k], sizeof(double) * n));
    c->ws_n = n;
  }
  if (need_p && !c->pbuf[0]) {
    for (int k = 0; k < 2; ++k) CK(cudaMalloc(&c->pbuf[k], sizeof(double) * c->ws_n));
  }
  return XMHD_OK;
}

// The interpolant pair of the current call.
inline double* pbuf_of(xmhd_ctx* c, int k) { return c->pbuf_ext[0] ? c->pbuf_ext[k] : c->pbuf[k]; }

// The current direction y of the call (v itself before the first term of an
// in-place call has completed).
inline const double* current_y(xmhd_ctx* c) {
  if (c->leja_v0 && c->ctl_h->m == 1 && c->ctl_h->cur == 0) return c->leja_v0;
  return c->ybuf[c->ctl_h->cur];
}

StencilArgs base_args(xmhd_ctx* c) {
  StencilArgs a;
  std::memset(&a, 0, sizeof(a));
  a.g = c->g;
  a.partials = c->partials;
  a.ticket = c->tickets;
  a.result = c->result;
  a.bad = c->bad;
  a.units_x = c->units_x;
  a.nunits = c->nunits;
  a.seg_rows = c->seg_rows;
  a.ws_units_x = c->ws_units_x;
  a.ws_nunits = c->ws_nunits;
  a.ws_seg_rows = c->ws_seg_rows;
  a.ws_grid = c->ws_grid;
  return a;
}

int fetch_doubles(xmhd_ctx* c, int n) {
  CK(cudaMemcpyAsync(c->h_dbl, c->result, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return XMHD_OK;
}

int fetch_bad(xmhd_ctx* c, int* out) {
  CK(cudaMemcpyAsync(c->h_int, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *out = c->h_int[0];
  return XMHD_OK;
}

// Python's max(a, b) for floats: the first argument unless the second is larger.
inline double py_max(double a, double b) { return (b > a) ? b : a; }

void fill_state(const LejaCtl& h, xmhd_leja_state* st) {
  if (!st) return;
  st->status = h.status;
  st->iterations = h.iters;
  st->rhs_calls = h.rhs_calls;
  st->m = h.m;
  st->residual = h.residual;
  st->eps = h.eps;
  st->ynorm = h.ynorm;
}

// One fused Leja term launch: the kernel variant compiled for the term's
// interpolant mode (single-domain lookahead pairs), else the generic one.
int launch_term(xmhd_ctx* c, const StencilArgs& a, bool peer = false) {
  const int defer = c->ctl_h->defer;
  const int m = c->leja_next_term;
  const int pm = (defer == 2) ? leja_pmode(m, 2) : PM_ANY;
  if (peer) {
    CK(launch_leja_peer(a, c->grid, pm, c->stream));
  } else if (defer == 2 && c->dual_from > 0 && c->ws_grid == 0 && c->g.bcy != BC_HALO) {
    // adaptive lookahead (kernels.h, leja_next_pmode): from term dual_from on, a
    // term is the pair {scheduled variant, PM_STORE}; exactly one of them runs
    StencilArgs b = a;
    b.dual_next = (m + 1 >= c->dual_from) ? 1 : 0;
    if (m >= c->dual_from) {
      b.term = m;
      if (pm != PM_STORE) {
        CK(launch_leja_term(b, c->grid, pm, c->stream));
        c->launches++;
      }
      CK(launch_leja_term(b, c->grid, PM_STORE, c->stream));
    } else {
      CK(launch_leja_term(b, c->grid, pm, c->stream));
    }
  } else {
    CK(launch_leja_term(a, c->grid, pm, c->stream));
  }
  c->leja_next_term++;
  c->launches++;
  return XMHD_OK;
}

// Term timing (xmhd_term_timing): one event before and one after every batch of
// fused-term launches; the pairs are read at the next host synchronisation.
static int tt_mark(xmhd_ctx* c) {
  if (!c->tt_on) return XMHD_OK;
  cudaEvent_t e;
  if (c->tt_free.empty()) {
    CK(cudaEventCreate(&e));
  } else {
    e = c->tt_free.back();
    c->tt_free.pop_back();
  }
  CK(cudaEventRecord(e, c->stream));
  c->tt_open.push_back(e);
  return XMHD_OK;
}

static int tt_harvest(xmhd_ctx* c) {
  for (size_t k = 0; k + 1 < c->tt_open.size(); k += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->tt_open[k], c->tt_open[k + 1]));
    c->tt_ms += (double)ms;
  }
  for (cudaEvent_t e : c->tt_open) c->tt_free.push_back(e);
  c->tt_open.clear();
  return XMHD_OK;
}

int sync_ctl(xmhd_ctx* c) {
  CK(cudaMemcpyAsync(c->ctl_h, c->ctl, sizeof(LejaCtl), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (!c->tt_open.empty()) return tt_harvest(c);
  return XMHD_OK;
}

StencilArgs leja_args(xmhd_ctx* c);

// First term of the variant pairs for a call expected to take `hint` terms: a
// few terms before the expected end (odd, >= 1); the pairs cost one empty
// launch per term, so long calls run the plain parity schedule until then.
inline int dual_start(int hint) {
  const int m0 = hint - 6;
  return m0 < 1 ? 1 : (m0 | 1);
}

// Device-resident fused Leja loop: launch iterations in growing batches; each
// kernel exits immediately once the control block left RUNNING, so the host
// only synchronises once per batch.
int leja_run(xmhd_ctx* c, xmhd_leja_state* st, bool peer = false) {
  StencilArgs a = leja_args(c);
  if (peer) a.p2p = c->p2p;
  // first batch: the caller's degree hint (xmhd_leja_hint; the host keys it by
  // phi order and interval scale), so most calls need a single sync
  const int done = c->ctl_h->iters;
  if (c->ctl_h->m > 0) c->leja_next_term = c->ctl_h->m;   // resume after a stop
  if (!peer && done == 0 && c->leja_adaptive) c->dual_from = dual_start(c->hint_iters);
  int batch = c->hint_iters - done;
  if (batch < 2) batch = 2;
  if (batch > c->batch_max) batch = c->batch_max;
  for (;;) {
    int rc = tt_mark(c);
    if (rc) return rc;
    for (int k = 0; k < batch; ++k) {
      rc = launch_term(c, a, peer);
      if (rc) return rc;
    }
    rc = tt_mark(c);
    if (rc) return rc;
    rc = sync_ctl(c);
    if (rc) return rc;
    c->leja_next_term = c->ctl_h->m;   // kernels launched past a stop exited
    if (c->ctl_h->status != LJ_RUNNING) break;
    batch = batch * 2 < c->batch_max ? batch * 2 : c->batch_max;
  }
  fill_state(*c->ctl_h, st);
  if (peer) {
    c->p2p_epoch = c->ctl_h->epoch;
    if (c->ctl_h->status == LJ_PEER_TIMEOUT)
      return fail(XMHD_CUDA_ERROR, "peer-memory exchange timed out (a rank stopped)");
  }
  return XMHD_OK;
}

int p2p_check_ready(xmhd_ctx* c) {
  if (c->g.bcy != BC_HALO) return fail(XMHD_BADARG, "peer transport needs a y-strip context");
  if (!c->p2p_ready) return fail(XMHD_BADARG, "peer transport not connected");
  if (!c->g.halo_lo) return fail(XMHD_BADARG, "state halo rows not set");
  return XMHD_OK;
}

int upload_coeffs(xmhd_ctx* c, const double* coeffs, int ncoef) {
  if (ncoef < 1 || ncoef > 512) return fail(XMHD_BADARG, "ncoef out of range");
  CK(cudaMemcpyAsync(c->coeffs_d, coeffs, sizeof(double) * ncoef, cudaMemcpyHostToDevice,
                     c->stream));
  return XMHD_OK;
}

int leja_setup(xmhd_ctx* c, const double* v, long long n, double unorm, double dt, double q,
               double theta, double tol, const double* xi, const double* coeffs, int ncoef,
               double* ext_sums = nullptr, bool generic = false, bool single = false,
               bool inplace = false) {
  // caller-owned interpolant buffers and the in-place start belong to the
  // single-domain fused calls with per-term launches (one-role kernel) only
  if (!single) c->pbuf_ext[0] = c->pbuf_ext[1] = nullptr;
  inplace = inplace && single && c->ws_grid == 0;
  c->dual_from = 0;
  int rc = ensure_ws(c, n, !c->pbuf_ext[0]);
  if (rc) return rc;
  c->leja_v0 = inplace ? v : nullptr;
  rc = upload_coeffs(c, coeffs, ncoef);
  if (rc) return rc;
  // the Leja points never change between calls: upload only what differs
  if (!c->xi_valid || std::memcmp(c->xi_h, xi, sizeof(double) * 500) != 0) {
    std::memcpy(c->xi_h, xi, sizeof(double) * 500);
    CK(cudaMemcpyAsync(c->xi_d, xi, sizeof(double) * 500, cudaMemcpyHostToDevice, c->stream));
    c->xi_valid = true;
  }
  LejaCtl h;
  std::memset(&h, 0, sizeof(h));
  h.ncoef = ncoef;
  h.unorm = unorm;
  h.dt = dt;
  h.q = q;
  h.theta = theta;
  h.tol = tol;
  h.thetad = make_divisor(theta, c->force_ieee);
  h.force_ieee = c->force_ieee ? 1 : 0;
  h.epoch = c->p2p_epoch;
  // the generic update stores every term; every fused call (one domain and
  // y-strips alike) uses the lookahead schedule, the strips all-reducing four
  // values per term [sum y'^2, sum p'^2, sum pending p^2, bad]
  h.defer = (!c->leja_defer || generic) ? 0 : 2;
  c->leja_next_term = 1;
  *c->ctl_h = h;
  // staged from pageable memory at the call: back-to-back asynchronous
  // phi-actions never race on the pinned mirror
  CK(cudaMemcpyAsync(c->ctl, &h, sizeof(LejaCtl), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  CK(launch_leja_init(v, n, inplace ? nullptr : c->ybuf[0], inplace ? nullptr : pbuf_of(c, 0),
                      c->ctl, c->coeffs_d, redbuf(c), c->stream, ext_sums));
  c->launches++;
  return XMHD_OK;
}

StencilArgs leja_args(xmhd_ctx* c) {
  StencilArgs a = base_args(c);
  a.u = c->leja_u;
  a.fu = c->leja_fu;
  a.ybuf[0] = c->ybuf[0];
  a.ybuf[1] = c->ybuf[1];
  a.pbuf[0] = pbuf_of(c, 0);
  a.pbuf[1] = pbuf_of(c, 1);
  a.coeffs = c->coeffs_d;
  a.xi = c->xi_d;
  a.ctl = c->ctl;
  a.v0 = c->leja_v0;
  return a;
}

}  // namespace

extern "C" {

const char* xmhd_last_error(void) { return g_err.c_str(); }

int xmhd_create(xmhd_ctx** out, int nx, int ny, double dx, double dy, double mu, double eta,
                double kappa, double gamma, double mu0, int bc_x, int bc_y, void* stream) {
  if (!out) return fail(XMHD_BADARG, "null out");
  if (nx < 2 || ny < 2) return fail(XMHD_BADARG, "grid must be at least 2x2");
  if (bc_x != XMHD_BC_PERIODIC && bc_x != XMHD_BC_REFLECTING)
    return fail(XMHD_BADARG, "bad bc_x");
  if (bc_y < XMHD_BC_PERIODIC || bc_y > XMHD_BC_HALO) return fail(XMHD_BADARG, "bad bc_y");
  // the kernels index a vector with 32-bit unsigned element offsets (34 GB)
  if (8.0 * (double)nx * (double)ny >= 4294967296.0)
    return fail(XMHD_BADARG, "8*nx*ny must stay below 2^32 elements per device (split into "
                             "y-strips over more GPUs)");
  xmhd_ctx* c = new xmhd_ctx();
  const bool ieee = std::getenv("XMHD_DIV_IEEE") && std::atoi(std::getenv("XMHD_DIV_IEEE"));
  c->force_ieee = ieee;
  if (const char* e = std::getenv("XMHD_PDEFER")) c->leja_defer = std::atoi(e) != 0;
  if (const char* e = std::getenv("XMHD_ADAPTIVE")) c->leja_adaptive = std::atoi(e) != 0;
  Geom& g = c->g;
  std::memset(&g, 0, sizeof(g));
  g.nx = nx;
  g.ny = ny;
  g.bcx = bc_x;
  g.bcy = bc_y;
  g.plane = (long long)nx * ny;
  g.diffusive = (mu != 0.0 || eta != 0.0 || kappa != 0.0) ? 1 : 0;
  g.mu0_one = (mu0 == 1.0) ? 1 : 0;
  g.h2x = make_divisor(2.0 * dx, ieee);   // mhd.py:115 folds 2.0*dx on the host
  g.h2y = make_divisor(2.0 * dy, ieee);
  g.mu0d = make_divisor(mu0, ieee);
  g.gm1 = gamma - 1.0;
  g.mu = mu;
  g.eta = eta;
  g.cond = mu * kappa * gamma / (gamma - 1.0);   // mhd.py:197, Python's order
  g.c23 = 2.0 / 3.0;
  c->stream = (cudaStream_t)stream;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(XMHD_CUDA_ERROR, std::string("device query: ") + cudaGetErrorString(e));
  }
  stencil_plan(g, c->nsm, c->units_x, c->nunits, c->seg_rows, c->grid);
  stencil_ws_plan(g, c->nsm, c->ws_units_x, c->ws_nunits, c->ws_seg_rows, c->ws_grid);
  if (const char* seg = std::getenv("XMHD_SEG_ROWS")) {
    // testing knob: another work decomposition = another (equally valid)
    // summation order of the norm partials; used to measure the rounding floor
    const int s = std::atoi(seg);
    if (s > 0 && s < ny) {
      const int slots = c->grid;   // persistent grid of the automatic plan
      c->seg_rows = s;
      c->nunits = c->units_x * ((ny + s - 1) / s);
      c->grid = c->nunits < slots ? c->nunits : slots;
      if (c->ws_grid > 0) {
        c->ws_seg_rows = s;
        c->ws_nunits = c->ws_units_x * ((ny + s - 1) / s);
        c->ws_grid = c->ws_nunits < c->nsm ? c->ws_nunits : c->nsm;
      }
    }
  }
  c->red_grid = 4 * c->nsm;
  const int slots = (c->red_grid > c->grid ? c->red_grid : c->grid) * 8 + 64;
  c->partial_slots = slots;
  if ((e = cudaMalloc(&c->partials, sizeof(double) * slots)) != cudaSuccess ||
      (e = cudaMalloc(&c->tickets, sizeof(unsigned) * 8)) != cudaSuccess ||
      (e = cudaMalloc(&c->result, sizeof(double) * 16)) != cudaSuccess ||
      (e = cudaMalloc(&c->bad, sizeof(int) * 4)) != cudaSuccess ||
      (e = cudaMalloc(&c->ctl, sizeof(LejaCtl))) != cudaSuccess ||
      (e = cudaMalloc(&c->coeffs_d, sizeof(double) * 512)) != cudaSuccess ||
      (e = cudaMalloc(&c->xi_d, sizeof(double) * 512)) != cudaSuccess ||
      (e = cudaMallocHost(&c->ctl_h, sizeof(LejaCtl))) != cudaSuccess ||
      (e = cudaMallocHost(&c->h_dbl, sizeof(double) * 16)) != cudaSuccess ||
      (e = cudaMallocHost(&c->h_int, sizeof(int) * 4)) != cudaSuccess ||
      (e = cudaMallocHost(&c->coef_h, sizeof(double) * 512)) != cudaSuccess ||
      (e = cudaMemsetAsync(c->tickets, 0, sizeof(unsigned) * 8, c->stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(c->bad, 0, sizeof(int) * 4, c->stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(c->stream)) != cudaSuccess) {
    xmhd_destroy(c);
    return fail(XMHD_CUDA_ERROR, std::string("context allocation: ") + cudaGetErrorString(e));
  }
  *out = c;
  return XMHD_OK;
}

int xmhd_destroy(xmhd_ctx* c) {
  if (!c) return XMHD_OK;
  cudaStreamSynchronize(c->stream);
  cudaFree(c->partials);
  cudaFree(c->tickets);
  cudaFree(c->result);
  cudaFree(c->bad);
  cudaFree(c->ctl);
  cudaFree(c->coeffs_d);
  cudaFree(c->xi_d);
  for (int k = 0; k < 2; ++k) {
    cudaFree(c->ybuf[k]);
    cudaFree(c->pbuf[k]);
  }
  for (cudaEvent_t e : c->tt_open) cudaEventDestroy(e);
  for (cudaEvent_t e : c->tt_free) cudaEventDestroy(e);
  cudaFreeHost(c->ctl_h);
  cudaFreeHost(c->h_dbl);
  cudaFreeHost(c->h_int);
  cudaFree(c->kry_d);
  cudaFreeHost(c->kry_h);
  cudaFree(c->pctl);
  cudaFreeHost(c->pctl_h);
  cudaFree(c->arec);
  cudaFreeHost(c->arec_h);
  cudaFree(c->jctl);
  cudaFreeHost(c->coef_h);
  for (int q = 0; q < P2P_MAX; ++q)
    if (c->p2p_peer[q]) cudaIpcCloseMemHandle(c->p2p_peer[q]);
  cudaFree(c->p2p_base);
  cudaFree(c->emul_args);
  delete c;
  return XMHD_OK;
}

int xmhd_set_stream(xmhd_ctx* c, void* stream) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  c->stream = (cudaStream_t)stream;
  return XMHD_OK;
}

int xmhd_plan_info(xmhd_ctx* c, int* out4) {
  if (!c || !out4) return fail(XMHD_BADARG, "null arg");
  const bool ws = c->ws_grid > 0;   // the plan the stencil launches use
  out4[0] = ws ? c->ws_units_x : c->units_x;
  out4[1] = ws ? c->ws_nunits : c->nunits;
  out4[2] = ws ? c->ws_seg_rows : c->seg_rows;
  out4[3] = ws ? c->ws_grid : c->grid;
  return XMHD_OK;
}

long long xmhd_launch_count(xmhd_ctx* c) { return c ? c->launches : -1; }

int xmhd_set_halo(xmhd_ctx* c, const double* lo, const double* hi, const double* lo_dir,
                  const double* hi_dir) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  if (c->g.bcy != BC_HALO) return fail(XMHD_BADARG, "context is not a y-strip (bc_y != HALO)");
  c->g.halo_lo = lo;
  c->g.halo_hi = hi;
  c->g.halo_lo_dir = lo_dir;
  c->g.halo_hi_dir = hi_dir;
  return XMHD_OK;
}

// RhsBlowupError.cells of mhd.py:225-231 from a device RHS output: out[0] =
// number of non-finite entries, then up to 8 (field, i, j) triples in C order
// (flat index order of the (8, ny, nx) layout); unused triples are -1.
static int scan_bad_cells(xmhd_ctx* c, const double* f, int* out) {
  if (!out) return XMHD_OK;
  for (int k = 0; k < XMHD_BAD_CELLS_LEN; ++k) out[k] = -1;
  if (!c->scan_d) {
    CK(cudaMalloc(&c->scan_d, 2 * sizeof(unsigned long long)));
    CK(cudaMallocHost(&c->scan_h, 2 * sizeof(unsigned long long)));
  }
  const long long n = NF * c->g.plane;
  long long after = -1;
  for (int k = 0; k < 8; ++k) {
    CK(cudaMemsetAsync(c->scan_d, 0xff, sizeof(unsigned long long), c->stream));
    if (k == 0) CK(cudaMemsetAsync(c->scan_d + 1, 0, sizeof(unsigned long long), c->stream));
    CK(launch_nonfinite_scan(f, n, after, c->scan_d, k == 0 ? c->scan_d + 1 : nullptr,
                             c->stream));
    c->launches++;
    CK(cudaMemcpyAsync(c->scan_h, c->scan_d, 2 * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (k == 0) out[0] = c->scan_h[1] > 0x7fffffffull ? 0x7fffffff : (int)c->scan_h[1];
    const unsigned long long idx = c->scan_h[0];
    if (idx == ~0ull) break;
    const long long plane = c->g.plane;
    const long long field = (long long)idx / plane, rem = (long long)idx - field * plane;
    out[1 + 3 * k] = (int)field;
    out[2 + 3 * k] = (int)(rem % c->g.nx);
    out[3 + 3 * k] = (int)(rem / c->g.nx);
    after = (long long)idx;
  }
  return XMHD_OK;
}

// F(u + eps*w) into scratch and its non-finite cells (the JVP / Leja failure
// path: the reference raises from mhd_rhs of that state, linearize.py:67).
static int scan_bad_cells_shifted(xmhd_ctx* c, const double* u, const double* w, double eps,
                                  int* out) {
  if (!out) return XMHD_OK;
  const long long n = NF * c->g.plane;
  double* x = nullptr;
  double* fx = nullptr;
  CK(cudaMallocAsync(&x, 2 * sizeof(double) * n, c->stream));
  fx = x + n;
  const double* v[2] = {u, w};
  const double cf[2] = {1.0, eps};
  int rc = XMHD_OK;
  if (launch_lincomb(x, n, v, cf, 2, 0, redbuf(c), c->stream) != cudaSuccess) {
    rc = fail(XMHD_CUDA_ERROR, "lincomb launch failed");
  } else {
    StencilArgs a = base_args(c);
    a.u = x;
    a.out = fx;
    if (launch_stencil(MODE_RHS, a, c->grid, c->stream) != cudaSuccess)
      rc = fail(XMHD_CUDA_ERROR, "rhs launch failed");
    else
      rc = scan_bad_cells(c, fx, out);
    c->launches += 2;
  }
  cudaFreeAsync(x, c->stream);
  return rc;
}

int xmhd_rhs(xmhd_ctx* c, const double* u, double* f, int* bad_cells) {
  if (!c || !u || !f) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO && !c->g.halo_lo) return fail(XMHD_BADARG, "halo rows not set");
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.out = f;
  CK(launch_stencil(MODE_RHS, a, c->grid, c->stream));
  c->launches++;
  int bad = 0;
  int rc = fetch_bad(c, &bad);
  if (rc) return rc;
  if (!bad) return XMHD_OK;
  rc = scan_bad_cells(c, f, bad_cells);
  return rc ? rc : XMHD_NONFINITE;
}

// jvp (linearize.py:56-67); wn_known >= 0: ||w|| already reduced by the caller
// (bit for bit the norm kernel's); stage_f != null: the fused tail of a stage
// difference, out = (stage_f - fu) - J w (integrators.py:146-153).
static int jvp_impl(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                    const double* w, double wn_known, const double* stage_f, double* out,
                    int* called, double* out_norm, int* bad_cells) {
  const long long n = NF * c->g.plane;
  double wn = wn_known;
  int rc;
  if (wn < 0.0) {
    CK(launch_norm(w, n, redbuf(c), c->stream));
    c->launches++;
    rc = fetch_doubles(c, 1);
    if (rc) return rc;
    wn = c->h_dbl[0];
  }
  if (called) *called = 0;
  // (stage_f - fu) - out, in place, for the paths whose kernel wrote J w (or zeros)
  auto tail = [&]() -> int {
    const double* v[3] = {stage_f, fu, out};
    const double cf[3] = {1.0, -1.0, -1.0};
    CK(launch_lincomb(out, n, v, cf, 3, 0, redbuf(c), c->stream));
    c->launches++;
    return XMHD_OK;
  };
  if (wn == 0.0) {  // linearize.py:63-64: zero vector, no RHS evaluation
    CK(cudaMemsetAsync(out, 0, sizeof(double) * n, c->stream));
    if (out_norm) *out_norm = 0.0;
    return stage_f ? tail() : XMHD_OK;
  }
  // linearize.py:65: eps = _SQRT_EPS * max(1.0, ||u||) / max(||w||, 1e-300)
  const double eps = (1.4901161193847656e-08 * py_max(1.0, unorm)) / py_max(wn, 1e-300);
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.dir = w;
  a.fu = fu;
  a.out = out;
  a.eps = eps;
  a.epsd = make_divisor(eps, c->force_ieee);
  const bool fused_tail = stage_f && c->ws_grid == 0;   // the one-role kernel's epilogue
  a.stage_f = fused_tail ? stage_f : nullptr;
  CK(launch_stencil(MODE_JVP, a, c->grid, c->stream));
  c->launches++;
  if (called) *called = 1;
  if (stage_f && !fused_tail) {
    rc = tail();
    if (rc) return rc;
  }
  rc = fetch_doubles(c, 1);
  if (rc) return rc;
  if (out_norm) *out_norm = c->h_dbl[0];
  int bad = 0;
  rc = fetch_bad(c, &bad);
  if (rc) return rc;
  if (!bad) return XMHD_OK;
  if (c->g.bcy != BC_HALO) {
    rc = scan_bad_cells_shifted(c, u, w, eps, bad_cells);
    if (rc) return rc;
  }
  return XMHD_NONFINITE;
}

int xmhd_jvp(xmhd_ctx* c, const double* u, const double* fu, double unorm, const double* w,
             double* out, int* called, double* out_norm, int* bad_cells) {
  if (!c || !u || !fu || !w || !out) return fail(XMHD_BADARG, "null arg");
  return jvp_impl(c, u, fu, unorm, w, -1.0, nullptr, out, called, out_norm, bad_cells);
}

int xmhd_stage_difference(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                          const double* d, double dnorm, const double* fstage, double* out,
                          int* called, int* bad_cells) {
  if (!c || !u || !fu || !d || !fstage || !out) return fail(XMHD_BADARG, "null arg");
  if (!(dnorm >= 0.0)) return fail(XMHD_BADARG, "dnorm must be the norm of d");
  return jvp_impl(c, u, fu, unorm, d, dnorm, fstage, out, called, nullptr, bad_cells);
}

// Device-resident power iteration of estimate_alpha (linearize.py:113-135).
// Per iteration one fused JVP (MODE_JVP reading its FD step from the control
// block, last block: ||J w||, magnitude list, stopping test) and one division
// (w = J w / mag, ||w||, next FD step); the host enqueues batches of
// iterations and reads the 1 KB control block once per batch.
int xmhd_power(xmhd_ctx* c, const double* u, const double* fu, double unorm, const double* w0,
               double* w, double* work, int maxit, double tol, double* mags, int* nit,
               int* rhs_calls, int* status) {
  if (!c || !u || !fu || !w0 || !w || !work || !mags || !nit || !rhs_calls || !status)
    return fail(XMHD_BADARG, "null arg");
  if (maxit < 1 || maxit > POWER_MAXIT) return fail(XMHD_BADARG, "maxit out of range");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "y-strip contexts use the host power loop");
  if (!c->pctl) {
    CK(cudaMalloc(&c->pctl, sizeof(PowerCtl)));
    CK(cudaMallocHost(&c->pctl_h, sizeof(PowerCtl)));
  }
  const long long n = NF * c->g.plane;
  // w = w0 / ||w0||, a vector of ones when w0 == 0 (linearize.py:114-117)
  CK(launch_norm(w0, n, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  double wn0 = c->h_dbl[0];
  if (wn0 == 0.0) {
    CK(launch_fill(work, n, 1.0, c->stream));
    CK(launch_norm(work, n, redbuf(c), c->stream));
    c->launches += 2;
    rc = fetch_doubles(c, 1);
    if (rc) return rc;
    wn0 = c->h_dbl[0];
  } else {
    CK(cudaMemcpyAsync(work, w0, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  }
  PowerCtl* h = c->pctl_h;
  std::memset(h, 0, sizeof(PowerCtl));
  h->status = PW_RUNNING;
  h->maxit = maxit;
  h->tol = tol;
  h->unorm = unorm;
  h->div = wn0;
  h->force_ieee = c->force_ieee ? 1 : 0;
  CK(cudaMemcpyAsync(c->pctl, h, sizeof(PowerCtl), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  CK(launch_power_divide(w, work, n, c->pctl, redbuf(c), c->stream));
  c->launches++;
  StencilArgs a = base_args(c);
  a.u = u;
  a.fu = fu;
  a.dir = w;
  a.out = work;
  a.pctl = c->pctl;
  int launched = 0, batch = 6;   // typical refreshes stop after 4-7 iterations
  for (;;) {
    for (int b = 0; b < batch && launched < maxit; ++b, ++launched) {
      CK(launch_stencil(MODE_JVP, a, c->grid, c->stream));
      CK(launch_power_divide(w, work, n, c->pctl, redbuf(c), c->stream));
      c->launches += 2;
    }
    CK(cudaMemcpyAsync(h, c->pctl, sizeof(PowerCtl), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h->status != PW_RUNNING || launched >= maxit) break;
    batch = 8;
  }
  if (h->status == PW_RUNNING) return fail(XMHD_CUDA_ERROR, "power iteration left RUNNING");
  *nit = h->k;
  *rhs_calls = h->rhs_calls;
  for (int k = 0; k < h->k; ++k) mags[k] = h->mags[k];
  *status = h->status == PW_DONE ? 0 : 1;
  return h->status == PW_RHS_BAD ? XMHD_NONFINITE : XMHD_OK;
}

// FrozenLinearization (linearize.py:46-53) in one host round trip:
// fu = F(u) and ||u|| enqueued back to back, then one read of both.
int xmhd_linearize(xmhd_ctx* c, const double* u, double* fu, double* unorm) {
  if (!c || !u || !fu || !unorm) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "y-strips reduce ||u|| across ranks");
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.out = fu;
  CK(launch_stencil(MODE_RHS, a, c->grid, c->stream));
  CK(launch_norm(u, NF * c->g.plane, redbuf(c), c->stream));
  c->launches += 2;
  CK(cudaMemcpyAsync(c->h_int, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_dbl, c->result, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *unorm = c->h_dbl[0];
  return c->h_int[0] ? XMHD_NONFINITE : XMHD_OK;
}

// FrozenLinearization without a host wait, ||u|| known to the caller: fu = F(u)
// with its non-finite flag in a slot of its own (bad[1]), read by
// xmhd_linearize_check or with the next step record.
int xmhd_linearize_async(xmhd_ctx* c, const double* u, double* fu) {
  if (!c || !u || !fu) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "single-domain contexts only");
  CK(cudaMemsetAsync(c->bad + 1, 0, sizeof(int), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.out = fu;
  a.bad = c->bad + 1;
  CK(launch_stencil(MODE_RHS, a, c->grid, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_linearize_check(xmhd_ctx* c, int* nonfinite) {
  if (!c || !nonfinite) return fail(XMHD_BADARG, "null arg");
  CK(cudaMemcpyAsync(c->h_int + 1, c->bad + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *nonfinite = c->h_int[1];
  return XMHD_OK;
}

// max |div B| of u into a device double (no host wait; harness.py:209-211).
int xmhd_divb_async(xmhd_ctx* c, const double* u, double* out_dev) {
  if (!c || !u || !out_dev) return fail(XMHD_BADARG, "null arg");
  RedBuf rb = redbuf(c);
  rb.result = out_dev;
  CK(launch_divb_max(c->g, u, nullptr, rb, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_norm(xmhd_ctx* c, const double* x, long long n, double* out) {
  if (!c || !x || !out) return fail(XMHD_BADARG, "null arg");
  CK(launch_norm(x, n, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  *out = c->h_dbl[0];
  return XMHD_OK;
}

int xmhd_lincomb(xmhd_ctx* c, double* out, long long n, const double* const* v, const double* cf,
                 int nterms, double* norm_out, int* nonfinite_out) {
  if (!c || !out || !v || !cf || nterms < 1 || nterms > 4) return fail(XMHD_BADARG, "bad lincomb");
  const int want = (norm_out || nonfinite_out) ? 1 : 0;
  CK(launch_lincomb(out, n, v, cf, nterms, want, redbuf(c), c->stream));
  c->launches++;
  if (!want) return XMHD_OK;
  int rc = fetch_doubles(c, 2);
  if (rc) return rc;
  if (norm_out) *norm_out = c->h_dbl[0];
  if (nonfinite_out) *nonfinite_out = c->h_dbl[1] != 0.0;
  return XMHD_OK;
}

int xmhd_lincomb_diff(xmhd_ctx* c, double* out, double* diff, long long n,
                      const double* const* v, const double* cf, int nterms, double* diff_norm) {
  if (!c || !out || !diff || !v || !cf || !diff_norm || nterms < 2 || nterms > 4)
    return fail(XMHD_BADARG, "bad lincomb_diff args");
  CK(launch_lincomb_diff(out, diff, n, v, cf, nterms, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  *diff_norm = c->h_dbl[0];
  return XMHD_OK;
}

int xmhd_lincomb_multi(xmhd_ctx* c, double* const* out, int nout, long long n,
                       const double* const* v, const double* coef) {
  if (!c || !out || !v || !coef || nout < 2 || nout > 4)
    return fail(XMHD_BADARG, "bad lincomb_multi args");
  for (int j = 0; j < nout; ++j) {
    if (!out[j]) return fail(XMHD_BADARG, "null output");
    if (coef[3 * j] == 0.0 && coef[3 * j + 1] == 0.0 && coef[3 * j + 2] == 0.0)
      return fail(XMHD_BADARG, "a combination needs a non-zero coefficient");
  }
  for (int k = 0; k < 3; ++k)
    if (!v[k]) return fail(XMHD_BADARG, "null input");
  CK(launch_lincomb_multi(out, nout, n, v, coef, redbuf(c), c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_divide(xmhd_ctx* c, double* out, const double* x, double d, long long n,
                double* norm_out) {
  if (!c || !out || !x) return fail(XMHD_BADARG, "null arg");
  CK(launch_divide(out, x, d, n, norm_out ? 1 : 0, redbuf(c), c->stream));
  c->launches++;
  if (!norm_out) return XMHD_OK;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  *norm_out = c->h_dbl[0];
  return XMHD_OK;
}

int xmhd_diff_norms(xmhd_ctx* c, const double* a, const double* b, long long n, double* out) {
  if (!c || !a || !b || !out) return fail(XMHD_BADARG, "null arg");
  CK(launch_diffnorm(a, b, n, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 2);
  if (rc) return rc;
  out[0] = c->h_dbl[0];
  out[1] = c->h_dbl[1];
  return XMHD_OK;
}

int xmhd_final_pair(xmhd_ctx* c, int scheme, double* out_hi, long long n,
                    const double* const* v, const double* cf, double* err_out,
                    int* nonfinite) {
  if (!c || !out_hi || !v || !cf || !err_out || !nonfinite) return fail(XMHD_BADARG, "null arg");
  const int kind = scheme == XMHD_SCHEME_EXPRB43 ? 43 : (scheme == XMHD_SCHEME_EXPRB54S4 ? 54 : 0);
  if (!kind) return fail(XMHD_BADARG, "scheme must be EXPRB43 or EXPRB54s4");
  for (int k = 0; k < (kind == 43 ? 4 : 6); ++k)
    if (!v[k]) return fail(XMHD_BADARG, "null input vector");
  CK(launch_final_pair(kind, out_hi, n, v, cf, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 3);
  if (rc) return rc;
  err_out[0] = c->h_dbl[0];
  err_out[1] = c->h_dbl[1];
  *nonfinite = c->h_dbl[2] > 0.0 ? 1 : 0;
  return XMHD_OK;
}

int xmhd_divb(xmhd_ctx* c, const double* u, double* field, double* out) {
  if (!c || !u || !out) return fail(XMHD_BADARG, "null arg");
  CK(launch_divb_max(c->g, u, field, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  *out = c->h_dbl[0];
  return XMHD_OK;
}

int xmhd_field_sums(xmhd_ctx* c, const double* u, double* out8) {
  if (!c || !u || !out8) return fail(XMHD_BADARG, "null arg");
  CK(launch_field_sums(u, c->g.plane, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 8);
  if (rc) return rc;
  for (int k = 0; k < 8; ++k) out8[k] = c->h_dbl[k];
  return XMHD_OK;
}

int xmhd_cfl_speeds(xmhd_ctx* c, const double* u, double* out2) {
  if (!c || !u || !out2) return fail(XMHD_BADARG, "null arg");
  const double gamma = c->g.gm1 + 1.0;
  CK(launch_cfl(u, c->g.plane, gamma, c->g.mu0d.d, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 2);
  if (rc) return rc;
  out2[0] = c->h_dbl[0];
  out2[1] = c->h_dbl[1];
  return XMHD_OK;
}

int xmhd_leja_start(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                    const double* v, double dt, double q, double theta, double tol,
                    const double* xi, const double* coeffs, int ncoef, xmhd_leja_state* st) {
  if (!c || !u || !fu || !v || !xi || !coeffs) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "use the strip driver for BC_HALO");
  const long long n = NF * c->g.plane;
  c->leja_u = u;
  c->leja_fu = fu;
  int rc = leja_setup(c, v, n, unorm, dt, q, theta, tol, xi, coeffs, ncoef, nullptr, false, true,
                      true);
  if (rc) return rc;
  return leja_run(c, st);
}

int xmhd_leja_start_async(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                          const double* v, double dt, double q, double theta, double tol,
                          const double* xi, const double* coeffs, int ncoef) {
  if (!c || !u || !fu || !v || !xi || !coeffs) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "use the strip driver for BC_HALO");
  c->leja_u = u;
  c->leja_fu = fu;
  return leja_setup(c, v, NF * c->g.plane, unorm, dt, q, theta, tol, xi, coeffs, ncoef, nullptr,
                    false, true, false);
}

int xmhd_leja_start_inplace(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                            const double* v, double dt, double q, double theta, double tol,
                            const double* xi, const double* coeffs, int ncoef) {
  if (!c || !u || !fu || !v || !xi || !coeffs) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "use the strip driver for BC_HALO");
  c->leja_u = u;
  c->leja_fu = fu;
  return leja_setup(c, v, NF * c->g.plane, unorm, dt, q, theta, tol, xi, coeffs, ncoef, nullptr,
                    false, true, true);
}

int xmhd_leja_resume(xmhd_ctx* c, const double* coeffs, int ncoef, xmhd_leja_state* st) {
  if (!c || !coeffs) return fail(XMHD_BADARG, "null arg");
  int rc = upload_coeffs(c, coeffs, ncoef);
  if (rc) return rc;
  c->ctl_h->ncoef = ncoef;
  c->ctl_h->status = LJ_RUNNING;
  CK(cudaMemcpyAsync(&c->ctl->ncoef, &c->ctl_h->ncoef, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->ctl->status, &c->ctl_h->status, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  return leja_run(c, st);
}

// Host-paced driver primitives: enqueue iteration kernels without waiting,
// extend the device coefficient table ahead of the terms that need it, sync.
int xmhd_leja_launch(xmhd_ctx* c, int n, int peer) {
  if (!c || n < 0 || n > 500) return fail(XMHD_BADARG, "bad launch count");
  if (peer) {
    int rc = p2p_check_ready(c);
    if (rc) return rc;
  }
  StencilArgs a = leja_args(c);
  if (peer) a.p2p = c->p2p;
  int rc = n > 0 ? tt_mark(c) : XMHD_OK;
  if (rc) return rc;
  for (int k = 0; k < n; ++k) {
    rc = launch_term(c, a, peer != 0);
    if (rc) return rc;
  }
  return n > 0 ? tt_mark(c) : XMHD_OK;
}

int xmhd_term_timing(xmhd_ctx* c, int enable, double* total_ms) {
  if (!c) return fail(XMHD_BADARG, "null arg");
  if (enable >= 0) {
    CK(cudaStreamSynchronize(c->stream));
    int rc = tt_harvest(c);
    if (rc) return rc;
    if (total_ms) *total_ms = c->tt_ms;
    c->tt_on = enable ? 1 : 0;
    c->tt_ms = 0.0;
    return XMHD_OK;
  }
  if (total_ms) *total_ms = c->tt_ms;
  return XMHD_OK;
}

int xmhd_leja_extend(xmhd_ctx* c, const double* coeffs, int from, int to) {
  if (!c || !coeffs || from < 1 || to <= from || to > 500)
    return fail(XMHD_BADARG, "bad coefficient extension");
  // the staging ranges of one call's extensions are disjoint, so an earlier
  // extension's copy still in flight is never overwritten
  std::memcpy(c->coef_h + from, coeffs + from, sizeof(double) * (to - from));
  CK(cudaMemcpyAsync(c->coeffs_d + from, c->coef_h + from, sizeof(double) * (to - from),
                     cudaMemcpyHostToDevice, c->stream));
  CK(launch_leja_extend(c->ctl, to, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_sync(xmhd_ctx* c, xmhd_leja_state* st) {
  if (!c || !st) return fail(XMHD_BADARG, "null arg");
  int rc = sync_ctl(c);
  if (rc) return rc;
  fill_state(*c->ctl_h, st);
  if (c->ctl_h->status == LJ_MODE_ERROR)
    return fail(XMHD_CUDA_ERROR, "Leja kernel variant / interpolant mode mismatch");
  if (c->ctl_h->status == LJ_RUNNING || c->ctl_h->status == LJ_NEED_COEFFS)
    c->leja_next_term = c->ctl_h->m;
  c->p2p_epoch = c->ctl_h->epoch;
  if (c->ctl_h->status == LJ_PEER_TIMEOUT)
    return fail(XMHD_CUDA_ERROR, "peer-memory exchange timed out (a rank stopped)");
  return XMHD_OK;
}

// ---- asynchronous single-domain steps ------------------------------------
// The whole Leja loop as one cooperative launch; no host read until the
// caller synchronises (xmhd_leja_sync, or xmhd_async_fetch at a step end).
// Which loop kernel: the 2D-tile loop (default) or the sliding-window loop
// (XMHD_TILE=0, A/B and tests).
static void loop_plan(xmhd_ctx* c) {
  if (c->tile_grid < 0) {
    const char* e = std::getenv("XMHD_TILE");
    const bool tile = !(e && std::atoi(e) == 0);
    c->tile_grid = tile ? leja_tile_loop_grid(c->g, c->nsm, &c->tile_minb) : 0;
    if (c->tile_grid * 8 > c->partial_slots) c->tile_grid = 0;
  }
  if (c->loop_blocks < 0) c->loop_blocks = leja_loop_max_blocks(c->nsm);
}

int xmhd_leja_loop(xmhd_ctx* c) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "y-strips use the strip drivers");
  if (c->leja_v0)
    return fail(XMHD_BADARG, "a call started in place runs per-term launches (xmhd_leja_launch)");
  loop_plan(c);
  StencilArgs a = leja_args(c);
  if (c->tile_grid > 0) {
    CK(launch_leja_tile_loop(a, c->tile_grid, c->tile_minb, c->stream));
  } else {
    if (c->grid > c->loop_blocks)
      return fail(XMHD_BADARG, "grid not co-resident: use xmhd_leja_launch batches");
    CK(launch_leja_loop(a, c->grid, c->stream));
  }
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_set_pbuf(xmhd_ctx* c, double* p0, double* p1) {
  if (!c || (p0 == nullptr) != (p1 == nullptr) || (p0 && p0 == p1))
    return fail(XMHD_BADARG, "pass two distinct buffers, or two nulls");
  c->pbuf_ext[0] = p0;
  c->pbuf_ext[1] = p1;
  return XMHD_OK;
}

int xmhd_leja_result_inplace(xmhd_ctx* c, int* which) {
  if (!c || !which) return fail(XMHD_BADARG, "null arg");
  if (!c->pbuf_ext[0]) return fail(XMHD_BADARG, "no caller-owned interpolant buffers set");
  int rc = sync_ctl(c);
  if (rc) return rc;
  const LejaCtl& h = *c->ctl_h;
  if (!h.ppend && !h.pvirt) {   // the last stored interpolant is the result
    *which = h.pcur;
    return XMHD_OK;
  }
  // p + c*y (or c0*v) into the buffer the call is not reading
  const int dst = h.pcur ^ 1;
  const long long n = NF * c->g.plane;
  const double* pb[2] = {c->pbuf_ext[0], c->pbuf_ext[1]};
  CK(launch_leja_copy_result(c->pbuf_ext[dst], pb, c->ybuf, c->leja_v0, c->ctl, n, c->stream));
  c->launches++;
  *which = dst;
  return XMHD_OK;
}

int xmhd_leja_set_dual_from(xmhd_ctx* c, int m0) {
  if (!c || m0 < 0) return fail(XMHD_BADARG, "bad term index");
  c->dual_from = (c->leja_adaptive && m0 > 0) ? (m0 | 1) : 0;
  return XMHD_OK;
}

int xmhd_set_leja_defer(xmhd_ctx* c, int on) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  c->leja_defer = on != 0;
  return XMHD_OK;
}

int xmhd_set_loop_kind(xmhd_ctx* c, int kind) {
  if (!c || kind < 0 || kind > 2) return fail(XMHD_BADARG, "bad loop kind");
  c->tile_grid = -1;
  if (kind == 1) c->tile_grid = 0;   // sliding-window loop
  c->loop_off = (kind == 2);         // no cooperative loop: per-term launches
  return XMHD_OK;
}

int xmhd_leja_loop_available(xmhd_ctx* c) {
  if (!c || c->g.bcy == BC_HALO || c->loop_off) return 0;
  loop_plan(c);
  return (c->tile_grid > 0 || c->grid <= c->loop_blocks) ? 1 : 0;
}

static int ensure_async(xmhd_ctx* c) {
  if (c->arec) return XMHD_OK;
  CK(cudaMalloc(&c->arec, sizeof(AsyncRec)));
  CK(cudaMallocHost(&c->arec_h, sizeof(AsyncRec)));
  CK(cudaMalloc(&c->jctl, sizeof(PowerCtl)));
  return XMHD_OK;
}

int xmhd_async_begin(xmhd_ctx* c) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  int rc = ensure_async(c);
  if (rc) return rc;
  CK(cudaMemsetAsync(c->arec, 0, sizeof(AsyncRec), c->stream));
  PowerCtl j;
  std::memset(&j, 0, sizeof(j));
  j.status = PW_RUNNING;
  j.jvp_only = 1;
  j.force_ieee = c->force_ieee ? 1 : 0;
  CK(cudaMemcpyAsync(c->jctl, &j, sizeof(PowerCtl), cudaMemcpyHostToDevice, c->stream));
  c->nleja_async = 0;
  return XMHD_OK;
}

int xmhd_rhs_async(xmhd_ctx* c, const double* u, double* f) {
  if (!c || !u || !f || !c->arec) return fail(XMHD_BADARG, "null arg or no xmhd_async_begin");
  StencilArgs a = base_args(c);
  a.u = u;
  a.out = f;
  a.bad = &c->arec->bad;
  CK(launch_stencil(MODE_RHS, a, c->grid, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_jvp_async(xmhd_ctx* c, const double* u, const double* fu, double unorm, const double* w,
                   double* out) {
  if (!c || !u || !fu || !w || !out || !c->arec)
    return fail(XMHD_BADARG, "null arg or no xmhd_async_begin");
  const long long n = NF * c->g.plane;
  CK(cudaMemsetAsync(out, 0, sizeof(double) * n, c->stream));   // zero w -> zero J w
  CK(launch_jvp_prep(w, n, unorm, c->jctl, redbuf(c), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.dir = w;
  a.fu = fu;
  a.out = out;
  a.pctl = c->jctl;
  a.bad = &c->arec->bad;
  CK(launch_stencil(MODE_JVP, a, c->grid, c->stream));
  c->launches += 2;
  return XMHD_OK;
}

int xmhd_leja_finish_async(xmhd_ctx* c, double* p_out) {
  if (!c || !p_out || !c->arec) return fail(XMHD_BADARG, "null arg or no xmhd_async_begin");
  if (c->nleja_async >= ASYNC_LEJA_MAX) return fail(XMHD_BADARG, "too many phi-actions in one step");
  const long long n = NF * c->g.plane;
  {
    const double* pb[2] = {pbuf_of(c, 0), pbuf_of(c, 1)};
    CK(launch_leja_copy_result(p_out, pb, c->ybuf, c->leja_v0, c->ctl, n, c->stream));
  }
  CK(cudaMemcpyAsync(&c->arec->leja[c->nleja_async], c->ctl, sizeof(LejaCtl),
                     cudaMemcpyDeviceToDevice, c->stream));
  c->nleja_async++;
  c->launches++;
  return XMHD_OK;
}

int xmhd_lincomb_async(xmhd_ctx* c, double* out, long long n, const double* const* v,
                       const double* cf, int nterms) {
  if (!c || !out || !v || !cf || nterms < 1 || nterms > 4 || !c->arec)
    return fail(XMHD_BADARG, "bad lincomb");
  RedBuf rb = redbuf(c);
  rb.result = c->arec->lc;
  CK(launch_lincomb(out, n, v, cf, nterms, 1, rb, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_diff_norms_async(xmhd_ctx* c, const double* a, const double* b, long long n) {
  if (!c || !a || !b || !c->arec) return fail(XMHD_BADARG, "null arg or no xmhd_async_begin");
  RedBuf rb = redbuf(c);
  rb.result = c->arec->err;
  CK(launch_diffnorm(a, b, n, rb, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_async_fetch(xmhd_ctx* c, xmhd_step_record* out) {
  if (!c || !out || !c->arec) return fail(XMHD_BADARG, "null arg or no xmhd_async_begin");
  CK(cudaMemcpyAsync(&c->arec->jvp_calls, &c->jctl->rhs_calls, sizeof(int),
                     cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->arec->pad_[0], c->bad + 1, sizeof(int), cudaMemcpyDeviceToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(c->arec_h, c->arec, sizeof(AsyncRec), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const AsyncRec& r = *c->arec_h;
  std::memset(out, 0, sizeof(*out));
  out->rhs_nonfinite = r.bad;
  out->lin_nonfinite = r.pad_[0];
  out->jvp_calls = r.jvp_calls;
  out->nleja = c->nleja_async;
  out->err_diff = r.err[0];
  out->err_ref = r.err[1];
  out->lc_norm = r.lc[0];
  out->lc_nonfinite = r.lc[1];
  for (int k = 0; k < c->nleja_async; ++k) fill_state(r.leja[k], &out->leja[k]);
  *c->ctl_h = r.leja[c->nleja_async ? c->nleja_async - 1 : 0];
  return XMHD_OK;
}

int xmhd_leja_hint(xmhd_ctx* c, int expected_iterations) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  c->hint_iters = expected_iterations < 2 ? 2 : expected_iterations;
  return XMHD_OK;
}

int xmhd_leja_result(xmhd_ctx* c, double* p_out) {
  if (!c || !p_out) return fail(XMHD_BADARG, "null arg");
  int rc = sync_ctl(c);
  if (rc) return rc;
  const long long n = c->gen_n ? c->gen_n : NF * c->g.plane;
  {
    const double* pb[2] = {pbuf_of(c, 0), pbuf_of(c, 1)};
    CK(launch_leja_copy_result(p_out, pb, c->ybuf, c->leja_v0, c->ctl, n, c->stream));
  }
  c->launches++;
  return XMHD_OK;
}

// apply_phi_leja (leja.py:103-150) in ONE call: the whole Newton loop runs
// on the device (one cooperative launch on small grids, host-paced batches of
// fused iteration kernels otherwise) against a coefficient table that already
// holds every entry the call may index, built with the reference's chunk
// schedule (xmhd_leja_schedule: entries [0,64) of the 64-chunk, [64,128) of
// the 128-chunk, ... as leja.py:119-130 fetches them for an uncached
// (l, q, theta)).  A table shorter than the degree the call reaches is an
// error (XMHD_BADARG), never a silent truncation.
int xmhd_leja(xmhd_ctx* c, int l, const double* u, const double* fu, double unorm,
              const double* v, double dt, double q, double theta, double tol,
              const double* xi, const double* coeffs, int ncoef, double* p_out,
              int* iterations, int* converged, double* residual, int* rhs_calls,
              int* bad_cells) {
  if (!c || !u || !fu || !v || !xi || !coeffs || !p_out)
    return fail(XMHD_BADARG, "null arg");
  if (l < 0 || l > 4) return fail(XMHD_BADARG, "phi order must be an integer in [0, 4]");
  if (!(tol > 0.0)) return fail(XMHD_BADARG, "tolerance must be positive");
  if (!(theta > 0.0)) return fail(XMHD_BADARG, "spectral magnitude must be positive");
  if (ncoef < 2 || ncoef > 500) return fail(XMHD_BADARG, "ncoef must lie in [2, 500]");
  if (c->g.bcy == BC_HALO) return fail(XMHD_BADARG, "use the strip driver for BC_HALO");
  const long long n = NF * c->g.plane;
  c->leja_u = u;
  c->leja_fu = fu;
  int rc = leja_setup(c, v, n, unorm, dt, q, theta, tol, xi, coeffs, ncoef, nullptr, false, true,
                      !xmhd_leja_loop_available(c));
  if (rc) return rc;
  xmhd_leja_state st;
  if (xmhd_leja_loop_available(c)) {
    rc = xmhd_leja_loop(c);
    if (rc) return rc;
    rc = sync_ctl(c);
    if (rc) return rc;
    fill_state(*c->ctl_h, &st);
  } else {
    rc = leja_run(c, &st);
    if (rc) return rc;
  }
  if (st.status == LJ_MODE_ERROR)
    return fail(XMHD_CUDA_ERROR, "Leja kernel variant / interpolant mode mismatch");
  if (st.status == LJ_NEED_COEFFS)
    return fail(XMHD_BADARG, "coefficient table ended at term " + std::to_string(st.m) +
                                 ": pass entries up to the reference's 500-entry chunk");
  if (iterations) *iterations = st.iterations;
  if (rhs_calls) *rhs_calls = st.rhs_calls;
  if (converged) *converged = st.status == LJ_CONVERGED;
  if (residual) *residual = st.residual;
  if (st.status == LJ_RHS_BAD) {
    rc = scan_bad_cells_shifted(c, u, current_y(c), st.eps, bad_cells);
    return rc ? rc : XMHD_NONFINITE;
  }
  {
    const double* pb[2] = {pbuf_of(c, 0), pbuf_of(c, 1)};
    CK(launch_leja_copy_result(p_out, pb, c->ybuf, c->leja_v0, c->ctl, n, c->stream));
  }
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  return XMHD_OK;
}

int xmhd_leja_current_y(xmhd_ctx* c, double* dst) {
  if (!c || !dst) return fail(XMHD_BADARG, "null arg");
  int rc = sync_ctl(c);
  if (rc) return rc;
  const long long n = c->gen_n ? c->gen_n : NF * c->g.plane;
  CK(cudaMemcpyAsync(dst, current_y(c), sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream));
  return XMHD_OK;
}

int xmhd_leja_generic_start(xmhd_ctx* c, const double* v, long long n, double dt, double q,
                            double theta, double tol, const double* xi, const double* coeffs,
                            int ncoef, xmhd_leja_state* st) {
  if (!c || !v || !xi || !coeffs || n < 1) return fail(XMHD_BADARG, "bad arg");
  int rc = leja_setup(c, v, n, 1.0, dt, q, theta, tol, xi, coeffs, ncoef, nullptr, true);
  if (rc) return rc;
  c->gen_n = n;
  rc = sync_ctl(c);
  if (rc) return rc;
  fill_state(*c->ctl_h, st);
  return XMHD_OK;
}

int xmhd_leja_generic_step(xmhd_ctx* c, const double* w, xmhd_leja_state* st) {
  if (!c || !c->gen_n) return fail(XMHD_BADARG, "no generic Leja call in progress");
  CK(launch_leja_update(w, c->gen_n, c->ctl, c->ybuf, c->pbuf, c->coeffs_d, c->xi_d, redbuf(c),
                        c->stream));
  c->launches++;
  int rc = sync_ctl(c);
  if (rc) return rc;
  fill_state(*c->ctl_h, st);
  return XMHD_OK;
}

int xmhd_leja_generic_resume(xmhd_ctx* c, const double* coeffs, int ncoef, xmhd_leja_state* st) {
  if (!c || !coeffs) return fail(XMHD_BADARG, "null arg");
  int rc = upload_coeffs(c, coeffs, ncoef);
  if (rc) return rc;
  c->ctl_h->ncoef = ncoef;
  c->ctl_h->status = LJ_RUNNING;
  CK(cudaMemcpyAsync(&c->ctl->ncoef, &c->ctl_h->ncoef, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->ctl->status, &c->ctl_h->status, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  rc = sync_ctl(c);
  if (rc) return rc;
  fill_state(*c->ctl_h, st);
  return XMHD_OK;
}

int xmhd_time_stencil(xmhd_ctx* c, int mode, const double* u, const double* fu, double unorm,
                      const double* w, double* out, int n_iter, double* ms_per_launch) {
  if (!c || !u || !out || !ms_per_launch) return fail(XMHD_BADARG, "null arg");
  if (mode != MODE_RHS && mode != MODE_JVP) return fail(XMHD_BADARG, "mode must be 0 (RHS) or 1 (JVP)");
  if (mode == MODE_JVP && (!fu || !w)) return fail(XMHD_BADARG, "null arg");
  if (n_iter < 1 || n_iter > 400) return fail(XMHD_BADARG, "n_iter must be in [1, 400]");
  StencilArgs a = base_args(c);
  a.u = u;
  a.out = out;
  if (mode == MODE_JVP) {
    const long long n = NF * c->g.plane;
    CK(launch_norm(w, n, redbuf(c), c->stream));
    c->launches++;
    int rc = fetch_doubles(c, 1);
    if (rc) return rc;
    const double wn = c->h_dbl[0];
    if (wn == 0.0) return fail(XMHD_BADARG, "zero direction");
    // the FD step of xmhd_jvp (linearize.py:65)
    const double eps = (1.4901161193847656e-08 * py_max(1.0, unorm)) / py_max(wn, 1e-300);
    a.dir = w;
    a.fu = fu;
    a.eps = eps;
    a.epsd = make_divisor(eps, c->force_ieee);
  }
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(launch_stencil(mode, a, c->grid, c->stream));   // warm-up
  CK(cudaEventRecord(e0, c->stream));
  for (int k = 0; k < n_iter; ++k) CK(launch_stencil(mode, a, c->grid, c->stream));
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaEventSynchronize(e1));
  c->launches += n_iter + 1;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  int bad = 0;
  int rc = fetch_bad(c, &bad);
  if (rc) return rc;
  *ms_per_launch = (double)ms / n_iter;
  return bad ? XMHD_NONFINITE : XMHD_OK;
}

int xmhd_time_leja_iterations(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                              const double* v, double dt, double q, double theta,
                              const double* xi, const double* coeffs500, int n_iter,
                              double* ms_per_iter, double* ms_by_kind) {
  if (!c || !u || !fu || !v || !xi || !coeffs500 || !ms_per_iter) return fail(XMHD_BADARG, "null arg");
  if (n_iter < 1 || n_iter > 400) return fail(XMHD_BADARG, "n_iter must be in [1, 400]");
  const long long n = NF * c->g.plane;
  c->leja_u = u;
  c->leja_fu = fu;
  // tol = 0: the convergence test never fires, every launch does a full term
  int rc = leja_setup(c, v, n, unorm, dt, q, theta, 0.0, xi, coeffs500, 500, nullptr, false, true,
                      true);
  if (rc) return rc;
  StencilArgs a = leja_args(c);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  rc = launch_term(c, a);  // warm-up term
  if (rc) return rc;
  float ms = 0.f;
  if (!ms_by_kind) {
    CK(cudaEventRecord(e0, c->stream));
    for (int k = 0; k < n_iter; ++k) {
      rc = launch_term(c, a);
      if (rc) return rc;
    }
    CK(cudaEventRecord(e1, c->stream));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
  } else {
    // one event between consecutive launches: the average duration of each
    // interpolant mode (lookahead: odd terms PM_SKIP, even terms PM_LOOK)
    std::vector<cudaEvent_t> ev(n_iter + 1);
    std::vector<int> kind(n_iter);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], c->stream));
    for (int k = 0; k < n_iter; ++k) {
      const int pm = c->ctl_h->defer == 2 ? leja_pmode(c->leja_next_term, 2) : PM_STORE;
      kind[k] = pm == PM_SKIP ? 0 : 1;
      rc = launch_term(c, a);
      if (rc) return rc;
      CK(cudaEventRecord(ev[k + 1], c->stream));
    }
    CK(cudaEventSynchronize(ev[n_iter]));
    double sum[2] = {0.0, 0.0};
    int cnt[2] = {0, 0};
    for (int k = 0; k < n_iter; ++k) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
      sum[kind[k]] += t;
      cnt[kind[k]]++;
    }
    CK(cudaEventElapsedTime(&ms, ev[0], ev[n_iter]));
    for (auto& e : ev) cudaEventDestroy(e);
    ms_by_kind[0] = cnt[0] ? sum[0] / cnt[0] : 0.0;
    ms_by_kind[1] = cnt[1] ? sum[1] / cnt[1] : 0.0;
  }
  c->launches += 1;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  rc = sync_ctl(c);
  if (rc) return rc;
  if (c->ctl_h->status != LJ_RUNNING)
    return fail(XMHD_BADARG, "timing run left RUNNING early (status " +
                                 std::to_string(c->ctl_h->status) + ")");
  *ms_per_iter = (double)ms / n_iter;
  return XMHD_OK;
}

// ---------------------------------------------------------------- y-strips
// Every norm on a strip is a cross-rank sum: these entry points expose the
// local partial sums (device or host) and the control updates that run after
// the caller's allreduce, so all ranks take identical decisions.

int xmhd_sumsq(xmhd_ctx* c, const double* x, long long n, double* out) {
  if (!c || !x || !out) return fail(XMHD_BADARG, "null arg");
  CK(launch_sumsq(x, n, redbuf(c), c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 1);
  if (rc) return rc;
  *out = c->h_dbl[0];
  return XMHD_OK;
}

// ---- Krylov baseline (krylov.py:34-84) ---------------------------------------

static int ensure_krylov(xmhd_ctx* c) {
  if (c->kry_d) return XMHD_OK;
  CK(cudaMalloc(&c->kry_d, sizeof(double) * 512));
  CK(cudaMallocHost(&c->kry_h, sizeof(double) * 512));
  return XMHD_OK;
}

int xmhd_krylov_mgs(xmhd_ctx* c, const double* const* basis, int nb, double* w, long long n,
                    double* coef_out, double* wsumsq_out) {
  if (!c || !basis || !w || !coef_out || !wsumsq_out || nb < 1 || nb > KRYLOV_MAX + 1)
    return fail(XMHD_BADARG, "bad krylov_mgs arguments");
  for (int i = 0; i < nb; ++i)
    if (!basis[i]) return fail(XMHD_BADARG, "null basis vector");
  int rc = ensure_krylov(c);
  if (rc) return rc;
  // slots: [0, nb) pass-1 coefficients, [nb, 2nb) pass-2, 2nb = sum w^2
  double* s = c->kry_d;
  const RedBuf rb = redbuf(c);
  CK(launch_mgs(w, n, nullptr, nullptr, 0.0, basis[0], s, rb, c->stream));
  c->launches++;
  for (int pass = 0; pass < 2; ++pass) {
    double* sp = s + pass * nb;
    for (int i = 0; i < nb; ++i) {
      const bool last = (i + 1 == nb);
      const double* next = !last ? basis[i + 1] : (pass == 0 ? basis[0] : nullptr);
      double* cout = !last ? sp + i + 1 : s + (pass + 1) * nb;
      CK(launch_mgs(w, n, basis[i], sp + i, 0.0, next, cout, rb, c->stream));
      c->launches++;
    }
  }
  CK(cudaMemcpyAsync(c->kry_h, s, sizeof(double) * (2 * nb + 1), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 2 * nb; ++k) coef_out[k] = c->kry_h[k];
  *wsumsq_out = c->kry_h[2 * nb];
  return XMHD_OK;
}

int xmhd_mgs_update(xmhd_ctx* c, double* w, long long n, const double* v, double coef,
                    const double* next, double* sum_out) {
  if (!c || !w || !sum_out) return fail(XMHD_BADARG, "null arg");
  int rc = ensure_krylov(c);
  if (rc) return rc;
  CK(launch_mgs(w, n, v, nullptr, coef, next, c->kry_d, redbuf(c), c->stream));
  c->launches++;
  CK(cudaMemcpyAsync(c->kry_h, c->kry_d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *sum_out = c->kry_h[0];
  return XMHD_OK;
}

int xmhd_krylov_combine(xmhd_ctx* c, const double* const* basis, const double* coef, int m,
                        double scale, long long n, double* out) {
  if (!c || !basis || !coef || !out || m < 1 || m > KRYLOV_MAX)
    return fail(XMHD_BADARG, "bad krylov_combine arguments");
  KrylovBasis B;
  std::memset(&B, 0, sizeof(B));
  for (int k = 0; k < m; ++k) {
    if (!basis[k]) return fail(XMHD_BADARG, "null basis vector");
    B.v[k] = basis[k];
    B.c[k] = coef[k];
  }
  CK(launch_krylov_combine(out, n, B, m, scale, redbuf(c), c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_jvp_eps(xmhd_ctx* c, const double* u, const double* fu, const double* w, double eps,
                 double* out, double* out_sumsq) {
  if (!c || !u || !fu || !w || !out) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO && !(c->g.halo_lo && c->g.halo_lo_dir))
    return fail(XMHD_BADARG, "halo rows (state and direction) not set");
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  StencilArgs a = base_args(c);
  a.u = u;
  a.dir = w;
  a.fu = fu;
  a.out = out;
  a.eps = eps;
  a.epsd = make_divisor(eps, c->force_ieee);
  CK(launch_stencil(MODE_JVP, a, c->grid, c->stream));
  c->launches++;
  int rc = fetch_doubles(c, 2);
  if (rc) return rc;
  if (out_sumsq) *out_sumsq = c->h_dbl[1];
  int bad = 0;
  rc = fetch_bad(c, &bad);
  if (rc) return rc;
  return bad ? XMHD_NONFINITE : XMHD_OK;
}

int xmhd_leja_strip_start(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                          const double* v, double dt, double q, double theta, double tol,
                          const double* xi, const double* coeffs, int ncoef, double* sums) {
  if (!c || !u || !fu || !v || !xi || !coeffs || !sums) return fail(XMHD_BADARG, "null arg");
  c->leja_u = u;
  c->leja_fu = fu;
  return leja_setup(c, v, NF * c->g.plane, unorm, dt, q, theta, tol, xi, coeffs, ncoef, sums);
}

int xmhd_leja_strip_start_finalize(xmhd_ctx* c, const double* sums) {
  if (!c || !sums) return fail(XMHD_BADARG, "null arg");
  CK(launch_leja_init_finalize(c->ctl, sums, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_strip_pack(xmhd_ctx* c, double* send_lo, double* send_hi, double* halo_lo_dir,
                         double* halo_hi_dir, int mirror_lo, int mirror_hi) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  CK(launch_leja_pack_halo(c->ctl, c->ybuf[0], c->ybuf[1], c->g.nx, c->g.ny, send_lo, send_hi,
                           halo_lo_dir, halo_hi_dir, mirror_lo, mirror_hi, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_strip_iterate(xmhd_ctx* c, double* sums) {
  if (!c || !sums) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy == BC_HALO && !(c->g.halo_lo && c->g.halo_lo_dir))
    return fail(XMHD_BADARG, "halo rows (state and direction) not set");
  StencilArgs a = leja_args(c);
  a.ext_sums = sums;
  return launch_term(c, a);
}

int xmhd_leja_strip_finalize(xmhd_ctx* c, const double* sums) {
  if (!c || !sums) return fail(XMHD_BADARG, "null arg");
  CK(launch_leja_finalize(c->ctl, sums, c->coeffs_d, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_query(xmhd_ctx* c, xmhd_leja_state* st) {
  if (!c || !st) return fail(XMHD_BADARG, "null arg");
  int rc = sync_ctl(c);
  if (rc) return rc;
  fill_state(*c->ctl_h, st);
  if (c->ctl_h->status == LJ_MODE_ERROR)
    return fail(XMHD_CUDA_ERROR, "Leja kernel variant / interpolant mode mismatch");
  if (c->ctl_h->status == LJ_RUNNING || c->ctl_h->status == LJ_NEED_COEFFS)
    c->leja_next_term = c->ctl_h->m;   // terms launched past a stop exited
  return XMHD_OK;
}

int xmhd_leja_set_coeffs(xmhd_ctx* c, const double* coeffs, int ncoef) {
  if (!c || !coeffs) return fail(XMHD_BADARG, "null arg");
  int rc = upload_coeffs(c, coeffs, ncoef);
  if (rc) return rc;
  c->ctl_h->ncoef = ncoef;
  c->ctl_h->status = LJ_RUNNING;
  CK(cudaMemcpyAsync(&c->ctl->ncoef, &c->ctl_h->ncoef, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->ctl->status, &c->ctl_h->status, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  return XMHD_OK;
}

// ---- y-strips over peer memory (NVLink / NVSwitch, CUDA IPC) -------------

namespace {

struct P2PLayout {
  size_t halo[2][2];   // [parity][lo, hi] byte offsets of [NF][2][nx] ghost rows
  size_t board, flag, bytes;
};

P2PLayout p2p_layout(int nx) {
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t hb = al(sizeof(double) * NF * 2 * (size_t)nx);
  P2PLayout L;
  for (int par = 0; par < 2; ++par)
    for (int side = 0; side < 2; ++side) L.halo[par][side] = hb * (par * 2 + side);
  L.board = 4 * hb;
  L.flag = L.board + al(sizeof(double) * 2 * P2P_MAX * 4);
  L.bytes = L.flag + al(sizeof(unsigned long long) * 2 * P2P_MAX);
  return L;
}

// Neighbours of `rank` on the strip chain (a ring when periodic in y); a
// missing neighbour is a reflecting wall whose ghost rows the rank builds itself.
void p2p_wire(xmhd_ctx* c, int rank, int nranks, char* const* bases, int periodic) {
  const P2PLayout L = p2p_layout(c->g.nx);
  P2PArgs& x = c->p2p;
  std::memset(&x, 0, sizeof(x));
  x.rank = rank;
  x.nranks = nranks;
  const int below = rank > 0 ? rank - 1 : (periodic ? nranks - 1 : -1);
  const int above = rank < nranks - 1 ? rank + 1 : (periodic ? 0 : -1);
  for (int par = 0; par < 2; ++par) {
    double* own_lo = (double*)(bases[rank] + L.halo[par][0]);
    double* own_hi = (double*)(bases[rank] + L.halo[par][1]);
    x.halo_lo_dir[par] = own_lo;
    x.halo_hi_dir[par] = own_hi;
    // my rows 0, 1 are the rows ny, ny+1 of the rank below (its "hi" ghost rows)
    x.dst_lo[par] = below >= 0 ? (double*)(bases[below] + L.halo[par][1]) : own_lo;
    x.dst_hi[par] = above >= 0 ? (double*)(bases[above] + L.halo[par][0]) : own_hi;
  }
  x.mirror_lo = below < 0;
  x.mirror_hi = above < 0;
  for (int q = 0; q < nranks; ++q) {
    x.board[q] = (double*)(bases[q] + L.board);
    x.flag[q] = (unsigned long long*)(bases[q] + L.flag);
  }
  c->p2p_ready = true;
}

// Ghost rows of y0 (parity 0) into the neighbours / my mirror rows.
int p2p_push_y0(xmhd_ctx* c) {
  const P2PArgs& x = c->p2p;
  CK(launch_leja_pack_halo(c->ctl, c->ybuf[0], c->ybuf[1], c->g.nx, c->g.ny,
                           x.mirror_lo ? nullptr : x.dst_lo[0],
                           x.mirror_hi ? nullptr : x.dst_hi[0],
                           x.mirror_lo ? x.dst_lo[0] : nullptr,
                           x.mirror_hi ? x.dst_hi[0] : nullptr, x.mirror_lo, x.mirror_hi,
                           c->stream));
  c->launches++;
  return XMHD_OK;
}

int p2p_check(xmhd_ctx* c) {
  if (!c) return fail(XMHD_BADARG, "null ctx");
  if (c->g.bcy != BC_HALO) return fail(XMHD_BADARG, "peer transport needs a y-strip context");
  if (!c->p2p_ready) return fail(XMHD_BADARG, "peer transport not connected");
  if (!c->g.halo_lo) return fail(XMHD_BADARG, "state halo rows not set");
  return XMHD_OK;
}

}  // namespace

int xmhd_p2p_alloc(xmhd_ctx* c, void* handle_out) {
  if (!c || !handle_out) return fail(XMHD_BADARG, "null arg");
  if (c->g.bcy != BC_HALO) return fail(XMHD_BADARG, "peer transport needs a y-strip context");
  if (!c->p2p_base) {
    const P2PLayout L = p2p_layout(c->g.nx);
    CK(cudaMalloc((void**)&c->p2p_base, L.bytes));
    CK(cudaMemset(c->p2p_base, 0, L.bytes));
    CK(cudaDeviceSynchronize());
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->p2p_base));
  std::memcpy(handle_out, &h, sizeof(h));
  return XMHD_OK;
}

int xmhd_p2p_connect(xmhd_ctx* c, int rank, int nranks, const void* handles, int periodic) {
  if (!c || !handles) return fail(XMHD_BADARG, "null arg");
  if (nranks < 2 || nranks > P2P_MAX || rank < 0 || rank >= nranks)
    return fail(XMHD_BADARG, "rank / nranks out of range (2..8 ranks per node)");
  if (!c->p2p_base) return fail(XMHD_BADARG, "xmhd_p2p_alloc first");
  char* bases[P2P_MAX] = {};
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      bases[q] = c->p2p_base;
      continue;
    }
    if (!c->p2p_peer[q]) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, (const char*)handles + q * sizeof(cudaIpcMemHandle_t), sizeof(h));
      CK(cudaIpcOpenMemHandle((void**)&c->p2p_peer[q], h, cudaIpcMemLazyEnablePeerAccess));
    }
    bases[q] = c->p2p_peer[q];
  }
  p2p_wire(c, rank, nranks, bases, periodic);
  return XMHD_OK;
}

int xmhd_p2p_connect_local(xmhd_ctx* const* ctxs, int nranks, int periodic) {
  if (!ctxs || nranks < 2 || nranks > P2P_MAX) return fail(XMHD_BADARG, "bad ranks");
  char* bases[P2P_MAX] = {};
  for (int q = 0; q < nranks; ++q) {
    if (!ctxs[q] || !ctxs[q]->p2p_base) return fail(XMHD_BADARG, "xmhd_p2p_alloc every rank first");
    if (ctxs[q]->g.nx != ctxs[0]->g.nx) return fail(XMHD_BADARG, "ranks differ in nx");
    bases[q] = ctxs[q]->p2p_base;
  }
  for (int r = 0; r < nranks; ++r) p2p_wire(ctxs[r], r, nranks, bases, periodic);
  return XMHD_OK;
}

int xmhd_p2p_probe(xmhd_ctx* c, double value) {
  if (!c || !c->p2p_ready) return fail(XMHD_BADARG, "peer transport not connected");
  CK(launch_p2p_probe(c->p2p, value, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return XMHD_OK;
}

int xmhd_p2p_read_board(xmhd_ctx* c, double* out) {
  if (!c || !out || !c->p2p_base) return fail(XMHD_BADARG, "null arg");
  const P2PLayout L = p2p_layout(c->g.nx);
  CK(cudaMemcpy(out, c->p2p_base + L.board, sizeof(double) * P2P_MAX * 4,
                cudaMemcpyDeviceToHost));
  return XMHD_OK;
}

int xmhd_leja_p2p_start(xmhd_ctx* c, const double* u, const double* fu, double unorm,
                        const double* v, double dt, double q, double theta, double tol,
                        const double* xi, const double* coeffs, int ncoef) {
  int rc = p2p_check(c);
  if (rc) return rc;
  if (!u || !fu || !v || !xi || !coeffs) return fail(XMHD_BADARG, "null arg");
  c->leja_u = u;
  c->leja_fu = fu;
  double* sums = c->result + 8;
  rc = leja_setup(c, v, NF * c->g.plane, unorm, dt, q, theta, tol, xi, coeffs, ncoef, sums);
  if (rc) return rc;
  rc = p2p_push_y0(c);
  if (rc) return rc;
  StencilArgs a = leja_args(c);
  a.ext_sums = sums;
  a.p2p = c->p2p;
  CK(launch_leja_p2p_init(a, c->stream));
  c->launches++;
  return XMHD_OK;
}

int xmhd_leja_p2p_run(xmhd_ctx* c, xmhd_leja_state* st) {
  int rc = p2p_check(c);
  if (rc) return rc;
  return leja_run(c, st, true);
}

// ---- the same driver with P ranks emulated on one GPU (tests) -------------

namespace {

int emul_args(xmhd_ctx* const* ctxs, int nranks, StencilArgs** dev) {
  xmhd_ctx* c0 = ctxs[0];
  if (!c0->emul_args) CK(cudaMalloc(&c0->emul_args, sizeof(StencilArgs) * P2P_MAX));
  static StencilArgs host[P2P_MAX];
  for (int r = 0; r < nranks; ++r) {
    host[r] = leja_args(ctxs[r]);
    host[r].ext_sums = ctxs[r]->result + 8;
    host[r].p2p = ctxs[r]->p2p;
  }
  CK(cudaMemcpy(c0->emul_args, host, sizeof(StencilArgs) * nranks, cudaMemcpyHostToDevice));
  *dev = c0->emul_args;
  return XMHD_OK;
}

int emul_check(xmhd_ctx* const* ctxs, int nranks) {
  if (!ctxs || nranks < 2 || nranks > P2P_MAX) return fail(XMHD_BADARG, "bad ranks");
  for (int r = 0; r < nranks; ++r) {
    int rc = p2p_check(ctxs[r]);
    if (rc) return rc;
    if (ctxs[r]->stream != ctxs[0]->stream) return fail(XMHD_BADARG, "ranks must share a stream");
  }
  return XMHD_OK;
}

}  // namespace

int xmhd_leja_p2p_emul_start(xmhd_ctx* const* ctxs, int nranks, const double* const* u,
                             const double* const* fu, double unorm, const double* const* v,
                             double dt, double q, double theta, double tol, const double* xi,
                             const double* coeffs, int ncoef) {
  int rc = emul_check(ctxs, nranks);
  if (rc) return rc;
  for (int r = 0; r < nranks; ++r) {
    xmhd_ctx* c = ctxs[r];
    c->leja_u = u[r];
    c->leja_fu = fu[r];
    rc = leja_setup(c, v[r], NF * c->g.plane, unorm, dt, q, theta, tol, xi, coeffs, ncoef,
                    c->result + 8);
    if (!rc) rc = p2p_push_y0(c);
    if (rc) return rc;
  }
  StencilArgs* dev = nullptr;
  rc = emul_args(ctxs, nranks, &dev);
  if (rc) return rc;
  CK(launch_leja_p2p_init_emul(dev, nranks, ctxs[0]->stream));
  CK(cudaStreamSynchronize(ctxs[0]->stream));
  return XMHD_OK;
}

int xmhd_leja_p2p_emul_run(xmhd_ctx* const* ctxs, int nranks, xmhd_leja_state* st) {
  int rc = emul_check(ctxs, nranks);
  if (rc) return rc;
  StencilArgs* dev = nullptr;
  rc = emul_args(ctxs, nranks, &dev);
  if (rc) return rc;
  const int cap = leja_emul_max_blocks(ctxs[0]->nsm) / nranks;
  int nblk = 0;
  for (int r = 0; r < nranks; ++r) nblk = ctxs[r]->grid > nblk ? ctxs[r]->grid : nblk;
  if (nblk > cap) nblk = cap;
  if (nblk < 1) return fail(XMHD_BADARG, "too many emulated ranks for one cooperative launch");
  const StencilArgs a0 = leja_args(ctxs[0]);
  rc = sync_ctl(ctxs[0]);
  if (rc) return rc;
  for (;;) {
    // one term per launch: its interpolant mode from the (synced) term index
    const LejaCtl& h0 = *ctxs[0]->ctl_h;
    const int pm = (h0.defer == 2) ? leja_pmode(h0.m, 2) : PM_ANY;
    CK(launch_leja_emul(dev, a0, nranks, nblk, pm, ctxs[0]->stream));
    for (int r = 0; r < nranks; ++r) ctxs[r]->launches++;
    for (int r = 0; r < nranks; ++r) {
      rc = sync_ctl(ctxs[r]);
      if (rc) return rc;
      const LejaCtl& h = *ctxs[r]->ctl_h;
      const LejaCtl& h0 = *ctxs[0]->ctl_h;
      if (h.status != h0.status || h.iters != h0.iters || h.epoch != h0.epoch)
        return fail(XMHD_CUDA_ERROR, "emulated ranks diverged");
    }
    if (ctxs[0]->ctl_h->status != LJ_RUNNING) break;
  }
  for (int r = 0; r < nranks; ++r) ctxs[r]->p2p_epoch = ctxs[r]->ctl_h->epoch;
  fill_state(*ctxs[0]->ctl_h, st);
  if (ctxs[0]->ctl_h->status == LJ_PEER_TIMEOUT)
    return fail(XMHD_CUDA_ERROR, "peer-memory exchange timed out");
  return XMHD_OK;
}

int xmhd_leja_generic_result(xmhd_ctx* c, double* p_out) {
  int rc = xmhd_leja_result(c, p_out);
  c->gen_n = 0;
  return rc;
}

}  // extern "C"
