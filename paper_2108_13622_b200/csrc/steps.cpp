// One exponential Rosenbrock step enqueued natively (integrators.py:146-199).
//
// The host-side stage algebra of EXPRB43 / EXPRB54s4 issues ~30 device
// operations per step; on small grids the Python/ctypes cost of issuing them
// exceeded the device time.  This is the same sequence of C-ABI operations
// the asynchronous Python step issues (integrators._step_async), in the same
// order with the same coefficients, so the results are bitwise those of that
// path; the caller reads the step record once (xmhd_async_fetch).
//
// Coefficients are Python's: `u + dt*a + dt*b` is ((1*u + dt*a) + dt*b) with
// one rounding per operation (xmhd_lincomb), constants such as (729/125)*dt
// are folded the way the reference's expressions fold them.
#include <cstring>

#include "xmhd_b200.h"

namespace {

struct StepCtx {
  xmhd_ctx* c;
  const double* u;
  const double* fu;
  double unorm;
  long long n;
  const double* par;     // [nphi][3]: dt_eff, q, theta
  const double* tables;  // [nphi][64]
  int tiny;              // alpha < 1e-14: phi_l(0) v = v / l!
  double tol;
  const double* xi;
  int k = 0;             // next phi-action
  int rc = XMHD_OK;
};

bool ok(StepCtx& s, int rc) {
  if (rc != XMHD_OK && s.rc == XMHD_OK) s.rc = rc;
  return s.rc == XMHD_OK;
}

// out = c0*v0 (+ c1*v1 (+ c2*v2 (+ c3*v3))), left to right
void lc(StepCtx& s, double* out, int nt, const double* cf, const double* const* v) {
  if (s.rc) return;
  ok(s, xmhd_lincomb(s.c, out, s.n, v, cf, nt, nullptr, nullptr));
}

void lc2(StepCtx& s, double* out, double c0, const double* v0, double c1, const double* v1) {
  const double cf[2] = {c0, c1};
  const double* v[2] = {v0, v1};
  lc(s, out, 2, cf, v);
}

void lc3(StepCtx& s, double* out, double c0, const double* v0, double c1, const double* v1,
         double c2, const double* v2) {
  const double cf[3] = {c0, c1, c2};
  const double* v[3] = {v0, v1, v2};
  lc(s, out, 3, cf, v);
}

void lc4(StepCtx& s, double* out, double c0, const double* v0, double c1, const double* v1,
         double c2, const double* v2, double c3, const double* v3, bool flagged) {
  if (s.rc) return;
  const double cf[4] = {c0, c1, c2, c3};
  const double* v[4] = {v0, v1, v2, v3};
  if (flagged) ok(s, xmhd_lincomb_async(s.c, out, s.n, v, cf, 4));
  else lc(s, out, 4, cf, v);
}

// phi_l(c J dt) vec (_PhiBroker.apply, integrators.py:120-136)
void phi(StepCtx& s, int l, const double* vec, double* out) {
  if (s.rc) return;
  const int k = s.k++;
  if (s.tiny) {
    const double fact = (l == 1) ? 1.0 : (l == 2) ? 2.0 : (l == 3) ? 6.0 : 24.0;
    ok(s, xmhd_divide(s.c, out, vec, fact, s.n, nullptr));
    return;
  }
  const double* p = s.par + 3 * k;
  if (!ok(s, xmhd_leja_start_async(s.c, s.u, s.fu, s.unorm, vec, p[0], p[1], p[2], s.tol, s.xi,
                                   s.tables + 64 * k, 64)))
    return;
  if (!ok(s, xmhd_leja_loop(s.c))) return;
  ok(s, xmhd_leja_finish_async(s.c, out));
}

// F(stage) - F(u) - J (stage - u)  (integrators.py:146-153); t0..t2 scratch
void stage_difference(StepCtx& s, const double* stage, double* out, double* t0, double* t1,
                      double* t2) {
  if (s.rc) return;
  if (!ok(s, xmhd_rhs_async(s.c, stage, t0))) return;
  lc2(s, t1, 1.0, stage, -1.0, s.u);
  if (s.rc) return;
  if (!ok(s, xmhd_jvp_async(s.c, s.u, s.fu, s.unorm, t1, t2))) return;
  lc3(s, out, 1.0, t0, -1.0, s.fu, -1.0, t2);
}

}  // namespace

extern "C" int xmhd_step_async(xmhd_ctx* ctx, int scheme, const double* u, const double* fu,
                               double unorm, long long n, double dt, const double* phi_param,
                               const double* tables, int tiny_alpha, double tol,
                               const double* xi, double* work, double* u_new) {
  if (!ctx || !u || !fu || !phi_param || !tables || !xi || !work || !u_new || n < 1)
    return XMHD_BADARG;
  if (scheme != XMHD_SCHEME_EXPRB43 && scheme != XMHD_SCHEME_EXPRB54S4) return XMHD_BADARG;
  StepCtx s;
  s.c = ctx;
  s.u = u;
  s.fu = fu;
  s.unorm = unorm;
  s.n = n;
  s.par = phi_param;
  s.tables = tables;
  s.tiny = tiny_alpha;
  s.tol = tol;
  s.xi = xi;
  int rc = xmhd_async_begin(ctx);
  if (rc) return rc;
  double* W[XMHD_STEP_WORK];
  for (int i = 0; i < XMHD_STEP_WORK; ++i) W[i] = work + (long long)i * n;
  double *t0 = W[0], *t1 = W[1], *t2 = W[2];

  if (scheme == XMHD_SCHEME_EXPRB43) {   // integrators.py:156-171
    double *p0 = W[3], *a = W[4], *da = W[5], *phi1 = W[6], *p2 = W[7], *b = W[8], *db = W[9],
           *w3 = W[10], *w4 = W[11], *u3 = W[12];
    phi(s, 1, fu, p0);                                    // apply(1, 0.5, fu)
    lc2(s, a, 1.0, u, 0.5 * dt, p0);
    stage_difference(s, a, da, t0, t1, t2);
    phi(s, 1, fu, phi1);                                  // apply(1, 1.0, fu)
    phi(s, 1, da, p2);                                    // apply(1, 1.0, da)
    lc3(s, b, 1.0, u, dt, phi1, dt, p2);
    stage_difference(s, b, db, t0, t1, t2);
    lc2(s, w3, 16.0, da, -2.0, db);
    lc2(s, w4, -48.0, da, 12.0, db);
    phi(s, 3, w3, p0);                                    // apply(3, 1.0, w3)
    lc3(s, u3, 1.0, u, dt, phi1, dt, p0);
    phi(s, 4, w4, p2);                                    // apply(4, 1.0, w4)
    if (s.rc == XMHD_OK) {
      const double cf[2] = {1.0, dt};
      const double* v[2] = {u3, p2};
      ok(s, xmhd_lincomb_async(ctx, u_new, n, v, cf, 2));   // u4 (flagged)
    }
    if (s.rc == XMHD_OK) ok(s, xmhd_diff_norms_async(ctx, u3, u_new, n));   // error_norm(u3, u4)
  } else {                                 // integrators.py:174-199
    double *p0 = W[3], *a = W[4], *da = W[5], *p = W[6], *q = W[7], *b = W[8], *db = W[9],
           *cc = W[10], *dc = W[11], *w1 = W[12], *w2 = W[13], *w3 = W[14], *w4 = W[15],
           *phi1 = W[16], *p3 = W[17], *p4 = W[18], *u4 = W[19];
    phi(s, 1, fu, p0);                                    // apply(1, 0.25, fu)
    lc2(s, a, 1.0, u, 0.25 * dt, p0);
    stage_difference(s, a, da, t0, t1, t2);
    phi(s, 1, fu, p);                                     // apply(1, 0.5, fu)
    phi(s, 3, da, q);                                     // apply(3, 0.5, da)
    lc3(s, b, 1.0, u, 0.5 * dt, p, 4.0 * dt, q);
    stage_difference(s, b, db, t0, t1, t2);
    phi(s, 1, fu, p);                                     // apply(1, 0.9, fu)
    phi(s, 3, db, q);                                     // apply(3, 0.9, db)
    lc3(s, cc, 1.0, u, 0.9 * dt, p, (729.0 / 125.0) * dt, q);
    stage_difference(s, cc, dc, t0, t1, t2);
    lc2(s, w1, 64.0, da, -8.0, db);
    lc3(s, w2, -60.0, da, -(285.0 / 8.0), db, 125.0 / 8.0, dc);
    lc2(s, w3, 18.0, db, -(250.0 / 81.0), dc);
    lc2(s, w4, -60.0, db, 500.0 / 27.0, dc);
    phi(s, 1, fu, phi1);                                  // apply(1, 1.0, fu)
    phi(s, 3, w1, p3);                                    // apply(3, 1.0, w1)
    phi(s, 4, w2, p4);                                    // apply(4, 1.0, w2)
    lc4(s, u4, 1.0, u, dt, phi1, dt, p3, dt, p4, false);
    phi(s, 3, w3, p3);                                    // apply(3, 1.0, w3)
    phi(s, 4, w4, p4);                                    // apply(4, 1.0, w4)
    lc4(s, u_new, 1.0, u, dt, phi1, dt, p3, dt, p4, true);   // u5 (flagged)
    if (s.rc == XMHD_OK) ok(s, xmhd_diff_norms_async(ctx, u4, u_new, n));   // error_norm(u4, u5)
  }
  return s.rc;
}
