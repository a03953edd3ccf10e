// Streaming fp64 vector kernels for the host-side stepper algebra, norms and
// per-step diagnostics.  Each kernel is a grid-stride loop over the flat
// (8, ny, nx) vector with 128-bit loads where alignment allows; reductions use
// a fixed grid and a fixed combination order, so results are bit-identical
// from run to run.
//
// Element-wise arithmetic reproduces NumPy's single-rounding-per-ufunc order
// (integrators.py:146-199, linearize.py:113-127, leja.py:121-123).
#include <cfloat>
#include <cstring>
#include <type_traits>
#include "kernels.h"

namespace xb {

namespace {

constexpr int VT = 256;  // threads per block

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// NaN-propagating max (np.max propagates NaN).
__device__ __forceinline__ double nanmax(double a, double b) {
  return (a != a || b != b) ? CUDART_NAN : fmax(a, b);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-reduce NV values (sum or max), publish per-block partials, and let the
// last block combine them in fixed order.  Returns true in thread 0 of the
// last block, with out[k] holding the totals.
template <int NV, bool MAX>
__device__ bool grid_reduce(double (&v)[NV], const RedBuf& rb, double (&out)[NV]) {
  __shared__ double red[NV][VT / 32];
  __shared__ int am_last;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = MAX ? warp_max(v[k]) : warp_sum(v[k]);
    if (l == 0) red[k][w] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = red[k][0];
      for (int j = 1; j < VT / 32; ++j) s = MAX ? nanmax(s, red[k][j]) : s + red[k][j];
      rb.partials[4 * blockIdx.x + k] = s;
    }
    __threadfence();
    am_last = (atomicAdd(rb.ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  if (threadIdx.x >= 32) return false;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = MAX ? -CUDART_INF : 0.0;
    for (int b = l; b < (int)gridDim.x; b += 32) {
      const double p = __ldcg(rb.partials + 4 * b + k);
      s = MAX ? nanmax(s, p) : s + p;
    }
    s = MAX ? warp_max(s) : warp_sum(s);
    out[k] = __shfl_sync(0xffffffffu, s, 0);
  }
  if (l != 0) return false;
  *rb.ticket = 0u;
  return true;
}

// ---------------------------------------------------------------------------
// Shared traversal of a flat vector.  The vector is cut into pairs (2p, 2p+1);
// global thread g of G visits pairs g, g+G, g+2G, ... in that order (the loop
// is unrolled so several 128-bit loads are in flight per thread), both
// elements of a pair in index order; an odd last element is visited by global
// thread 0 after everything else.  Every reducing kernel below accumulates in
// visit order, so the same data gives the same sum, bit for bit, whichever
// kernel reduces it (||w|| of the asynchronous jvp prologue == xmhd_norm(w),
// the flagged combination's ||out|| == xmhd_norm(out), ...).  V2: every
// pointer is 16-byte aligned (128-bit accesses); otherwise the same order
// with 64-bit accesses.
// Measured at n = 1.3e8 (B200, HBM copy peak 6537 GB/s): the former one-element
// grid-stride loops reached 51-60% of peak in every kernel that stores
// (lincomb 3.4-4.0 TB/s, divide 3.9), 83-95% in the read-only ones.
template <bool V2>
__device__ __forceinline__ double2 ld2(const double* p, long long pair) {
  if (V2) return __ldg(reinterpret_cast<const double2*>(p) + pair);
  return make_double2(__ldg(p + 2 * pair), __ldg(p + 2 * pair + 1));
}

template <bool V2>
__device__ __forceinline__ void st2(double* p, long long pair, double a, double b) {
  if (V2) reinterpret_cast<double2*>(p)[pair] = make_double2(a, b);
  else { p[2 * pair] = a; p[2 * pair + 1] = b; }
}

template <int NIN, int NOUT>
struct Ptrs {
  const double* in[NIN > 0 ? NIN : 1];
  double* out[NOUT > 0 ? NOUT : 1];
};

// op(x[NIN], y[NOUT]) handles one element (its accumulators live in op).
template <int NIN, int NOUT, bool V2, typename Op>
__device__ __forceinline__ void stream(long long n, const Ptrs<NIN, NOUT>& P, Op& op) {
  constexpr int U = (NIN + NOUT >= 4) ? 2 : 4;
  constexpr int NI = NIN > 0 ? NIN : 1, NO = NOUT > 0 ? NOUT : 1;
  const long long npairs = n >> 1, G = (long long)gridDim.x * VT;
  long long p = (long long)blockIdx.x * VT + threadIdx.x;
  for (; p + (U - 1) * G < npairs; p += U * G) {
    double2 x[U][NI];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < NIN; ++k) x[u][k] = ld2<V2>(P.in[k], p + u * G);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double xa[NI], xb[NI], ya[NO], yb[NO];
#pragma unroll
      for (int k = 0; k < NIN; ++k) { xa[k] = x[u][k].x; xb[k] = x[u][k].y; }
      op(xa, ya);
      op(xb, yb);
#pragma unroll
      for (int k = 0; k < NOUT; ++k) st2<V2>(P.out[k], p + u * G, ya[k], yb[k]);
    }
  }
  for (; p < npairs; p += G) {
    double xa[NI], xb[NI], ya[NO], yb[NO];
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
      const double2 v = ld2<V2>(P.in[k], p);
      xa[k] = v.x;
      xb[k] = v.y;
    }
    op(xa, ya);
    op(xb, yb);
#pragma unroll
    for (int k = 0; k < NOUT; ++k) st2<V2>(P.out[k], p, ya[k], yb[k]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double xa[NI], ya[NO];
#pragma unroll
    for (int k = 0; k < NIN; ++k) xa[k] = __ldg(P.in[k] + (n - 1));
    op(xa, ya);
#pragma unroll
    for (int k = 0; k < NOUT; ++k) P.out[k][n - 1] = ya[k];
  }
}

template <int NIN, int NOUT>
bool aligned16(const Ptrs<NIN, NOUT>& P) {
  unsigned long long bits = 0;
  for (int k = 0; k < NIN; ++k) bits |= (unsigned long long)P.in[k];
  for (int k = 0; k < NOUT; ++k) bits |= (unsigned long long)P.out[k];
  return (bits & 15ull) == 0;
}

struct SumSqOp {
  double acc = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[1], double (&)[1]) {
    acc = __fma_rn(x[0], x[0], acc);
  }
};

template <bool V2>
__global__ void __launch_bounds__(VT) norm_kernel(Ptrs<1, 0> P, long long n, RedBuf rb) {
  SumSqOp op;
  stream<1, 0, V2>(n, P, op);
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = sqrt(tot[0]);
}

// out = ((c0*v0 + c1*v1) + c2*v2) + c3*v3, one rounding per operation.
template <int NT>
struct LincombOp {
  double c[4];
  double acc = 0.0, bad = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[NT], double (&y)[1]) {
    double s = __dmul_rn(c[0], x[0]);
#pragma unroll
    for (int k = 1; k < NT; ++k) s = __dadd_rn(s, __dmul_rn(c[k], x[k]));
    y[0] = s;
    acc = __fma_rn(s, s, acc);
    if (!isfinite(s)) bad = 1.0;
  }
};

struct Coef4 {
  double c[4];
};

template <int NT, bool V2>
__global__ void __launch_bounds__(VT) lincomb_kernel(Ptrs<NT, 1> P, long long n, Coef4 cf,
                                                     int want_norm, RedBuf rb) {
  LincombOp<NT> op;
#pragma unroll
  for (int k = 0; k < 4; ++k) op.c[k] = cf.c[k];
  stream<NT, 1, V2>(n, P, op);
  if (!want_norm) return;
  double acc[2] = {op.acc, op.bad}, tot[2];
  if (grid_reduce<2, false>(acc, rb, tot)) {
    rb.result[0] = sqrt(tot[0]);
    rb.result[1] = tot[1] > 0.0 ? 1.0 : 0.0;
  }
}

// Stage vector and its offset from the base state in one pass
// (integrators.py:139-153): out = the combination above, diff = out - v0 (v0 =
// the base state u, coefficient 1), result[0] = ||diff|| -- the direction of
// the stage difference's jvp and the norm its FD step needs.
template <int NT>
struct LincombDiffOp {
  double c[4];
  double acc = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[NT], double (&y)[2]) {
    double s = __dmul_rn(c[0], x[0]);
#pragma unroll
    for (int k = 1; k < NT; ++k) s = __dadd_rn(s, __dmul_rn(c[k], x[k]));
    y[0] = s;
    const double d = __dsub_rn(s, x[0]);
    y[1] = d;
    acc = __fma_rn(d, d, acc);
  }
};

template <int NT, bool V2>
__global__ void __launch_bounds__(VT) lincomb_diff_kernel(Ptrs<NT, 2> P, long long n, Coef4 cf,
                                                          RedBuf rb) {
  LincombDiffOp<NT> op;
#pragma unroll
  for (int k = 0; k < 4; ++k) op.c[k] = cf.c[k];
  stream<NT, 2, V2>(n, P, op);
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = sqrt(tot[0]);
}

// Up to four combinations of the same three vectors in one pass (the w_k of
// integrators.py:166-167, 186-189): out_j = sum over the terms of row j in
// order, terms with a zero coefficient skipped (the reference's expressions
// simply do not contain them).
struct MultiCoef {
  double c[4][3];
  int nout;
};

template <int NOUT>
struct MultiOp {
  MultiCoef m;
  __device__ __forceinline__ void operator()(const double (&x)[3], double (&y)[NOUT]) {
#pragma unroll
    for (int j = 0; j < NOUT; ++j) {
      double s = 0.0;
      bool first = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        if (m.c[j][k] != 0.0) {
          const double t = __dmul_rn(m.c[j][k], x[k]);
          s = first ? t : __dadd_rn(s, t);
          first = false;
        }
      }
      y[j] = s;
    }
  }
};

template <int NOUT, bool V2>
__global__ void __launch_bounds__(VT) lincomb_multi_kernel(Ptrs<3, NOUT> P, long long n,
                                                           MultiCoef mc) {
  MultiOp<NOUT> op;
  op.m = mc;
  stream<3, NOUT, V2>(n, P, op);
}

// The two embedded solutions of a step and their distance in one pass
// (integrators.py:168-171, 190-199): the lower-order solution `lo` is formed
// in registers only, the higher-order one is stored, and ||lo - hi||, ||hi|| and
// the non-finite flag of hi are reduced like diffnorm_kernel / the flagged
// combination would reduce them on materialised vectors (same traversal).
//   KIND 43: lo = (c0*v0 + c1*v1) + c2*v2;  hi = 1.0*lo + c3*v3
//   KIND 54: s = c0*v0 + c1*v1;  lo = (s + c2*v2) + c3*v3;  hi = (s + c4*v4) + c5*v5
struct Coef6 {
  double c[6];
};

template <int KIND>
struct FinalPairOp {
  static constexpr int NIN = (KIND == 43) ? 4 : 6;
  double c[6];
  double acc_d = 0.0, acc_h = 0.0, bad = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[NIN], double (&y)[1]) {
    double lo, hi;
    if (KIND == 43) {
      lo = __dadd_rn(__dadd_rn(__dmul_rn(c[0], x[0]), __dmul_rn(c[1], x[1])), __dmul_rn(c[2], x[2]));
      hi = __dadd_rn(__dmul_rn(1.0, lo), __dmul_rn(c[3], x[3 < NIN ? 3 : 0]));
    } else {
      const double s = __dadd_rn(__dmul_rn(c[0], x[0]), __dmul_rn(c[1], x[1]));
      lo = __dadd_rn(__dadd_rn(s, __dmul_rn(c[2], x[2])), __dmul_rn(c[3], x[3]));
      hi = __dadd_rn(__dadd_rn(s, __dmul_rn(c[4], x[4 < NIN ? 4 : 0])),
                     __dmul_rn(c[5], x[5 < NIN ? 5 : 0]));
    }
    y[0] = hi;
    const double d = __dsub_rn(lo, hi);
    acc_d = __fma_rn(d, d, acc_d);
    acc_h = __fma_rn(hi, hi, acc_h);
    if (!isfinite(hi)) bad = 1.0;
  }
};

template <int KIND, bool V2>
__global__ void __launch_bounds__(VT) final_pair_kernel(Ptrs<FinalPairOp<KIND>::NIN, 1> P,
                                                        long long n, Coef6 cf, RedBuf rb) {
  FinalPairOp<KIND> op;
#pragma unroll
  for (int k = 0; k < 6; ++k) op.c[k] = cf.c[k];
  stream<FinalPairOp<KIND>::NIN, 1, V2>(n, P, op);
  double acc[3] = {op.acc_d, op.acc_h, op.bad}, tot[3];
  if (grid_reduce<3, false>(acc, rb, tot)) {
    rb.result[0] = sqrt(tot[0]);
    rb.result[1] = sqrt(tot[1]);
    rb.result[2] = tot[2] > 0.0 ? 1.0 : 0.0;
  }
}

struct DivideOp {
  double d;
  double acc = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[1], double (&y)[1]) {
    const double q = __ddiv_rn(x[0], d);
    y[0] = q;
    acc = __fma_rn(q, q, acc);
  }
};

template <bool V2>
__global__ void __launch_bounds__(VT) divide_kernel(Ptrs<1, 1> P, double d, long long n,
                                                    int want_norm, RedBuf rb) {
  DivideOp op;
  op.d = d;
  stream<1, 1, V2>(n, P, op);
  if (!want_norm) return;
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = sqrt(tot[0]);
}

// One division of the device power iteration (linearize.py:115-116, 124):
// out = x / div, then ||out|| and the next FD step in the last block.
template <bool V2>
__global__ void __launch_bounds__(VT) power_divide_kernel(Ptrs<1, 1> P, long long n,
                                                          PowerCtl* pc, RedBuf rb) {
  if (pc->status != PW_RUNNING) return;
  DivideOp op;
  op.d = pc->div;
  stream<1, 1, V2>(n, P, op);
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) power_after_divide(pc, tot[0]);
}

struct DiffNormOp {
  double acc0 = 0.0, acc1 = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[2], double (&)[1]) {
    const double d = __dsub_rn(x[0], x[1]);
    acc0 = __fma_rn(d, d, acc0);
    acc1 = __fma_rn(x[1], x[1], acc1);
  }
};

template <bool V2>
__global__ void __launch_bounds__(VT) diffnorm_kernel(Ptrs<2, 0> P, long long n, RedBuf rb) {
  DiffNormOp op;
  stream<2, 0, V2>(n, P, op);
  double acc[2] = {op.acc0, op.acc1}, tot[2];
  if (grid_reduce<2, false>(acc, rb, tot)) {
    rb.result[0] = sqrt(tot[0]);
    rb.result[1] = sqrt(tot[1]);
  }
}

// max |div B| with the 1-ghost extension of mhd.py:235-240.
__global__ void __launch_bounds__(VT) divb_kernel(Geom g, const double* __restrict__ u,
                                                  double* __restrict__ field, RedBuf rb) {
  double acc[1] = {0.0};
  const double* bx = u + (long long)BX * g.plane;
  const double* by = u + (long long)BY * g.plane;
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < g.plane;
       i += (long long)gridDim.x * VT) {
    const int j = (int)(i / g.nx), c = (int)(i % g.nx);
    // x neighbours of bx (odd under an x mirror)
    int cl = c - 1, cr = c + 1;
    double sl = 1.0, sr = 1.0;
    if (cl < 0) { if (g.bcx == BC_PERIODIC) cl += g.nx; else { cl = 0; sl = -1.0; } }
    if (cr >= g.nx) { if (g.bcx == BC_PERIODIC) cr -= g.nx; else { cr = g.nx - 1; sr = -1.0; } }
    int jd = j - 1, ju = j + 1;
    double sd = 1.0, su = 1.0;
    const double* byd = by;
    const double* byu = by;
    long long od, ou;
    if (g.bcy == BC_HALO) {
      od = (long long)jd * g.nx + c;
      ou = (long long)ju * g.nx + c;
      if (jd < 0) { byd = g.halo_lo + (long long)BY * 2 * g.nx; od = (long long)(jd + 2) * g.nx + c; }
      if (ju >= g.ny) { byu = g.halo_hi + (long long)BY * 2 * g.nx; ou = (long long)(ju - g.ny) * g.nx + c; }
    } else {
      if (jd < 0) { if (g.bcy == BC_PERIODIC) jd += g.ny; else { jd = 0; sd = -1.0; } }
      if (ju >= g.ny) { if (g.bcy == BC_PERIODIC) ju -= g.ny; else { ju = g.ny - 1; su = -1.0; } }
      od = (long long)jd * g.nx + c;
      ou = (long long)ju * g.nx + c;
    }
    const double xr = __dmul_rn(sr, bx[(long long)j * g.nx + cr]);
    const double xl = __dmul_rn(sl, bx[(long long)j * g.nx + cl]);
    const double yu = __dmul_rn(su, byu[ou]);
    const double yd = __dmul_rn(sd, byd[od]);
    const double dv = __dadd_rn(__ddiv_rn(__dsub_rn(xr, xl), g.h2x.d),
                                __ddiv_rn(__dsub_rn(yu, yd), g.h2y.d));
    if (field) field[i] = dv;
    acc[0] = nanmax(acc[0], fabs(dv));
  }
  double tot[1];
  if (grid_reduce<1, true>(acc, rb, tot)) rb.result[0] = tot[0];
}

__global__ void __launch_bounds__(VT) field_sum_kernel(const double* __restrict__ u,
                                                       long long plane, RedBuf rb) {
  // one launch per field pair would be simpler; 8 accumulators stay in regs
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int f0 = blockIdx.y * 4;
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < plane;
       i += (long long)gridDim.x * VT) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k] += __ldg(u + (long long)(f0 + k) * plane + i);
  }
  // blockIdx.y selects a disjoint partial slab
  RedBuf r2 = rb;
  r2.partials = rb.partials + 4LL * gridDim.x * blockIdx.y;
  r2.ticket = rb.ticket + blockIdx.y;
  double tot[4];
  if (grid_reduce<4, false>(acc, r2, tot)) {
#pragma unroll
    for (int k = 0; k < 4; ++k) rb.result[f0 + k] = tot[k];
  }
}

// Advective CFL surrogate of harness.py:105-116 (max over cells).
__global__ void __launch_bounds__(VT) cfl_kernel(const double* __restrict__ u, long long plane,
                                                 double gamma, double mu0, RedBuf rb) {
  double acc[2] = {-CUDART_INF, -CUDART_INF};
  const double gm1 = gamma - 1.0;
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < plane;
       i += (long long)gridDim.x * VT) {
    const double rho = u[i], mx = u[plane + i], my = u[2 * plane + i], mz = u[3 * plane + i];
    const double bx = u[4 * plane + i], by = u[5 * plane + i], bz = u[6 * plane + i];
    const double en = u[7 * plane + i];
    const double vx = fabs(__ddiv_rn(mx, rho));
    const double vy = fabs(__ddiv_rn(my, rho));
    const double b2 = __dadd_rn(__dadd_rn(__dmul_rn(bx, bx), __dmul_rn(by, by)), __dmul_rn(bz, bz));
    const double kin = __ddiv_rn(
        __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(my, my)), __dmul_rn(mz, mz))),
        rho);
    const double pres = __dmul_rn(gm1, __dsub_rn(__dsub_rn(en, kin), __ddiv_rn(__dmul_rn(0.5, b2), mu0)));
    double a2 = __dadd_rn(__dmul_rn(gamma, pres), __ddiv_rn(b2, mu0));
    if (!(a2 != a2) && a2 < 0.0) a2 = 0.0;   // np.maximum(x, 0.0) keeps NaN
    const double cf = __dsqrt_rn(__ddiv_rn(a2, rho));
    acc[0] = nanmax(acc[0], __dadd_rn(vx, cf));
    acc[1] = nanmax(acc[1], __dadd_rn(vy, cf));
  }
  double tot[2];
  if (grid_reduce<2, true>(acc, rb, tot)) {
    rb.result[0] = tot[0];
    rb.result[1] = tot[1];
  }
}

// Start of a phi-action (leja.py:121-123): y = v, p = c0*v, ||v||, control
// block.  In-place start (y0 == null): nothing is copied -- the first term
// reads v itself as its direction and the interpolant stays "virtual" (c0 * v,
// LejaCtl::pvirt) until the first term that stores it; one read pass for ||v||.
struct LejaInitOp {
  double c0;
  double acc = 0.0;
  __device__ __forceinline__ void operator()(const double (&x)[1], double (&y)[2]) {
    y[0] = x[0];
    y[1] = __dmul_rn(c0, x[0]);
    acc = __fma_rn(x[0], x[0], acc);
  }
};

template <bool V2, bool INPLACE>
__global__ void __launch_bounds__(VT) leja_init_kernel(Ptrs<1, 2> P, long long n, LejaCtl* ctl,
                                                       const double* __restrict__ coeffs,
                                                       RedBuf rb, double* ext_sums) {
  double acc[1];
  if (INPLACE) {
    SumSqOp op;
    Ptrs<1, 0> Q;
    Q.in[0] = P.in[0];
    Q.out[0] = nullptr;
    stream<1, 0, V2>(n, Q, op);
    acc[0] = op.acc;
  } else {
    LejaInitOp op;
    op.c0 = coeffs[0];
    stream<1, 2, V2>(n, P, op);
    acc[0] = op.acc;
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) {
    if (ext_sums) ext_sums[0] = tot[0];   // y-strips: global sum first (allreduce)
    else {
      leja_init_ctl(ctl, tot[0]);
      ctl->pvirt = INPLACE ? 1 : 0;
      ctl->c0 = coeffs[0];
    }
  }
}

// One-thread control kernels of the y-strip driver: run after the allreduce of
// the per-rank partial sums, so every rank takes identical decisions.
__global__ void leja_init_finalize_kernel(LejaCtl* ctl, const double* sums) {
  leja_init_ctl(ctl, sums[0]);
}

__global__ void leja_finalize_kernel(LejaCtl* ctl, const double* sums,
                                     const double* __restrict__ coeffs) {
  if (ctl->status != LJ_RUNNING) return;
  leja_finalize(ctl, sums[0], sums[1], sums[2], sums[3] > 0.0, !ctl->zero_dir, coeffs[ctl->m]);
}

// Halo rows of the current Newton basis vector (y-strips): rows 0,1 go to the
// rank below, rows ny-2, ny-1 to the rank above; a mirror edge builds its own
// ghost rows (mhd.py:77-105: MY, BY odd).  Layout of every buffer: [field][2][nx].
__global__ void leja_pack_halo_kernel(const LejaCtl* ctl, const double* y0, const double* y1,
                                      int nx, int ny, double* send_lo, double* send_hi,
                                      double* halo_lo, double* halo_hi, int mirror_lo,
                                      int mirror_hi) {
  const double* y = ctl->cur ? y1 : y0;
  const long long plane = (long long)nx * ny;
  const int total = NF * 2 * nx;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int f = k / (2 * nx), rr = (k / nx) % 2, i = k % nx;
    const double lo = y[f * plane + (long long)rr * nx + i];               // row rr
    const double hi = y[f * plane + (long long)(ny - 2 + rr) * nx + i];    // row ny-2+rr
    if (send_lo) send_lo[k] = lo;
    if (send_hi) send_hi[k] = hi;
    const double s = (f == MY || f == BY) ? -1.0 : 1.0;
    // ghost row -2 = s*row 1, -1 = s*row 0; ny = s*row ny-1, ny+1 = s*row ny-2
    if (mirror_lo) halo_lo[k] = __dmul_rn(s, y[f * plane + (long long)(1 - rr) * nx + i]);
    if (mirror_hi) halo_hi[k] = __dmul_rn(s, y[f * plane + (long long)(ny - 1 - rr) * nx + i]);
  }
  __threadfence_system();   // the destinations may be peer memory (y-strips over NVLink)
}

template <bool V2>
__global__ void __launch_bounds__(VT) sumsq_kernel(Ptrs<1, 0> P, long long n, RedBuf rb) {
  SumSqOp op;
  stream<1, 0, V2>(n, P, op);
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = tot[0];
}

// Newton-term update for an externally supplied w = matvec(y) (leja.py:133-148).
__global__ void __launch_bounds__(VT) leja_update_kernel(const double* __restrict__ w, long long n,
                                                         LejaCtl* ctl, double* y0, double* y1,
                                                         double* p0, double* p1,
                                                         const double* __restrict__ coeffs,
                                                         const double* __restrict__ xi,
                                                         RedBuf rb) {
  if (ctl->status != LJ_RUNNING) return;
  const int cur = ctl->cur, m = ctl->m, pc = ctl->pcur;   // generic calls never defer
  const double* y = cur ? y1 : y0;
  double* yo = cur ? y0 : y1;
  const double* p = pc ? p1 : p0;
  double* po = pc ? p0 : p1;
  const double dt = ctl->dt, q = ctl->q, theta = ctl->theta;
  const double xim = xi[m - 1], cm = coeffs[m];
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double yv = y[i];
    const double wv = w ? __ldg(w + i) : 0.0;
    const double yn = __dsub_rn(__ddiv_rn(__dsub_rn(__dmul_rn(dt, wv), __dmul_rn(q, yv)), theta),
                                __dmul_rn(xim, yv));
    const double pn = __dadd_rn(p[i], __dmul_rn(cm, yn));
    yo[i] = yn;
    po[i] = pn;
    acc[0] = __fma_rn(yn, yn, acc[0]);
    acc[1] = __fma_rn(pn, pn, acc[1]);
  }
  double tot[2];
  if (grid_reduce<2, false>(acc, rb, tot)) leja_finalize(ctl, tot[0], tot[1], 0.0, 0, 0, cm);
}

// One modified Gram-Schmidt update of the Arnoldi loop (krylov.py:60-67):
// w -= c*v (NumPy's rounded product, then the subtraction), then the dot of
// the updated w with `next` (with w itself when next is null) reduced into
// *cout.  c is read from the device slot cin (the previous launch's reduced
// dot) or, when cin is null, taken from c_host.  v == null: dot only.
__global__ void __launch_bounds__(VT) mgs_kernel(double* __restrict__ w, long long n,
                                                 const double* __restrict__ v,
                                                 const double* cin, double c_host,
                                                 const double* __restrict__ next,
                                                 double* cout, RedBuf rb) {
  const double c = cin ? *cin : c_host;
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    double x = w[i];
    if (v) {
      x = __dsub_rn(x, __dmul_rn(c, __ldg(v + i)));
      w[i] = x;
    }
    const double y = next ? __ldg(next + i) : x;
    acc[0] = __fma_rn(y, x, acc[0]);
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) *cout = tot[0];
}

// out = scale * (sum_k c_k v_k), k = 0..m-1 in order (krylov.py:79-80).
__global__ void __launch_bounds__(VT) krylov_combine_kernel(double* __restrict__ out, long long n,
                                                            KrylovBasis B, int m, double scale) {
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    double s = __dmul_rn(B.c[0], __ldg(B.v[0] + i));
    for (int k = 1; k < m; ++k) s = __dadd_rn(s, __dmul_rn(B.c[k], __ldg(B.v[k] + i)));
    out[i] = __dmul_rn(scale, s);
  }
}

// Start of a peer-memory strip Leja call (one thread per rank): all-reduce of
// the local sum(v^2) in ext_sums[0], then the control-block start on the
// global sum (leja.py:121-123) -- the peer counterpart of
// leja_init_finalize_kernel.
template <bool EMUL>
__global__ void leja_p2p_init_kernel(const StencilArgs a0, const StencilArgs* args) {
  if (threadIdx.x != 0) return;
  const StencilArgs& a = EMUL ? args[blockIdx.x] : a0;
  LejaCtl* c = a.ctl;
  const double v[4] = {a.ext_sums[0], 0.0, 0.0, 0.0};
  double tot[4];
  const unsigned long long ep = c->epoch + 1;
  c->epoch = ep;
  if (p2p_allreduce4(a.p2p, ep, v, tot)) leja_init_ctl(c, tot[0]);
  else c->status = LJ_PEER_TIMEOUT;
}

// The device coefficient table now holds `to` entries: leave NEED_COEFFS
// if the loop stopped at the old end (stream order puts this between the
// term that reached the boundary and the next one).
__global__ void leja_extend_kernel(LejaCtl* ctl, int to) {
  if (ctl->ncoef < to) ctl->ncoef = to;
  if (ctl->status == LJ_NEED_COEFFS && ctl->m < ctl->ncoef) ctl->status = LJ_RUNNING;
}

// Connectivity probe: `value` into slot 0, row `rank`, of every rank's board.
__global__ void p2p_probe_kernel(const P2PArgs x, double value) {
  const int q = threadIdx.x;
  if (q < x.nranks) {
    volatile double* b = x.board[q] + x.rank * 4;
    b[0] = value;
    b[1] = (double)x.rank;
  }
  __threadfence_system();
}

// Blocks for a vector of n elements: the traversal hands out pairs.
int grid_for(long long n, int maxg) {
  long long g = ((n + 1) / 2 + VT - 1) / VT;
  if (g > maxg) g = maxg;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

cudaError_t launch_mgs(double* w, long long n, const double* v, const double* cin,
                       double c_host, const double* next, double* cout, RedBuf rb,
                       cudaStream_t s) {
  mgs_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(w, n, v, cin, c_host, next, cout, rb);
  return cudaGetLastError();
}

cudaError_t launch_krylov_combine(double* out, long long n, const KrylovBasis& B, int m,
                                  double scale, RedBuf rb, cudaStream_t s) {
  krylov_combine_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(out, n, B, m, scale);
  return cudaGetLastError();
}

cudaError_t launch_leja_p2p_init(const StencilArgs& a, cudaStream_t s) {
  leja_p2p_init_kernel<false><<<1, 32, 0, s>>>(a, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_leja_p2p_init_emul(const StencilArgs* args_dev, int nranks, cudaStream_t s) {
  StencilArgs dummy;
  memset(&dummy, 0, sizeof(dummy));
  void* kargs[] = {(void*)&dummy, (void*)&args_dev};
  return cudaLaunchCooperativeKernel((const void*)leja_p2p_init_kernel<true>, dim3(nranks),
                                     dim3(32), kargs, 0, s);
}

cudaError_t launch_leja_extend(LejaCtl* ctl, int to, cudaStream_t s) {
  leja_extend_kernel<<<1, 1, 0, s>>>(ctl, to);
  return cudaGetLastError();
}

cudaError_t launch_p2p_probe(const P2PArgs& x, double value, cudaStream_t s) {
  p2p_probe_kernel<<<1, 32, 0, s>>>(x, value);
  return cudaGetLastError();
}

cudaError_t launch_norm(const double* x, long long n, RedBuf rb, cudaStream_t s) {
  Ptrs<1, 0> P;
  P.in[0] = x;
  P.out[0] = nullptr;
  if (aligned16(P)) norm_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  else norm_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  return cudaGetLastError();
}

cudaError_t launch_lincomb(double* out, long long n, const double* const* v, const double* c,
                           int nterms, int want_norm, RedBuf rb, cudaStream_t s) {
  Coef4 cf;
  for (int k = 0; k < 4; ++k) cf.c[k] = k < nterms ? c[k] : 0.0;
  const int grid = grid_for(n, rb.grid);
  auto go = [&](auto NTc) {
    constexpr int NT = decltype(NTc)::value;
    Ptrs<NT, 1> P;
    for (int k = 0; k < NT; ++k) P.in[k] = v[k];
    P.out[0] = out;
    if (aligned16(P)) lincomb_kernel<NT, true><<<grid, VT, 0, s>>>(P, n, cf, want_norm, rb);
    else lincomb_kernel<NT, false><<<grid, VT, 0, s>>>(P, n, cf, want_norm, rb);
  };
  switch (nterms) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_lincomb_diff(double* out, double* diff, long long n, const double* const* v,
                                const double* c, int nterms, RedBuf rb, cudaStream_t s) {
  Coef4 cf;
  for (int k = 0; k < 4; ++k) cf.c[k] = k < nterms ? c[k] : 0.0;
  const int grid = grid_for(n, rb.grid);
  auto go = [&](auto NTc) {
    constexpr int NT = decltype(NTc)::value;
    Ptrs<NT, 2> P;
    for (int k = 0; k < NT; ++k) P.in[k] = v[k];
    P.out[0] = out;
    P.out[1] = diff;
    if (aligned16(P)) lincomb_diff_kernel<NT, true><<<grid, VT, 0, s>>>(P, n, cf, rb);
    else lincomb_diff_kernel<NT, false><<<grid, VT, 0, s>>>(P, n, cf, rb);
  };
  switch (nterms) {
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_lincomb_multi(double* const* out, int nout, long long n,
                                 const double* const* v, const double* coef12, RedBuf rb,
                                 cudaStream_t s) {
  MultiCoef mc;
  mc.nout = nout;
  for (int j = 0; j < 4; ++j)
    for (int k = 0; k < 3; ++k) mc.c[j][k] = j < nout ? coef12[3 * j + k] : 0.0;
  const int grid = grid_for(n, rb.grid);
  auto go = [&](auto NOc) {
    constexpr int NO = decltype(NOc)::value;
    Ptrs<3, NO> P;
    for (int k = 0; k < 3; ++k) P.in[k] = v[k];
    for (int j = 0; j < NO; ++j) P.out[j] = out[j];
    if (aligned16(P)) lincomb_multi_kernel<NO, true><<<grid, VT, 0, s>>>(P, n, mc);
    else lincomb_multi_kernel<NO, false><<<grid, VT, 0, s>>>(P, n, mc);
  };
  switch (nout) {
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_final_pair(int kind, double* out_hi, long long n, const double* const* v,
                              const double* c, RedBuf rb, cudaStream_t s) {
  Coef6 cf;
  for (int k = 0; k < 6; ++k) cf.c[k] = c[k];
  const int grid = grid_for(n, rb.grid);
  if (kind == 43) {
    Ptrs<4, 1> P;
    for (int k = 0; k < 4; ++k) P.in[k] = v[k];
    P.out[0] = out_hi;
    if (aligned16(P)) final_pair_kernel<43, true><<<grid, VT, 0, s>>>(P, n, cf, rb);
    else final_pair_kernel<43, false><<<grid, VT, 0, s>>>(P, n, cf, rb);
  } else if (kind == 54) {
    Ptrs<6, 1> P;
    for (int k = 0; k < 6; ++k) P.in[k] = v[k];
    P.out[0] = out_hi;
    if (aligned16(P)) final_pair_kernel<54, true><<<grid, VT, 0, s>>>(P, n, cf, rb);
    else final_pair_kernel<54, false><<<grid, VT, 0, s>>>(P, n, cf, rb);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_divide(double* out, const double* x, double d, long long n, int want_norm,
                          RedBuf rb, cudaStream_t s) {
  Ptrs<1, 1> P;
  P.in[0] = x;
  P.out[0] = out;
  if (aligned16(P)) divide_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, d, n, want_norm, rb);
  else divide_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, d, n, want_norm, rb);
  return cudaGetLastError();
}

struct FillOp {
  double v;
  __device__ __forceinline__ void operator()(const double (&)[1], double (&y)[1]) { y[0] = v; }
};

template <bool V2>
__global__ void __launch_bounds__(VT) fill_kernel(Ptrs<0, 1> P, long long n, double v) {
  FillOp op;
  op.v = v;
  stream<0, 1, V2>(n, P, op);
}

cudaError_t launch_fill(double* x, long long n, double v, cudaStream_t s) {
  Ptrs<0, 1> P;
  P.in[0] = nullptr;
  P.out[0] = x;
  if (aligned16(P)) fill_kernel<true><<<grid_for(n, 4 * 148), VT, 0, s>>>(P, n, v);
  else fill_kernel<false><<<grid_for(n, 4 * 148), VT, 0, s>>>(P, n, v);
  return cudaGetLastError();
}

// The interpolant of a finished call into `out`: pbuf[pcur] (c0 * v while it
// is still virtual), plus pend_coef * ybuf[cur] when a term is pending (p + c*y,
// leja.py:140).
struct CopyResultOp {
  int pend, pvirt;
  double c, c0;
  __device__ __forceinline__ void operator()(const double (&x)[2], double (&y)[1]) {
    const double p = pvirt ? __dmul_rn(c0, x[0]) : x[0];
    y[0] = pend ? __dadd_rn(p, __dmul_rn(c, x[1])) : p;
  }
};

template <bool V2>
__global__ void __launch_bounds__(VT) leja_copy_result_kernel(double* out, const double* p0,
                                                              const double* p1, const double* y0,
                                                              const double* y1, const double* v0,
                                                              const LejaCtl* ctl, long long n) {
  CopyResultOp op;
  op.pend = ctl->ppend;
  op.pvirt = ctl->pvirt;
  op.c = ctl->pend_coef;
  op.c0 = ctl->c0;
  Ptrs<2, 1> P;
  P.in[0] = op.pvirt ? v0 : (ctl->pcur ? p1 : p0);
  // the pending term's y is the current direction (v itself before any term ran)
  P.in[1] = (v0 && ctl->m == 1 && ctl->cur == 0) ? v0 : (ctl->cur ? y1 : y0);
  P.out[0] = out;
  stream<2, 1, V2>(n, P, op);
}

cudaError_t launch_leja_copy_result(double* p_out, const double* const* pbuf,
                                    const double* const* ybuf, const double* v0,
                                    const LejaCtl* ctl, long long n, cudaStream_t s) {
  const unsigned long long bits = (unsigned long long)p_out | (unsigned long long)pbuf[0] |
                                  (unsigned long long)pbuf[1] | (unsigned long long)ybuf[0] |
                                  (unsigned long long)ybuf[1] | (unsigned long long)v0;
  if ((bits & 15ull) == 0)
    leja_copy_result_kernel<true><<<grid_for(n, 4 * 148), VT, 0, s>>>(
        p_out, pbuf[0], pbuf[1], ybuf[0], ybuf[1], v0, ctl, n);
  else
    leja_copy_result_kernel<false><<<grid_for(n, 4 * 148), VT, 0, s>>>(
        p_out, pbuf[0], pbuf[1], ybuf[0], ybuf[1], v0, ctl, n);
  return cudaGetLastError();
}

// jvp prologue (linearize.py:62-65) without a host round trip.
template <bool V2>
__global__ void __launch_bounds__(VT) jvp_prep_kernel(Ptrs<1, 0> P, long long n, double unorm,
                                                      PowerCtl* jc, RedBuf rb) {
  SumSqOp op;
  stream<1, 0, V2>(n, P, op);
  double acc[1] = {op.acc}, tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) {
    jc->stop = 0;
    jc->status = PW_RUNNING;
    jc->unorm = unorm;
    power_after_divide(jc, tot[0]);   // wn == 0 -> PW_ZERO, else the FD step
  }
}

cudaError_t launch_jvp_prep(const double* w, long long n, double unorm, PowerCtl* jc, RedBuf rb,
                            cudaStream_t s) {
  Ptrs<1, 0> P;
  P.in[0] = w;
  P.out[0] = nullptr;
  if (aligned16(P)) jvp_prep_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, unorm, jc, rb);
  else jvp_prep_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, unorm, jc, rb);
  return cudaGetLastError();
}

cudaError_t launch_power_divide(double* out, const double* x, long long n, PowerCtl* pctl,
                                RedBuf rb, cudaStream_t s) {
  Ptrs<1, 1> P;
  P.in[0] = x;
  P.out[0] = out;
  if (aligned16(P)) power_divide_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, pctl, rb);
  else power_divide_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, pctl, rb);
  return cudaGetLastError();
}

cudaError_t launch_diffnorm(const double* a, const double* b, long long n, RedBuf rb,
                            cudaStream_t s) {
  Ptrs<2, 0> P;
  P.in[0] = a;
  P.in[1] = b;
  P.out[0] = nullptr;
  if (aligned16(P)) diffnorm_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  else diffnorm_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  return cudaGetLastError();
}

cudaError_t launch_divb_max(const Geom& g, const double* u, double* field, RedBuf rb,
                            cudaStream_t s) {
  divb_kernel<<<grid_for(g.plane, rb.grid), VT, 0, s>>>(g, u, field, rb);
  return cudaGetLastError();
}

cudaError_t launch_field_sums(const double* u, long long plane, RedBuf rb, cudaStream_t s) {
  const int gx = grid_for(plane, rb.grid / 2);
  field_sum_kernel<<<dim3(gx, 2), VT, 0, s>>>(u, plane, rb);
  return cudaGetLastError();
}

cudaError_t launch_cfl(const double* u, long long plane, double gamma, double mu0, RedBuf rb,
                       cudaStream_t s) {
  cfl_kernel<<<grid_for(plane, rb.grid), VT, 0, s>>>(u, plane, gamma, mu0, rb);
  return cudaGetLastError();
}

cudaError_t launch_leja_init(const double* v, long long n, double* y0, double* p0, LejaCtl* ctl,
                             const double* coeffs, RedBuf rb, cudaStream_t s, double* ext_sums) {
  Ptrs<1, 2> P;
  P.in[0] = v;
  P.out[0] = y0;
  P.out[1] = p0;
  const int grid = grid_for(n, rb.grid);
  const bool v2 = aligned16(P);
  if (!y0) {   // in-place start: ||v|| only
    if (v2) leja_init_kernel<true, true><<<grid, VT, 0, s>>>(P, n, ctl, coeffs, rb, ext_sums);
    else leja_init_kernel<false, true><<<grid, VT, 0, s>>>(P, n, ctl, coeffs, rb, ext_sums);
  } else {
    if (v2) leja_init_kernel<true, false><<<grid, VT, 0, s>>>(P, n, ctl, coeffs, rb, ext_sums);
    else leja_init_kernel<false, false><<<grid, VT, 0, s>>>(P, n, ctl, coeffs, rb, ext_sums);
  }
  return cudaGetLastError();
}

cudaError_t launch_leja_init_finalize(LejaCtl* ctl, const double* sums, cudaStream_t s) {
  leja_init_finalize_kernel<<<1, 1, 0, s>>>(ctl, sums);
  return cudaGetLastError();
}

cudaError_t launch_leja_finalize(LejaCtl* ctl, const double* sums, const double* coeffs,
                                 cudaStream_t s) {
  leja_finalize_kernel<<<1, 1, 0, s>>>(ctl, sums, coeffs);
  return cudaGetLastError();
}

cudaError_t launch_leja_pack_halo(const LejaCtl* ctl, const double* y0, const double* y1, int nx,
                                  int ny, double* send_lo, double* send_hi, double* halo_lo,
                                  double* halo_hi, int mirror_lo, int mirror_hi, cudaStream_t s) {
  const int total = NF * 2 * nx;
  const int grid = (total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024;
  leja_pack_halo_kernel<<<grid, 256, 0, s>>>(ctl, y0, y1, nx, ny, send_lo, send_hi, halo_lo,
                                             halo_hi, mirror_lo, mirror_hi);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const double* x, long long n, RedBuf rb, cudaStream_t s) {
  Ptrs<1, 0> P;
  P.in[0] = x;
  P.out[0] = nullptr;
  if (aligned16(P)) sumsq_kernel<true><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  else sumsq_kernel<false><<<grid_for(n, rb.grid), VT, 0, s>>>(P, n, rb);
  return cudaGetLastError();
}

cudaError_t launch_leja_update(const double* w, long long n, LejaCtl* ctl, double* const* ybuf,
                               double* const* pbuf, const double* coeffs, const double* xi,
                               RedBuf rb, cudaStream_t s) {
  leja_update_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(w, n, ctl, ybuf[0], ybuf[1], pbuf[0],
                                                          pbuf[1], coeffs, xi, rb);
  return cudaGetLastError();
}

}  // namespace xb

// ---------------------------------------------------------------------------
// Non-finite cell scan of an RHS output (failure path of xmhd_rhs / xmhd_jvp /
// xmhd_leja): the count of non-finite entries and the smallest flat index
// above `after` (C order (field, j, i) of mhd.py:225-231).  One pass per
// reported cell; only runs after a kernel already flagged the output.
namespace xb {

__global__ void __launch_bounds__(VT) nonfinite_scan_kernel(const double* __restrict__ f,
                                                             long long n, long long after,
                                                             unsigned long long* minidx,
                                                             unsigned long long* count) {
  unsigned long long cnt = 0, best = ~0ull;
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const unsigned hi = (unsigned)__double2hiint(__ldg(f + i));
    if ((hi & 0x7ff00000u) == 0x7ff00000u) {
      ++cnt;
      if (i > after && (unsigned long long)i < best) best = (unsigned long long)i;
    }
  }
  if (count && cnt) atomicAdd(count, cnt);
  if (best != ~0ull) atomicMin(minidx, best);
}

cudaError_t launch_nonfinite_scan(const double* f, long long n, long long after,
                                  unsigned long long* minidx, unsigned long long* count,
                                  cudaStream_t s) {
  nonfinite_scan_kernel<<<grid_for(n, 4 * 148), VT, 0, s>>>(f, n, after, minidx, count);
  return cudaGetLastError();
}

}  // namespace xb
