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

__global__ void __launch_bounds__(VT) norm_kernel(const double* __restrict__ x, long long n,
                                                  RedBuf rb) {
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double v = __ldg(x + i);
    acc[0] = __fma_rn(v, v, acc[0]);
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = sqrt(tot[0]);
}

struct Lin4 {
  const double* v[4];
  double c[4];
  int nterms;
};

__global__ void __launch_bounds__(VT) lincomb_kernel(double* __restrict__ out, long long n,
                                                     Lin4 L, int want_norm, RedBuf rb) {
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    double s = __dmul_rn(L.c[0], __ldg(L.v[0] + i));
    if (L.nterms > 1) s = __dadd_rn(s, __dmul_rn(L.c[1], __ldg(L.v[1] + i)));
    if (L.nterms > 2) s = __dadd_rn(s, __dmul_rn(L.c[2], __ldg(L.v[2] + i)));
    if (L.nterms > 3) s = __dadd_rn(s, __dmul_rn(L.c[3], __ldg(L.v[3] + i)));
    out[i] = s;
    acc[0] = __fma_rn(s, s, acc[0]);
    if (!isfinite(s)) acc[1] = 1.0;
  }
  if (!want_norm) return;
  double tot[2];
  if (grid_reduce<2, false>(acc, rb, tot)) {
    rb.result[0] = sqrt(tot[0]);
    rb.result[1] = tot[1] > 0.0 ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(VT) divide_kernel(double* __restrict__ out,
                                                    const double* __restrict__ x, double d,
                                                    long long n, int want_norm, RedBuf rb) {
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double q = __ddiv_rn(__ldg(x + i), d);
    out[i] = q;
    acc[0] = __fma_rn(q, q, acc[0]);
  }
  if (!want_norm) return;
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) rb.result[0] = sqrt(tot[0]);
}

// One division of the device power iteration (linearize.py:115-116, 124):
// out = x / div, then ||out|| and the next FD step in the last block.
__global__ void __launch_bounds__(VT) power_divide_kernel(double* __restrict__ out,
                                                          const double* __restrict__ x,
                                                          long long n, PowerCtl* pc, RedBuf rb) {
  if (pc->status != PW_RUNNING) return;
  const double d = pc->div;
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double q = __ddiv_rn(__ldg(x + i), d);
    out[i] = q;
    acc[0] = __fma_rn(q, q, acc[0]);
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) power_after_divide(pc, tot[0]);
}

__global__ void __launch_bounds__(VT) diffnorm_kernel(const double* __restrict__ a,
                                                      const double* __restrict__ b,
                                                      long long n, RedBuf rb) {
  double acc[2] = {0.0, 0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double bv = __ldg(b + i);
    const double d = __dsub_rn(__ldg(a + i), bv);
    acc[0] = __fma_rn(d, d, acc[0]);
    acc[1] = __fma_rn(bv, bv, acc[1]);
  }
  double tot[2];
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

// y = v (copy), p = c0*v, ||v|| -> control block (leja.py:121-123).
__global__ void __launch_bounds__(VT) leja_init_kernel(const double* __restrict__ v, long long n,
                                                       double* __restrict__ y0,
                                                       double* __restrict__ p0, LejaCtl* ctl,
                                                       const double* __restrict__ coeffs,
                                                       RedBuf rb, double* ext_sums) {
  const double c0 = coeffs[0];
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double x = __ldg(v + i);
    y0[i] = x;
    p0[i] = __dmul_rn(c0, x);
    acc[0] = __fma_rn(x, x, acc[0]);
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) {
    if (ext_sums) ext_sums[0] = tot[0];   // y-strips: global sum first (allreduce)
    else leja_init_ctl(ctl, tot[0]);
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

__global__ void __launch_bounds__(VT) sumsq_kernel(const double* __restrict__ x, long long n,
                                                   RedBuf rb) {
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double v = __ldg(x + i);
    acc[0] = __fma_rn(v, v, acc[0]);
  }
  double tot[1];
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

int grid_for(long long n, int maxg) {
  long long g = (n + VT - 1) / VT;
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
  norm_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(x, n, rb);
  return cudaGetLastError();
}

cudaError_t launch_lincomb(double* out, long long n, const double* const* v, const double* c,
                           int nterms, int want_norm, RedBuf rb, cudaStream_t s) {
  Lin4 L;
  L.nterms = nterms;
  for (int k = 0; k < 4; ++k) {
    L.v[k] = k < nterms ? v[k] : nullptr;
    L.c[k] = k < nterms ? c[k] : 0.0;
  }
  lincomb_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(out, n, L, want_norm, rb);
  return cudaGetLastError();
}

cudaError_t launch_divide(double* out, const double* x, double d, long long n, int want_norm,
                          RedBuf rb, cudaStream_t s) {
  divide_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(out, x, d, n, want_norm, rb);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(VT) fill_kernel(double* __restrict__ x, long long n, double v) {
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT)
    x[i] = v;
}

cudaError_t launch_fill(double* x, long long n, double v, cudaStream_t s) {
  fill_kernel<<<grid_for(n, 4 * 148), VT, 0, s>>>(x, n, v);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(VT) leja_copy_result_kernel(double* __restrict__ out,
                                                              const double* p0, const double* p1,
                                                              const double* y0, const double* y1,
                                                              const LejaCtl* ctl, long long n) {
  const double* __restrict__ src = ctl->pcur ? p1 : p0;
  const double* __restrict__ y = ctl->cur ? y1 : y0;
  const int pend = ctl->ppend;
  const double c = ctl->pend_coef;
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT)
    out[i] = pend ? __dadd_rn(src[i], __dmul_rn(c, y[i])) : src[i];   // p + c*y (leja.py:140)
}

cudaError_t launch_leja_copy_result(double* p_out, const double* const* pbuf,
                                    const double* const* ybuf, const LejaCtl* ctl, long long n,
                                    cudaStream_t s) {
  leja_copy_result_kernel<<<grid_for(n, 4 * 148), VT, 0, s>>>(p_out, pbuf[0], pbuf[1], ybuf[0],
                                                               ybuf[1], ctl, n);
  return cudaGetLastError();
}

// jvp prologue (linearize.py:62-65) without a host round trip.
__global__ void __launch_bounds__(VT) jvp_prep_kernel(const double* __restrict__ w, long long n,
                                                      double unorm, PowerCtl* jc, RedBuf rb) {
  double acc[1] = {0.0};
  for (long long i = (long long)blockIdx.x * VT + threadIdx.x; i < n;
       i += (long long)gridDim.x * VT) {
    const double v = __ldg(w + i);
    acc[0] = __fma_rn(v, v, acc[0]);
  }
  double tot[1];
  if (grid_reduce<1, false>(acc, rb, tot)) {
    jc->stop = 0;
    jc->status = PW_RUNNING;
    jc->unorm = unorm;
    power_after_divide(jc, tot[0]);   // wn == 0 -> PW_ZERO, else the FD step
  }
}

cudaError_t launch_jvp_prep(const double* w, long long n, double unorm, PowerCtl* jc, RedBuf rb,
                            cudaStream_t s) {
  jvp_prep_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(w, n, unorm, jc, rb);
  return cudaGetLastError();
}

cudaError_t launch_power_divide(double* out, const double* x, long long n, PowerCtl* pctl,
                                RedBuf rb, cudaStream_t s) {
  power_divide_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(out, x, n, pctl, rb);
  return cudaGetLastError();
}

cudaError_t launch_diffnorm(const double* a, const double* b, long long n, RedBuf rb,
                            cudaStream_t s) {
  diffnorm_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(a, b, n, rb);
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
  leja_init_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(v, n, y0, p0, ctl, coeffs, rb, ext_sums);
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
  sumsq_kernel<<<grid_for(n, rb.grid), VT, 0, s>>>(x, n, rb);
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
