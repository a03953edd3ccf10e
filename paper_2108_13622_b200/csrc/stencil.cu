// Fused fp64 resistive-MHD stencil for sm_100a: RHS, FD-JVP and the fused
// Leja/Newton iteration in one pass over HBM.
//
// Reference path (arxiv/paper_2108_13622, pkg/src/xmhd):
//   mhd_rhs            mhd.py:127-232   (MODE_RHS)
//   jvp                linearize.py:56-67 (MODE_JVP: x = u + eps*w, (F(x) - F(u))/eps)
//   apply_phi_leja     leja.py:133-148  (MODE_LEJA: the JVP above plus
//                      y' = ((dt*w) - (q*y))/theta - xi*y, p' = p + c*y',
//                      ||y'||, ||p'|| and the convergence control, on device)
//
// Data layout: the reference's flat field-major (8, ny, nx) fp64 vector.
//
// Dataflow (one CTA = one y-segment of one column strip, sliding window):
//   CTA of SW=128 threads owns ghost-extended columns [X0-2, X0+126) and marches
//   the rows r = Y0-2 .. Y1+1.  Per row step:
//     P1  thread t forms x(r, c_t) (= u or u + eps*y, with boundary mirror /
//         wrap), computes the primitives once, stores the 8 differentiated
//         primitives (PD) and the 7 ideal x-fluxes (FX) in shared-memory rings
//         and keeps its 7 ideal y-fluxes (FY) in registers;
//     P2  level-1 derivatives at row r-1 (PD of rows r-2, r-1, r) -> diffusive
//         fluxes GX (shared ring) and GY (registers);
//     P3  output row r-2: centred differences of FX, FY, GX, GY in the
//         reference's association order, then the mode epilogue.
//   Every primitive / flux is evaluated once per cell (plus the 4-column and
//   4-row halo of each CTA), so the kernel streams u, y, F(u), p once and
//   writes y', p' once: 384 B per cell per Leja iteration.
#include <cfloat>
#include <climits>
#include "kernels.h"

namespace xb {

namespace {

// Slot -> field maps for the non-zero flux rows (compile-time in unrolled loops).
__host__ __device__ constexpr int fx_field(int k) { return k < 4 ? k : k + 1; }          // skip BX
__host__ __device__ constexpr int fy_field(int k) { return k < 5 ? k : k + 1; }          // skip BY

struct RowSrc {
  const double* u;     // row base of field 0 in the base state
  const double* d;     // row base of field 0 in the direction vector
  long long fs;        // stride between fields
  int flip;            // mirror ghost row: negate MY, BY
};

__device__ __forceinline__ RowSrc row_source(int r, const Geom& g, const double* u,
                                             const double* d) {
  RowSrc s;
  s.flip = 0;
  s.fs = g.plane;
  int rr = r;
  if (g.bcy == BC_PERIODIC) {
    rr = r % g.ny;
    if (rr < 0) rr += g.ny;
  } else if (g.bcy == BC_REFLECT) {
    if (r < 0) { rr = -1 - r; s.flip = 1; }
    else if (r >= g.ny) { rr = 2 * g.ny - 1 - r; s.flip = 1; }
    rr = min(max(rr, 0), g.ny - 1);
  } else {  // BC_HALO: rows owned by the y-neighbours, [field][2][nx]
    if (r < 0) {
      s.u = g.halo_lo + (long long)(r + 2) * g.nx;
      s.d = g.halo_lo_dir ? g.halo_lo_dir + (long long)(r + 2) * g.nx : nullptr;
      s.fs = 2LL * g.nx;
      return s;
    }
    if (r >= g.ny) {
      s.u = g.halo_hi + (long long)(r - g.ny) * g.nx;
      s.d = g.halo_hi_dir ? g.halo_hi_dir + (long long)(r - g.ny) * g.nx : nullptr;
      s.fs = 2LL * g.nx;
      return s;
    }
  }
  s.u = u + (long long)rr * g.nx;
  s.d = d ? d + (long long)rr * g.nx : nullptr;
  return s;
}

__device__ __forceinline__ void col_source(int cg, const Geom& g, int& cs, int& flip) {
  flip = 0;
  if (g.bcx == BC_PERIODIC) {
    cs = cg % g.nx;
    if (cs < 0) cs += g.nx;
  } else {
    cs = cg;
    if (cg < 0) { cs = -1 - cg; flip = 1; }
    else if (cg >= g.nx) { cs = 2 * g.nx - 1 - cg; flip = 1; }
    cs = min(max(cs, 0), g.nx - 1);
  }
}

// Deterministic block sum (fixed shuffle tree + fixed warp order); valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
  return s;
}

// Deterministic sum of per-block partials (called by one full warp).
__device__ __forceinline__ double sum_partials(const double* p, int nblk, int stride, int k) {
  const int l = threadIdx.x & 31;
  double s = 0.0;
  for (int b = l; b < nblk; b += 32) s += __ldcg(p + (long long)b * stride + k);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return __shfl_sync(0xffffffffu, s, 0);
}

}  // namespace

template <int MODE>
__global__ void __launch_bounds__(SW, 2) stencil_kernel(const StencilArgs a) {
  extern __shared__ double smem[];
  double (*pd)[NPD][SW] = reinterpret_cast<double (*)[NPD][SW]>(smem);
  double (*fxs)[NFX][SW] = reinterpret_cast<double (*)[NFX][SW]>(smem + 3 * NPD * SW);
  double (*gxs)[NG][SW] = reinterpret_cast<double (*)[NG][SW]>(smem + 3 * NPD * SW + 3 * NFX * SW);
  __shared__ double red[SW / 32];
  __shared__ int am_last;

  const Geom& g = a.g;
  const int t = threadIdx.x;

  // Per-launch scalars.
  double eps = a.eps;
  const double* dir = a.dir;
  double* yout = nullptr;
  const double* pin = nullptr;
  double* pout = nullptr;
  double dt = 0.0, q = 0.0, theta = 1.0, xim = 0.0, cm = 0.0;
  int zero_dir = 0;
  if (MODE == MODE_LEJA) {
    const LejaCtl* c = a.ctl;
    if (c->status != LJ_RUNNING) return;
    const int cur = c->cur, m = c->m;
    eps = c->eps;
    zero_dir = c->zero_dir;
    dir = a.ybuf[cur];
    yout = a.ybuf[cur ^ 1];
    pin = a.pbuf[cur];
    pout = a.pbuf[cur ^ 1];
    dt = c->dt;
    q = c->q;
    theta = c->theta;
    xim = __ldg(a.xi + (m - 1));
    cm = __ldg(a.coeffs + m);
  }

  double acc0 = 0.0, acc1 = 0.0;
  int bad = 0;

  if (MODE == MODE_LEJA && zero_dir) {
    // jvp of a zero vector is exactly zero and costs no RHS call (linearize.py:63-64)
    const long long n = (long long)NF * g.plane;
    for (long long i = (long long)blockIdx.x * SW + t; i < n; i += (long long)gridDim.x * SW) {
      const double y = dir[i];
      const double yn = __dsub_rn(__ddiv_rn(__dsub_rn(__dmul_rn(dt, 0.0), __dmul_rn(q, y)), theta),
                                  __dmul_rn(xim, y));
      const double pn = __dadd_rn(pin[i], __dmul_rn(cm, yn));
      yout[i] = yn;
      pout[i] = pn;
      acc0 = __fma_rn(yn, yn, acc0);
      acc1 = __fma_rn(pn, pn, acc1);
    }
  } else {
    for (int unit = blockIdx.x; unit < a.nunits; unit += gridDim.x) {
      const int ux = unit % a.units_x, uy = unit / a.units_x;
      const int X0 = ux * SOUT;
      const int Y0 = uy * a.seg_rows;
      const int Y1 = min(Y0 + a.seg_rows, g.ny);
      const int cg = X0 - 2 + t;
      int cs, flipx;
      col_source(cg, g, cs, flipx);
      const int c_out = X0 + t - 2;
      const bool col_ok = (t >= 2) && (t < SW - 2) && (c_out < g.nx);
      const int tl = max(t - 1, 0), tr = min(t + 1, SW - 1);

      double fy1[NFY], fy2[NFY], fy3[NFY], gy1[NG], gy2[NG];
#pragma unroll
      for (int k = 0; k < NFY; ++k) fy1[k] = fy2[k] = fy3[k] = 0.0;
#pragma unroll
      for (int k = 0; k < NG; ++k) gy1[k] = gy2[k] = 0.0;

      const int nsteps = (Y1 - Y0) + 4;
      int s3 = 0;  // s % 3
      for (int s = 0; s < nsteps; ++s) {
        const int r = Y0 - 2 + s;
        const int m1 = (s3 + 2) % 3;  // ring slot of row r-1
        const int m2 = (s3 + 1) % 3;  // ring slot of row r-2

        // ---- P1: state at (r, cg), primitives, PD + FX to smem, FY to regs
        double fyn[NFY];
        {
          const RowSrc rs = row_source(r, g, a.u, MODE == MODE_RHS ? nullptr : dir);
          double x[NF];
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            double v = __ldg(rs.u + f * rs.fs + cs);
            if (MODE != MODE_RHS) v = __dadd_rn(v, __dmul_rn(eps, __ldg(rs.d + f * rs.fs + cs)));
            x[f] = v;
          }
          if (flipx) { x[MX] = -x[MX]; x[BX] = -x[BX]; }
          if (rs.flip) { x[MY] = -x[MY]; x[BY] = -x[BY]; }
          Prim p;
          primitives(x, g, p);
          pd[s3][PD_VX][t] = p.vx;
          pd[s3][PD_VY][t] = p.vy;
          pd[s3][PD_VZ][t] = p.vz;
          pd[s3][PD_BX][t] = p.bx;
          pd[s3][PD_BY][t] = p.by;
          pd[s3][PD_BZ][t] = p.bz;
          pd[s3][PD_T][t] = p.temp;
          pd[s3][PD_B2][t] = p.b2;
          double fxv[NFX];
          flux_x(p, g, fxv);
#pragma unroll
          for (int k = 0; k < NFX; ++k) fxs[s3][k][t] = fxv[k];
          flux_y(p, g, fyn);
        }
        __syncthreads();

        // ---- P2: diffusive fluxes at row r-1
        double gyn[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) gyn[k] = 0.0;
        if (g.diffusive && s >= 2) {
          double xl[NPD], xr[NPD], yd[NPD], yu[NPD], own[NPD];
#pragma unroll
          for (int k = 0; k < NPD; ++k) {
            xl[k] = pd[m1][k][tl];
            xr[k] = pd[m1][k][tr];
            yd[k] = pd[m2][k][t];
            yu[k] = pd[s3][k][t];
            own[k] = pd[m1][k][t];
          }
          double gxv[NG];
          diffusive_fluxes(xl, xr, yd, yu, own, g, gxv, gyn);
#pragma unroll
          for (int k = 0; k < NG; ++k) gxs[(s + 1) & 1][k][t] = gxv[k];
        }
        __syncthreads();

        // ---- P3: output row o = r-2
        if (s >= 4 && col_ok) {
          const int o = r - 2;
          const int gs = s & 1;  // GX ring slot of row r-2
          double F[NF];
          // ideal part: out = -(dFX/2dx); out -= dFY/2dy       (mhd.py:177-178)
#pragma unroll
          for (int k = 0; k < NFX; ++k) {
            const int f = fx_field(k);
            F[f] = -exact_div(__dsub_rn(fxs[m2][k][tr], fxs[m2][k][tl]), g.h2x);
          }
          F[BX] = -0.0;
#pragma unroll
          for (int k = 0; k < NFY; ++k) {
            const int f = fy_field(k);
            F[f] = __dsub_rn(F[f], exact_div(__dsub_rn(fy1[k], fy3[k]), g.h2y));
          }
          F[BY] = __dsub_rn(F[BY], 0.0);
          if (g.diffusive) {
            // out += dGX/2dx; out += dGY/2dy                 (mhd.py:222-223)
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BX] = __dadd_rn(F[BX], 0.0);
            F[MX] = __dadd_rn(F[MX], exact_div(__dsub_rn(gxs[gs][0][tr], gxs[gs][0][tl]), g.h2x));
            F[MY] = __dadd_rn(F[MY], exact_div(__dsub_rn(gxs[gs][1][tr], gxs[gs][1][tl]), g.h2x));
            F[MZ] = __dadd_rn(F[MZ], exact_div(__dsub_rn(gxs[gs][2][tr], gxs[gs][2][tl]), g.h2x));
            F[BY] = __dadd_rn(F[BY], exact_div(__dsub_rn(gxs[gs][3][tr], gxs[gs][3][tl]), g.h2x));
            F[BZ] = __dadd_rn(F[BZ], exact_div(__dsub_rn(gxs[gs][4][tr], gxs[gs][4][tl]), g.h2x));
            F[EN] = __dadd_rn(F[EN], exact_div(__dsub_rn(gxs[gs][5][tr], gxs[gs][5][tl]), g.h2x));
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BY] = __dadd_rn(F[BY], 0.0);
            F[MX] = __dadd_rn(F[MX], exact_div(__dsub_rn(gyn[0], gy2[0]), g.h2y));
            F[MY] = __dadd_rn(F[MY], exact_div(__dsub_rn(gyn[1], gy2[1]), g.h2y));
            F[MZ] = __dadd_rn(F[MZ], exact_div(__dsub_rn(gyn[2], gy2[2]), g.h2y));
            F[BX] = __dadd_rn(F[BX], exact_div(__dsub_rn(gyn[3], gy2[3]), g.h2y));
            F[BZ] = __dadd_rn(F[BZ], exact_div(__dsub_rn(gyn[4], gy2[4]), g.h2y));
            F[EN] = __dadd_rn(F[EN], exact_div(__dsub_rn(gyn[5], gy2[5]), g.h2y));
          }
          const long long base = (long long)o * g.nx + c_out;
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const long long i = base + f * g.plane;
            if (!isfinite(F[f])) bad = 1;
            if (MODE == MODE_RHS) {
              a.out[i] = F[f];
            } else if (MODE == MODE_JVP) {
              const double jv = __ddiv_rn(__dsub_rn(F[f], __ldg(a.fu + i)), eps);
              a.out[i] = jv;
              acc0 = __fma_rn(jv, jv, acc0);
            } else {
              const double w = __ddiv_rn(__dsub_rn(F[f], __ldg(a.fu + i)), eps);
              const double y = dir[i];
              const double yn = __dsub_rn(
                  __ddiv_rn(__dsub_rn(__dmul_rn(dt, w), __dmul_rn(q, y)), theta),
                  __dmul_rn(xim, y));
              const double pn = __dadd_rn(pin[i], __dmul_rn(cm, yn));
              yout[i] = yn;
              pout[i] = pn;
              acc0 = __fma_rn(yn, yn, acc0);
              acc1 = __fma_rn(pn, pn, acc1);
            }
          }
        }
        __syncthreads();

#pragma unroll
        for (int k = 0; k < NFY; ++k) { fy3[k] = fy2[k]; fy2[k] = fy1[k]; fy1[k] = fyn[k]; }
#pragma unroll
        for (int k = 0; k < NG; ++k) { gy2[k] = gy1[k]; gy1[k] = gyn[k]; }
        s3 = (s3 == 2) ? 0 : s3 + 1;
      }
    }
  }

  if (bad) atomicOr(a.bad, 1);
  if (MODE == MODE_RHS) return;

  const double s0 = block_sum(acc0, red);
  const double s1 = (MODE == MODE_LEJA) ? block_sum(acc1, red) : 0.0;
  if (t == 0) {
    a.partials[2 * blockIdx.x] = s0;
    a.partials[2 * blockIdx.x + 1] = s1;
    __threadfence();
    const unsigned prev = atomicAdd(a.ticket, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  if (t < 32) {
    const double sy = sum_partials(a.partials, gridDim.x, 2, 0);
    const double sp = (MODE == MODE_LEJA) ? sum_partials(a.partials, gridDim.x, 2, 1) : 0.0;
    if (t == 0) {
      if (MODE == MODE_JVP) {
        a.result[0] = sqrt(sy);
      } else {
        const int flag = *((volatile int*)a.bad);
        leja_finalize(a.ctl, sy, sp, flag, !zero_dir, cm);
      }
      *a.ticket = 0u;
    }
  }
}

size_t stencil_smem_bytes() {
  return sizeof(double) * (size_t)SW * (3 * NPD + 3 * NFX + 2 * NG);
}

// Work decomposition: column strips of SOUT outputs x y-segments; the
// persistent grid is 2 CTAs per SM.  The segment length trades warm-up rows
// (4 per segment) against wave quantisation of the units over the grid.
void stencil_plan(const Geom& g, int nsm, int& units_x, int& nunits, int& seg_rows, int& grid) {
  units_x = (g.nx + SOUT - 1) / SOUT;
  const int slots = 2 * nsm;
  double best = 1e300;
  int best_seg = g.ny;
  for (int seg = 8; seg <= g.ny + 8; seg += (seg < 64 ? 1 : 8)) {
    const int s = seg > g.ny ? g.ny : seg;
    const int nseg = (g.ny + s - 1) / s;
    const long long units = (long long)units_x * nseg;
    const long long waves = (units + slots - 1) / slots;
    const double cost = (double)waves * (s + 4);
    if (cost < best - 1e-9) { best = cost; best_seg = s; }
    if (seg > g.ny) break;
  }
  seg_rows = best_seg;
  nunits = units_x * ((g.ny + seg_rows - 1) / seg_rows);
  grid = nunits < slots ? nunits : slots;
}

cudaError_t launch_stencil(int mode, const StencilArgs& a, int grid, cudaStream_t s) {
  static bool attr_done[3] = {false, false, false};
  const size_t smem = stencil_smem_bytes();
  cudaError_t err = cudaSuccess;
  switch (mode) {
    case MODE_RHS:
      if (!attr_done[0]) {
        err = cudaFuncSetAttribute(stencil_kernel<MODE_RHS>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        attr_done[0] = true;
      }
      stencil_kernel<MODE_RHS><<<grid, SW, smem, s>>>(a);
      break;
    case MODE_JVP:
      if (!attr_done[1]) {
        err = cudaFuncSetAttribute(stencil_kernel<MODE_JVP>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        attr_done[1] = true;
      }
      stencil_kernel<MODE_JVP><<<grid, SW, smem, s>>>(a);
      break;
    default:
      if (!attr_done[2]) {
        err = cudaFuncSetAttribute(stencil_kernel<MODE_LEJA>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        attr_done[2] = true;
      }
      stencil_kernel<MODE_LEJA><<<grid, SW, smem, s>>>(a);
      break;
  }
  return cudaGetLastError();
}

}  // namespace xb
