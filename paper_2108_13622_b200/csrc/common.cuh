// Shared device definitions for the sm_100a MHD / FD-JVP / Leja kernels.
//
// Bitwise contract: every arithmetic expression below reproduces the IEEE
// operation sequence NumPy executes in the reference (pkg/src/xmhd/mhd.py,
// linearize.py, leja.py): one rounding per ufunc, Python's left-to-right
// association, no FMA contraction (the .so is compiled with -fmad=false; the
// only FMAs are the explicit __fma_rn calls inside the exact-division helpers
// and the norm accumulators, which are not part of the bitwise contract).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace xb {

constexpr int NF = 8;
enum Field { RHO = 0, MX, MY, MZ, BX, BY, BZ, EN };

// Boundary kinds (mhd.py:34-36).  GHOST_HALO = rows supplied by a neighbour
// rank (y-strip decomposition); never used for x.
enum Bc { BC_PERIODIC = 0, BC_REFLECT = 1, BC_HALO = 2 };

// How a constant divisor d is applied given r = RN(1/d) (see exact_div):
//   DIV_MUL  : d is a power of two, a*r == a/d exactly;
//   DIV_MK1  : |1 - d*r| <= 2^-54, one Markstein correction is exact;
//   DIV_MK2  : general d, two corrections (faithful q1, then Markstein);
//   DIV_IEEE : hardware-sequence IEEE division a/d.
enum DivKind { DIV_MUL = 0, DIV_MK1 = 1, DIV_MK2 = 2, DIV_IEEE = 3 };

struct Divisor {
  double d;   // the divisor as NumPy sees it (e.g. the host double 2.0*dx)
  double r;   // RN(1/d)
  int kind;   // DivKind
};

// Correctly rounded a/d for a constant divisor d (no under/overflow).
// Markstein: if r = RN(1/d) and q is within 1 ulp of a/d, then
// RN(q + RN(a - d*q)*r) = RN(a/d) (the remainder is exact by FMA).
// RN(a*r) is within 1 ulp when |1 - d*r| <= 2^-54 (checked on the host);
// otherwise one extra correction first makes q faithful.
// Signed zeros: a == -0 yields +0 on the Markstein paths (value-equal).
__device__ __forceinline__ double exact_div(double a, const Divisor& v) {
  switch (v.kind) {
    case DIV_MUL:
      return __dmul_rn(a, v.r);
    case DIV_MK1: {
      double q = __dmul_rn(a, v.r);
      double e = __fma_rn(-q, v.d, a);
      return __fma_rn(e, v.r, q);
    }
    case DIV_MK2: {
      double q = __dmul_rn(a, v.r);
      double e = __fma_rn(-q, v.d, a);
      q = __fma_rn(e, v.r, q);
      e = __fma_rn(-q, v.d, a);
      return __fma_rn(e, v.r, q);
    }
    default:
      return __ddiv_rn(a, v.d);
  }
}

// Geometry + physics constants, host-folded exactly like Python does.
struct Geom {
  int nx, ny;              // local grid (ny = rows owned by this rank)
  int bcx, bcy;            // Bc
  int diffusive;           // mu != 0 or eta != 0 or kappa != 0   (mhd.py:181)
  int mu0_one;             // mu0 == 1.0 exactly: x/mu0 == x, skip the division
  long long plane;         // nx * ny
  Divisor h2x, h2y;        // 2.0*dx, 2.0*dy                      (mhd.py:113-120)
  Divisor mu0d;            // mu0
  double gm1;              // gamma - 1.0                          (mhd.py:150)
  double mu, eta;
  double cond;             // mu*kap*gamma/(gamma-1.0)             (mhd.py:197)
  double c23;              // 2.0/3.0                              (mhd.py:185)
  // y-strip halo rows (BC_HALO): rows -2,-1 and ny, ny+1 of every field,
  // layout [field][2][nx]; null otherwise.
  const double* halo_lo;
  const double* halo_hi;
  const double* halo_lo_dir;   // same for the JVP direction vector
  const double* halo_hi_dir;
};

// Diffusive terms present (mhd.py:181)?  Only the generic variant
// (K == DIV_IEEE) is launched for mu = eta = kappa = 0, so the others skip the
// runtime test.
template <int K>
__device__ __forceinline__ bool diff_on(const Geom& g) {
  return K == DIV_IEEE ? g.diffusive != 0 : true;
}
// Compile-time variant of exact_div (the kind is a template parameter).
template <int K>
__device__ __forceinline__ double qdiv(double a, const Divisor& v) {
  if (K == DIV_MUL) return __dmul_rn(a, v.r);
  if (K == DIV_IEEE) return __ddiv_rn(a, v.d);
  double q = __dmul_rn(a, v.r);
  double e = __fma_rn(-q, v.d, a);
  q = __fma_rn(e, v.r, q);
  if (K == DIV_MK2) {
    e = __fma_rn(-q, v.d, a);
    q = __fma_rn(e, v.r, q);
  }
  return q;
}

// Runtime divisor for per-launch scalars (eps, theta): one or two corrections.
__device__ __forceinline__ double rdiv(double a, const Divisor& v) {
  double q = __dmul_rn(a, v.r);
  double e = __fma_rn(-q, v.d, a);
  q = __fma_rn(e, v.r, q);
  if (v.kind == DIV_MK2) {
    e = __fma_rn(-q, v.d, a);
    q = __fma_rn(e, v.r, q);
  } else if (v.kind == DIV_IEEE) {
    q = __ddiv_rn(a, v.d);
  }
  return q;
}

// Divisor for a value known only on the device (RN reciprocal + exactness class).
__device__ __forceinline__ Divisor make_divisor_dev(double d) {
  Divisor v;
  v.d = d;
  v.r = __drcp_rn(d);
  const double e = __fma_rn(-d, v.r, 1.0);   // exact: 1 - d*r
  v.kind = (fabs(e) <= 5.551115123125783e-17) ? DIV_MK1 : DIV_MK2;   // 2^-54
  return v;
}

// GM = false: the launch was dispatched for mu0 == 1.0 (x/1.0 == x exactly),
// so no per-call branch on the runtime flag (6 uniform branches and their
// register moves per cell in the fused kernels); GM = true: any mu0.
template <bool GM>
__device__ __forceinline__ double over_mu0(double a, const Geom& g) {
  if (!GM) return a;
  return g.mu0_one ? a : rdiv(a, g.mu0d);
}

// Primitive variables at one (ghost-extended) cell, mhd.py:144-155.
struct Prim {
  double rho, vx, vy, vz, bx, by, bz, en;
  double b2, pres, ptot, bdotv, emf, temp;
};

template <bool GM>
__device__ __forceinline__ void primitives(const double x[NF], const Geom& g, Prim& p) {
  p.rho = x[RHO];
  // the four divisions by the density share one correctly rounded reciprocal;
  // each quotient is then exact by the two-correction Markstein sequence
  Divisor rd;
  rd.d = p.rho;
  rd.r = __drcp_rn(p.rho);
  p.vx = qdiv<DIV_MK2>(x[MX], rd);
  p.vy = qdiv<DIV_MK2>(x[MY], rd);
  p.vz = qdiv<DIV_MK2>(x[MZ], rd);
  p.bx = x[BX];
  p.by = x[BY];
  p.bz = x[BZ];
  p.en = x[EN];
  // b2 = bx*bx + by*by + bz*bz
  p.b2 = __dadd_rn(__dadd_rn(__dmul_rn(p.bx, p.bx), __dmul_rn(p.by, p.by)),
                   __dmul_rn(p.bz, p.bz));
  // kin = 0.5*rho*(vx*vx + vy*vy + vz*vz)
  double vv = __dadd_rn(__dadd_rn(__dmul_rn(p.vx, p.vx), __dmul_rn(p.vy, p.vy)),
                        __dmul_rn(p.vz, p.vz));
  double kin = __dmul_rn(__dmul_rn(0.5, p.rho), vv);
  // 0.5*b2/mu0
  double hb = over_mu0<GM>(__dmul_rn(0.5, p.b2), g);
  // pres = (gamma-1)*(E - kin - 0.5*b2/mu0); ptot = pres + 0.5*b2/mu0
  p.pres = __dmul_rn(g.gm1, __dsub_rn(__dsub_rn(p.en, kin), hb));
  p.ptot = __dadd_rn(p.pres, hb);
  // bdotv = bx*vx + by*vy + bz*vz
  p.bdotv = __dadd_rn(__dadd_rn(__dmul_rn(p.bx, p.vx), __dmul_rn(p.by, p.vy)),
                      __dmul_rn(p.bz, p.vz));
  // emf_z = vy*bx - by*vx
  p.emf = __dsub_rn(__dmul_rn(p.vy, p.bx), __dmul_rn(p.by, p.vx));
  // temp = pres/rho  (mhd.py:198)
  p.temp = qdiv<DIV_MK2>(p.pres, rd);
}

// Non-zero ideal x-flux rows, mhd.py:161-175.  Slot order:
// RHO, MX, MY, MZ, BY, BZ, EN  (flux_x[BX] == 0).
constexpr int NFX = 7;
template <bool GM>
__device__ __forceinline__ void flux_x(const Prim& p, const Geom& g, double f[NFX]) {
  double rv = __dmul_rn(p.rho, p.vx);
  f[0] = rv;
  f[1] = __dsub_rn(__dadd_rn(__dmul_rn(rv, p.vx), p.ptot), over_mu0<GM>(__dmul_rn(p.bx, p.bx), g));
  f[2] = __dsub_rn(__dmul_rn(rv, p.vy), over_mu0<GM>(__dmul_rn(p.bx, p.by), g));
  f[3] = __dsub_rn(__dmul_rn(rv, p.vz), over_mu0<GM>(__dmul_rn(p.bx, p.bz), g));
  f[4] = -p.emf;
  f[5] = __dsub_rn(__dmul_rn(p.vx, p.bz), __dmul_rn(p.bx, p.vz));
  f[6] = __dsub_rn(__dmul_rn(__dadd_rn(p.en, p.ptot), p.vx), over_mu0<GM>(__dmul_rn(p.bx, p.bdotv), g));
}

// Non-zero ideal y-flux rows, mhd.py:162-176.  Slot order:
// RHO, MX, MY, MZ, BX, BZ, EN  (flux_y[BY] == 0).
constexpr int NFY = 7;
template <bool GM>
__device__ __forceinline__ void flux_y(const Prim& p, const Geom& g, double f[NFY]) {
  double rv = __dmul_rn(p.rho, p.vy);
  f[0] = rv;
  f[1] = __dsub_rn(__dmul_rn(rv, p.vx), over_mu0<GM>(__dmul_rn(p.by, p.bx), g));
  f[2] = __dsub_rn(__dadd_rn(__dmul_rn(rv, p.vy), p.ptot), over_mu0<GM>(__dmul_rn(p.by, p.by), g));
  f[3] = __dsub_rn(__dmul_rn(rv, p.vz), over_mu0<GM>(__dmul_rn(p.by, p.bz), g));
  f[4] = p.emf;
  f[5] = __dsub_rn(__dmul_rn(p.vy, p.bz), __dmul_rn(p.by, p.vz));
  f[6] = __dsub_rn(__dmul_rn(__dadd_rn(p.en, p.ptot), p.vy), over_mu0<GM>(__dmul_rn(p.by, p.bdotv), g));
}

// Quantities of a cell that neighbours differentiate (mhd.py:182-201).
constexpr int NPD = 8;
enum PdSlot { PD_VX = 0, PD_VY, PD_VZ, PD_BX, PD_BY, PD_BZ, PD_T, PD_B2 };

// Diffusive flux rows on the level-1 ring, mhd.py:182-221.
// GX slots: MX, MY, MZ, BY, BZ, EN  (gx[RHO] = gx[BX] = 0)
// GY slots: MX, MY, MZ, BX, BZ, EN  (gy[RHO] = gy[BY] = 0)
constexpr int NG = 6;

// d/dx inputs: xl, xr = PD at (j, i-1), (j, i+1); d/dy inputs: yd, yu = PD at
// (j-1, i), (j+1, i); own = PD at (j, i).
template <int KX, int KY>
__device__ __forceinline__ void diffusive_fluxes(const double xl[NPD], const double xr[NPD],
                                                 const double yd[NPD], const double yu[NPD],
                                                 const double own[NPD], const Geom& g,
                                                 double gx[NG], double gy[NG]) {
#define DX(k) qdiv<KX>(__dsub_rn(xr[k], xl[k]), g.h2x)
#define DY(k) qdiv<KY>(__dsub_rn(yu[k], yd[k]), g.h2y)
  double dvx_dx = DX(PD_VX), dvy_dx = DX(PD_VY), dvz_dx = DX(PD_VZ);
  double dvx_dy = DY(PD_VX), dvy_dy = DY(PD_VY), dvz_dy = DY(PD_VZ);
  double divv = __dadd_rn(dvx_dx, dvy_dy);
  double c23dv = __dmul_rn(g.c23, divv);
  double txx = __dsub_rn(__dmul_rn(2.0, dvx_dx), c23dv);
  double tyy = __dsub_rn(__dmul_rn(2.0, dvy_dy), c23dv);
  double txy = __dadd_rn(dvx_dy, dvy_dx);
  double txz = dvz_dx;
  double tyz = dvz_dy;
  double dbx_dx = DX(PD_BX), dbx_dy = DY(PD_BX);
  double dby_dx = DX(PD_BY), dby_dy = DY(PD_BY);
  double curl = __dmul_rn(g.eta, __dsub_rn(dby_dx, dbx_dy));
  double dbz_dx = DX(PD_BZ), dbz_dy = DY(PD_BZ);
  double dT_dx = DX(PD_T), dT_dy = DY(PD_T);
  double db2_dx = DX(PD_B2), db2_dy = DY(PD_B2);
#undef DX
#undef DY
  double vx1 = own[PD_VX], vy1 = own[PD_VY], vz1 = own[PD_VZ];
  double bx1 = own[PD_BX], by1 = own[PD_BY];
  gx[0] = __dmul_rn(g.mu, txx);
  gy[0] = __dmul_rn(g.mu, txy);
  gx[1] = __dmul_rn(g.mu, txy);
  gy[1] = __dmul_rn(g.mu, tyy);
  gx[2] = __dmul_rn(g.mu, txz);
  gy[2] = __dmul_rn(g.mu, tyz);
  gy[3] = -curl;
  gx[3] = curl;
  gx[4] = __dmul_rn(g.eta, dbz_dx);
  gy[4] = __dmul_rn(g.eta, dbz_dy);
  // gx[EN] = mu*(txx*vx1 + txy*vy1 + txz*vz1) + cond*dT/dx
  //          + eta*(0.5*db2/dx - (bx1*dbx/dx + by1*dbx/dy))
  {
    double a = __dmul_rn(g.mu, __dadd_rn(__dadd_rn(__dmul_rn(txx, vx1), __dmul_rn(txy, vy1)),
                                         __dmul_rn(txz, vz1)));
    double b = __dmul_rn(g.cond, dT_dx);
    double c = __dmul_rn(g.eta, __dsub_rn(__dmul_rn(0.5, db2_dx),
                                          __dadd_rn(__dmul_rn(bx1, dbx_dx), __dmul_rn(by1, dbx_dy))));
    gx[5] = __dadd_rn(__dadd_rn(a, b), c);
  }
  {
    double a = __dmul_rn(g.mu, __dadd_rn(__dadd_rn(__dmul_rn(txy, vx1), __dmul_rn(tyy, vy1)),
                                         __dmul_rn(tyz, vz1)));
    double b = __dmul_rn(g.cond, dT_dy);
    double c = __dmul_rn(g.eta, __dsub_rn(__dmul_rn(0.5, db2_dy),
                                          __dadd_rn(__dmul_rn(bx1, dby_dx), __dmul_rn(by1, dby_dy))));
    gy[5] = __dadd_rn(__dadd_rn(a, b), c);
  }
}

}  // namespace xb
