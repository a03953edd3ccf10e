// Fused fp64 resistive-MHD stencil for sm_100a: RHS, FD-JVP and the fused
// Leja/Newton iteration in one pass over HBM.
//
// Reference path (arxiv/paper_2108_13622, pkg/src/xmhd):
//   mhd_rhs            mhd.py:127-232     (MODE_RHS)
//   jvp                linearize.py:56-67 (MODE_JVP: x = u + eps*w, (F(x) - F(u))/eps)
//   apply_phi_leja     leja.py:133-148    (MODE_LEJA: the JVP above plus
//                      y' = ((dt*w) - (q*y))/theta - xi*y, p' = p + c*y',
//                      ||y'||, ||p'|| and the convergence control, on device)
//
// Data layout: the reference's flat field-major (8, ny, nx) fp64 vector.
//
// Dataflow (one CTA = one y-segment of one column strip, sliding window):
//   a CTA of SW=128 threads owns ghost-extended columns [X0-2, X0+126) and
//   marches the rows r = Y0-2 .. Y1+1.  Per row step:
//     P1  thread t forms x(r, c_t) (= u or u + eps*y, with boundary mirror /
//         wrap) from registers loaded one step earlier, immediately issues the
//         loads of row r+1, computes the primitives once and stores the 8
//         differentiated primitives (PD), the 7 ideal x-fluxes (FX) and its 7
//         ideal y-fluxes (FY) in shared-memory rings;
//     P2  level-1 derivatives at row r-1 (PD of rows r-2, r-1, r) -> diffusive
//         fluxes GX (shared ring, x-neighbours read it) and GY (registers);
//     P3  output row r-2: centred differences of FX, FY, GX, GY in the
//         reference's association order, then the mode epilogue whose
//         operands (F(u), y, p at row r-2) were loaded at the start of the step.
//   Every primitive / flux is evaluated once per cell (plus the 4-column and
//   4-row halo of each CTA), so the kernel streams u, y, F(u), p once and
//   writes y', p' once: 384 B per cell per Leja iteration.
//   Two barriers per row step; the rings are sized so no other hazard exists.
//
// Divisions: constant divisors (2dx, 2dy, eps, theta, mu0) use a precomputed
// RN reciprocal with Markstein correction (common.cuh), which is the correctly
// rounded quotient; 2dx / 2dy kinds are template parameters.  Divisions by the
// per-cell density share one correctly rounded reciprocal (__drcp_rn) and are
// completed by the two-correction Markstein sequence (exact for any divisor).
#include <cfloat>
#include <cstdlib>
#include <climits>
#include <type_traits>
#include <cooperative_groups.h>
#include "kernels.h"

namespace cg = cooperative_groups;

// L2 prefetch ahead of the per-thread loads (measured on B200, 2048^2 / 4096^2:
// off 0.343 / 1.300 ms; rows 2 ahead + epilogue 1 ahead 0.313 / 1.243 ms;
// epilogue 2 ahead 0.323; rows 3 / 4 / 5 ahead 0.353 / 0.328 / 0.352; rows 3 +
// epilogue 2 ahead 0.329; bulk cp.async.bulk.prefetch instead of per-line
// prefetches 0.339).
#ifndef XB_L2PF
#ifndef XB_EPI_K1
#define XB_EPI_K1 0   // measured: 0.284 vs 0.280 ms at 2048^2 (four epilogue copies; i-cache)
#endif
#define XB_L2PF 2   // row steps of the state / direction prefetch (0: no prefetch)
#endif
#ifndef XB_L2PF_E
#define XB_L2PF_E 1   // lead (row steps) of the epilogue-operand L2 prefetch
#endif
#ifndef XB_BULKPF
#define XB_BULKPF 0   // bulk (cp.async.bulk.prefetch.L2) instead of per-line prefetches
#endif
// Variants measured and dropped: epilogue operands staged by
// cp.async (-43%: the larger shared-memory carve-out starves L1), epilogue
// prefetch to L2 only (neutral), GY ring in shared memory (-35%), L1 cache
// hints (-10%), double2 shared-memory rings (neutral), 256-thread strips with
// one CTA per SM (XB_SW=256: -20%, barrier stalls hit all 8 warps at once),
// one-correction bodies for eps / theta when exact (neutral), the lookahead
// interpolant schedule with runtime mode branches in one kernel (0.338 vs
// 0.305 ms at 2048^2: hence one compiled variant per mode), 64-thread strips
// (0.327 vs 0.315 ms), the row loop unrolled by 3 so the PD / GY register
// rings need no copies (-30% MOVs, but 0.337 ms: code size and scheduling), the
// output phase of row r-3 moved into the same barrier phase as the primitives
// of row r (two independent chains per phase, 5-slot FY ring; commit 40988eb:
// odd / even term 0.286 / 0.396 ms vs 0.250 / 0.320 ms on the same box), an
// interior-row fast path around row_source plus a launch-uniform test around
// the mirror negations (~100 fewer integer / branch instructions of the ~1060
// per row step, yet odd / even term 0.2527 / 0.3241 ms vs 0.2491 / 0.3206 ms,
// 4096^2 0.9396 / 1.2419 vs 0.9257 / 1.2272: the integer work is not on the
// critical path, the fp64 and shared-memory dependency chains of two warps per
// scheduler are), the epilogue operand loads issued after P2 instead of at the
// step start (same 238 / 252 registers; odd term 0.245 vs 0.250 ms but even
// term 0.342 vs 0.322 ms, 4096^2 1.000 / 1.339 vs 0.927 / 1.222 ms: their L2
// latency needs the whole step to hide).

namespace xb {

namespace {

// Slot -> field maps for the non-zero flux rows (compile-time in unrolled loops).
__host__ __device__ constexpr int fx_field(int k) { return k < 4 ? k : k + 1; }   // skip BX
__host__ __device__ constexpr int fy_field(int k) { return k < 5 ? k : k + 1; }   // skip BY

// One barrier per row step (XB_ONEBAR): with a 3-slot PD ring, P1 of step s+1
// writes a PD slot no P2 of step s reads, so the barrier between P2 and the
// next P1 goes; every other ring hazard is still separated by the barrier
// after P1 (FX: P3(s) reads slot s-2 while P1(s+1) writes s+1; GX: P2(s)
// writes s+1 while P3(s) reads s; FY is read by its own column only).
#ifndef XB_FYREG
#define XB_FYREG 1
#endif
#ifndef XB_ONEBAR
#define XB_ONEBAR 0   // measured: 0.282 vs 0.281 ms (2048^2), 1.088 vs 1.080 (4096^2): the larger carve-out costs more than the barrier
#endif
constexpr int RING_PD = XB_ONEBAR ? 3 : 2, RING_FX = 4, RING_FY = 4, RING_GX = 2;

// Source of one ghost-extended row.  Element offsets are 32-bit unsigned: a
// per-GPU vector of 8*nx*ny < 2^32 doubles (34 GB) covers every grid that fits
// a 180 GB device (checked at context creation), and unsigned offsets turn
// each access into a single IMAD.WIDE.U32 address.
struct RowSrc {
  const double* u;     // base of the base state (or its halo buffer)
  const double* d;     // base of the direction vector (or its halo buffer)
  unsigned off;        // element offset of the row's field-0 start
  unsigned fs;         // stride between fields
  int flip;            // mirror ghost row: negate MY, BY
};

__device__ __forceinline__ RowSrc row_source(int r, const Geom& g, const double* u,
                                             const double* d, const double* hlo_dir,
                                             const double* hhi_dir) {
  RowSrc s;
  s.flip = 0;
  s.fs = (unsigned)g.plane;
  s.u = u;
  s.d = d;
  int rr = r;
  if (g.bcy == BC_PERIODIC) {
    // r lies in [-2, ny+2) and ny >= 2: one conditional wrap, no integer division
    rr = r < 0 ? r + g.ny : (r >= g.ny ? r - g.ny : r);
  } else if (g.bcy == BC_REFLECT) {
    if (r < 0) { rr = -1 - r; s.flip = 1; }
    else if (r >= g.ny) { rr = 2 * g.ny - 1 - r; s.flip = 1; }
    rr = min(max(rr, 0), g.ny - 1);
  } else {  // BC_HALO: rows owned by the y-neighbours, [field][2][nx]
    if (r < 0) {
      s.u = g.halo_lo;
      s.d = hlo_dir;
      s.off = (unsigned)(r + 2) * (unsigned)g.nx;
      s.fs = 2u * (unsigned)g.nx;
      return s;
    }
    if (r >= g.ny) {
      s.u = g.halo_hi;
      s.d = hhi_dir;
      s.off = (unsigned)(r - g.ny) * (unsigned)g.nx;
      s.fs = 2u * (unsigned)g.nx;
      return s;
    }
  }
  s.off = (unsigned)rr * (unsigned)g.nx;
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

// Exchange kind of a MODE_LEJA launch: none (single domain, or y-strips over
// NCCL with ext_sums), peer memory (one launch per rank), or P ranks emulated
// in one cooperative launch on one GPU.
// XR_LOOP: the single-domain persistent loop (leja_loop_kernel), where y and p
// are rewritten between terms inside one launch, so their loads bypass L1.
enum { XR_NONE = 0, XR_PEER = 1, XR_EMUL = 2, XR_LOOP = 3 };

// Load of data another block rewrites inside the same launch (XR_LOOP): L2 only.
template <bool COH>
__device__ __forceinline__ double ld_dir(const double* p) {
  return COH ? __ldcg(p) : __ldg(p);
}

// y' of boundary row o of this strip into the ghost-row buffers it feeds
// ([field][2][nx]): rows 0, 1 -> the rank below (its rows ny, ny+1) or, at a
// reflecting wall, my own ghost rows -1, -2 with MY, BY odd; rows ny-2, ny-1
// likewise upwards.  Same values as leja_pack_halo_kernel (vec.cu).
__device__ __forceinline__ void push_ghost(double* dlo, int mlo, double* dhi, int mhi, int f,
                                           int o, int ny, int nx, int c, double y) {
  const double s = (f == MY || f == BY) ? -1.0 : 1.0;
  if (o < 2 && dlo) {
    const int k = mlo ? 1 - o : o;
    dlo[(f * 2 + k) * nx + c] = mlo ? __dmul_rn(s, y) : y;
  }
  if (o >= ny - 2 && dhi) {
    const int k = mhi ? ny - 1 - o : o - (ny - 2);
    dhi[(f * 2 + k) * nx + c] = mhi ? __dmul_rn(s, y) : y;
  }
}

}  // namespace

// One launch of the fused stencil.  bid / nblk: this block's index among the
// nblk blocks working on this rank's grid (the launch grid, except in the
// one-launch emulation of several ranks).
template <int MODE, int KX, int KY, int XR, int PM = PM_ANY>
__device__ __forceinline__ void stencil_body(const StencilArgs& a, const int bid,
                                             const int nblk) {
  constexpr bool P2P = (XR == XR_PEER || XR == XR_EMUL);
  constexpr bool COH = (XR == XR_LOOP);
  // The ideal y-fluxes are read by their own column only.  The RHS kernel has
  // the registers (170 of 255) to keep its three pending rows there instead of
  // in the shared-memory ring: 21 of its 84 shared-memory accesses per cell and
  // row step go, and the L1 data pipe is its busiest unit.
  constexpr bool FYREG = XB_FYREG && (MODE == MODE_RHS);
  extern __shared__ __align__(16) double smem[];
  double (*pd)[NPD][SW] = reinterpret_cast<double (*)[NPD][SW]>(smem);
  double (*fxs)[NFX][SW] = reinterpret_cast<double (*)[NFX][SW]>(smem + RING_PD * NPD * SW);
  double (*fys)[NFY][SW] =
      reinterpret_cast<double (*)[NFY][SW]>(smem + (RING_PD * NPD + RING_FX * NFX) * SW);
  double (*gxs)[NG][SW] = reinterpret_cast<double (*)[NG][SW]>(
      smem + (RING_PD * NPD + RING_FX * NFX + RING_FY * NFY) * SW);
  __shared__ double red[SW / 32];
  __shared__ int am_last;

  const Geom& g = a.g;
  const int t = threadIdx.x;

  // Per-launch scalars.
  double eps = a.eps;
  Divisor epsd = a.epsd;
  Divisor thd = epsd;
  const double* dir = a.dir;
  double* yout = nullptr;
  const double* pin = nullptr;
  double* pout = nullptr;
  double dt = 0.0, q = 0.0, xim = 0.0, cm = 0.0;
  double pcoef = 0.0;          // coefficient of a pending interpolant term
  int ppend = 0;               // a term is pending (pbuf[pcur] + pcoef * y)
  int pm_rt = PM_STORE;        // LejaPMode of this term (control block)
  int zero_dir = 0;
  int pvirt = 0;               // the stored interpolant is still c0 * v (in-place start)
  double c0 = 0.0;
  // MODE_JVP as the tail of a stage difference (integrators.py:146-153):
  // out = (F(stage) - F(u)) - J w instead of J w
  const double* sfp = (MODE == MODE_JVP) ? a.stage_f : nullptr;
  const double* hlo_dir = g.halo_lo_dir;
  const double* hhi_dir = g.halo_hi_dir;
  double* push_lo = nullptr;
  double* push_hi = nullptr;
  if (MODE == MODE_LEJA) {
    const volatile LejaCtl* c = a.ctl;   // rewritten by the last block of every term
    if (c->status != LJ_RUNNING) return;
    const int cur = c->cur, m = c->m;
    if (XR == XR_NONE && a.term && m != a.term) return;   // a pair's variant for another term
    if (P2P) {
      hlo_dir = a.p2p.halo_lo_dir[cur];
      hhi_dir = a.p2p.halo_hi_dir[cur];
      push_lo = a.p2p.dst_lo[cur ^ 1];
      push_hi = a.p2p.dst_hi[cur ^ 1];
    }
    eps = c->eps;
    epsd.d = c->epsd.d;
    epsd.r = c->epsd.r;
    epsd.kind = c->epsd.kind;
    thd.d = c->thetad.d;
    thd.r = c->thetad.r;
    thd.kind = c->thetad.kind;
    zero_dir = c->zero_dir;
    dir = a.ybuf[cur];
    yout = a.ybuf[cur ^ 1];
    const int pc = c->pcur;
    pin = a.pbuf[pc];
    pout = a.pbuf[pc ^ 1];
    if (XR == XR_NONE && a.v0) {
      // in-place start: term 1 reads the caller's v as its direction, and until
      // a term has stored p the interpolant read here is c0 * v
      if (m == 1) dir = a.v0;
      pvirt = c->pvirt;
      if (pvirt) { pin = a.v0; c0 = c->c0; }
    }
    ppend = c->ppend;
    pcoef = c->pend_coef;
    pm_rt = c->pmode;
    if (PM != PM_ANY && pm_rt != PM) {   // variant launched for another mode
      if (XR == XR_NONE && a.term) return;   // the other variant of the pair runs this term
      if (bid == 0 && threadIdx.x == 0) a.ctl->status = LJ_MODE_ERROR;
      return;
    }
    dt = c->dt;
    q = c->q;
    xim = __ldg(a.xi + (m - 1));
    cm = __ldg(a.coeffs + m);
  }

  if (MODE == MODE_JVP && a.pctl) {
    // device power iteration: the FD step comes from the control block
    const PowerCtl* pc = a.pctl;
    if (pc->status != PW_RUNNING) return;
    eps = pc->eps;
    epsd = pc->epsd;
  }

  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;   // sums of y'^2, p'^2, pending p^2
  int bad = 0;
  // interpolant handling of this term: compile-time for the PM variants
  const int pmode = (PM == PM_ANY) ? pm_rt : PM;
  const bool pread = (pmode != PM_SKIP);
  const bool pstore = (pmode == PM_STORE || pmode == PM_LOOK);
  const bool padd = (PM == PM_LOOK) ? true : (PM == PM_SKIP ? false : (ppend != 0));
  const bool pnorm2 = (pmode == PM_LOOK);

  if (MODE == MODE_LEJA && zero_dir) {
    // jvp of a zero vector is exactly zero and costs no RHS call (linearize.py:63-64)
    const long long n = (long long)NF * g.plane;
    for (long long i = (long long)bid * SW + t; i < n; i += (long long)nblk * SW) {
      const double y = ld_dir<COH>(dir + i);
      const double yn = __dsub_rn(__ddiv_rn(__dsub_rn(__dmul_rn(dt, 0.0), __dmul_rn(q, y)), thd.d),
                                  __dmul_rn(xim, y));
      yout[i] = yn;
      double pn = 0.0;
      if (pread) {
        double pb = ld_dir<COH>(pin + i);
        if (XR == XR_NONE && pvirt) pb = __dmul_rn(c0, pb);
        if (padd) {   // the pending term first
          pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
          if (pnorm2) acc2 = __fma_rn(pb, pb, acc2);
        }
        pn = __dadd_rn(pb, __dmul_rn(cm, yn));
        if (pstore) pout[i] = pn;
      }
      if (P2P) {
        const int f = (int)(i / g.plane);
        const long long rem = i - (long long)f * g.plane;
        const int o = (int)(rem / g.nx), c = (int)(rem - (long long)o * g.nx);
        push_ghost(push_lo, a.p2p.mirror_lo, push_hi, a.p2p.mirror_hi, f, o, g.ny, g.nx, c, yn);
      }
      acc0 = __fma_rn(yn, yn, acc0);
      acc1 = __fma_rn(pn, pn, acc1);
    }
  } else {
    for (int unit = bid; unit < a.nunits; unit += nblk) {
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
      const double* dsrc = (MODE == MODE_RHS) ? nullptr : dir;

      double gy1[NG], gy2[NG];
#pragma unroll
      for (int k = 0; k < NG; ++k) gy1[k] = gy2[k] = 0.0;
      int s3 = 0;  // s % 3 (PD ring)
      // own-column differentiated primitives of rows r-1 and r-2 (registers);
      // shared memory holds only the row x-neighbours read (PD of row r-1)
      double pr1[NPD], pr2[NPD];
#pragma unroll
      for (int k = 0; k < NPD; ++k) pr1[k] = pr2[k] = 0.0;
      // FYREG: ideal y-fluxes of rows r-1, r-2, r-3 of this column
      double fq1[NFY], fq2[NFY], fq3[NFY];
#pragma unroll
      for (int k = 0; k < NFY; ++k) fq1[k] = fq2[k] = fq3[k] = 0.0;

      // prefetch registers: state (and direction) of the next row to consume
      double nu[NF], nd[NF];
      int nflip;   // mirror flag of the prefetched row
      {
        const RowSrc rs = row_source(Y0 - 2, g, a.u, dsrc, hlo_dir, hhi_dir);
        nflip = rs.flip;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          nu[f] = __ldg(rs.u + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
          if (MODE != MODE_RHS) nd[f] = ld_dir<COH>(rs.d + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
        }
      }

      const int nsteps = (Y1 - Y0) + 4;
      int s4 = 0;  // s % 4
      for (int s = 0; s < nsteps; ++s) {
        const int r = Y0 - 2 + s;
        const bool out_row = (s >= 4) && col_ok;
        const unsigned obase = (unsigned)(r - 2) * (unsigned)g.nx + (unsigned)c_out;
        const unsigned plane = (unsigned)g.plane;

#if XB_L2PF
        // L2 prefetch of the rows the next steps will load: the state /
        // direction row XB_L2PF steps ahead and the epilogue operands of the
        // next output row, so the per-thread loads of those steps hit L2 and
        // hold their L1 miss slots for far less time (+8% at 2048^2).
        if (MODE != MODE_RHS) {
          const int rp = r + XB_L2PF;
          const int ro = r - 2 + XB_L2PF_E;   // output row of step s + XB_L2PF_E
          const bool do_rows = s + XB_L2PF < nsteps && rp >= 0 && rp < g.ny;
          const bool do_epi = s + XB_L2PF_E < nsteps && s + XB_L2PF_E >= 4 && ro >= 0 &&
                              ro < g.ny;
#if XB_BULKPF
          // one bulk (TMA-engine) L2 prefetch per field row of the CTA's columns
          const int c0 = max(X0 - 2, 0) & ~1;                  // 16-byte aligned start
          const int c1 = min(X0 + SW - 2, g.nx);
          const unsigned bytes = (unsigned)((c1 - c0 + 1) & ~1) * 8u;
          const int nrow = (MODE == MODE_LEJA) ? 24 : 8;
          if (t < 16 + nrow) {
            const double* base;
            int row, f;
            bool on;
            if (t < 16) { base = (t < 8) ? a.u : dir; f = t & 7; row = rp; on = do_rows; }
            else {
              const int k = t - 16;
              base = (k < 8) ? a.fu : (k < 16 ? dir : pin);
              f = k & 7; row = ro; on = do_epi;
            }
            if (on && bytes)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                  base + ((unsigned)f * plane + (unsigned)row * (unsigned)g.nx + (unsigned)c0)),
                  "r"(bytes) : "memory");
          }
#else
          // one 128-B line per thread: LPR lines per field row, 2*8*LPR == SW
          constexpr int LPR = SW / 16;
          const int seg = t % LPR, f = (t / LPR) & 7;
          const int c0 = min(max(X0 - 2 + seg * 16, 0), g.nx - 1);
          if (do_rows) {
            const double* base = (t >= 8 * LPR) ? dir : a.u;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(
                base + ((unsigned)f * plane + (unsigned)rp * (unsigned)g.nx + (unsigned)c0)));
          }
          if (do_epi) {
#pragma unroll
            for (int k = t; k < (MODE == MODE_LEJA ? (pread ? 24 : 16) : (sfp ? 16 : 8)) * LPR;
                 k += SW) {
              const double* base = (k < 8 * LPR) ? a.fu
                                                 : (k < 16 * LPR ? (MODE == MODE_JVP ? sfp : dir) : pin);
              const int ff = (k / LPR) & 7, sg = k % LPR;
              const int cc = min(max(X0 - 2 + sg * 16, 0), g.nx - 1);
              asm volatile("prefetch.global.L2 [%0];" ::"l"(
                  base + ((unsigned)ff * plane + (unsigned)ro * (unsigned)g.nx + (unsigned)cc)));
            }
          }
#endif
        }
#endif
        // epilogue operands of output row r-2: issue now, consume in P3
        double efu[NF], ey[NF], ep[NF], esf[NF];
        if (MODE != MODE_RHS && out_row) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const unsigned i = obase + (unsigned)f * plane;
            efu[f] = __ldg(a.fu + i);
            if (MODE == MODE_JVP && sfp) esf[f] = __ldg(sfp + i);
            if (MODE == MODE_LEJA) {
              ey[f] = ld_dir<COH>(dir + i);
              if (pread) ep[f] = ld_dir<COH>(pin + i);
            }
          }
        }

        // ---- P1: state at (r, cg) from the prefetch registers
        double pn[NPD];
        double fyn[NFY];   // FYREG: ideal y-fluxes of row r
        {
          double x[NF];
#pragma unroll
          for (int f = 0; f < NF; ++f)
            x[f] = (MODE == MODE_RHS) ? nu[f] : __dadd_rn(nu[f], __dmul_rn(eps, nd[f]));
          if (flipx) { x[MX] = -x[MX]; x[BX] = -x[BX]; }
          if (nflip) { x[MY] = -x[MY]; x[BY] = -x[BY]; }
          if (s + 1 < nsteps) {
            const RowSrc rs = row_source(r + 1, g, a.u, dsrc, hlo_dir, hhi_dir);
            nflip = rs.flip;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              nu[f] = __ldg(rs.u + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
              if (MODE != MODE_RHS) nd[f] = ld_dir<COH>(rs.d + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
            }
          }
          Prim p;
          primitives<KX == DIV_IEEE>(x, g, p);
          pn[PD_VX] = p.vx;
          pn[PD_VY] = p.vy;
          pn[PD_VZ] = p.vz;
          pn[PD_BX] = p.bx;
          pn[PD_BY] = p.by;
          pn[PD_BZ] = p.bz;
          pn[PD_T] = p.temp;
          pn[PD_B2] = p.b2;
          double fv[NFX];
#pragma unroll
          for (int k = 0; k < NPD; ++k) pd[XB_ONEBAR ? s3 : (s & 1)][k][t] = pn[k];
          flux_x<KX == DIV_IEEE>(p, g, fv);
#pragma unroll
          for (int k = 0; k < NFX; ++k) fxs[s4][k][t] = fv[k];
          flux_y<KX == DIV_IEEE>(p, g, fv);
          if (FYREG) {
#pragma unroll
            for (int k = 0; k < NFY; ++k) fyn[k] = fv[k];
          } else {
#pragma unroll
            for (int k = 0; k < NFY; ++k) fys[s4][k][t] = fv[k];
          }
        }
        __syncthreads();

        // ---- P2: diffusive fluxes at row r-1
        double gyn[NG];
#pragma unroll
        for (int k = 0; k < NG; ++k) gyn[k] = 0.0;
        if (diff_on<KX>(g) && s >= 2) {
          double xl[NPD], xr[NPD];   // PD of row r-1 at t-1, t+1
          const int sp = XB_ONEBAR ? (s3 == 0 ? 2 : s3 - 1) : ((s + 1) & 1);   // row r-1
#pragma unroll
          for (int k = 0; k < NPD; ++k) {
            xl[k] = pd[sp][k][tl];
            xr[k] = pd[sp][k][tr];
          }
          double gxv[NG];
          diffusive_fluxes<KX, KY>(xl, xr, pr2, pn, pr1, g, gxv, gyn);
#pragma unroll
          for (int k = 0; k < NG; ++k) gxs[(s + 1) & 1][k][t] = gxv[k];
        }
#pragma unroll
        for (int k = 0; k < NPD; ++k) { pr2[k] = pr1[k]; pr1[k] = pn[k]; }
        if (!XB_ONEBAR) __syncthreads();

        // ---- P3: output row o = r-2
        if (out_row) {
          const int fx2 = (s4 + 2) & 3;   // FX / FY slot of row r-2 (s-2 mod 4)
          const int fy1 = (s4 + 3) & 3;   // FY slot of row r-1
          const int fy3 = (s4 + 1) & 3;   // FY slot of row r-3
          const int gs = s & 1;           // GX slot of row r-2
          double F[NF];
          // ideal part: out = -(dFX/2dx); out -= dFY/2dy       (mhd.py:177-178)
          {
            double a[NFX], b[NFX];
#pragma unroll
            for (int k = 0; k < NFX; ++k) { a[k] = fxs[fx2][k][tr]; b[k] = fxs[fx2][k][tl]; }
#pragma unroll
            for (int k = 0; k < NFX; ++k)
              F[fx_field(k)] = -qdiv<KX>(__dsub_rn(a[k], b[k]), g.h2x);
          }
          F[BX] = -0.0;
          {
            double a[NFY], b[NFY];
#pragma unroll
            for (int k = 0; k < NFY; ++k) {
              a[k] = FYREG ? fq1[k] : fys[fy1][k][t];
              b[k] = FYREG ? fq3[k] : fys[fy3][k][t];
            }
#pragma unroll
            for (int k = 0; k < NFY; ++k) {
              const int f = fy_field(k);
              F[f] = __dsub_rn(F[f], qdiv<KY>(__dsub_rn(a[k], b[k]), g.h2y));
            }
          }
          F[BY] = __dsub_rn(F[BY], 0.0);
          if (diff_on<KX>(g)) {
            // out += dGX/2dx; out += dGY/2dy                 (mhd.py:222-223)
            double gr[NG], gl[NG];
#pragma unroll
            for (int k = 0; k < NG; ++k) { gr[k] = gxs[gs][k][tr]; gl[k] = gxs[gs][k][tl]; }
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BX] = __dadd_rn(F[BX], 0.0);
            F[MX] = __dadd_rn(F[MX], qdiv<KX>(__dsub_rn(gr[0], gl[0]), g.h2x));
            F[MY] = __dadd_rn(F[MY], qdiv<KX>(__dsub_rn(gr[1], gl[1]), g.h2x));
            F[MZ] = __dadd_rn(F[MZ], qdiv<KX>(__dsub_rn(gr[2], gl[2]), g.h2x));
            F[BY] = __dadd_rn(F[BY], qdiv<KX>(__dsub_rn(gr[3], gl[3]), g.h2x));
            F[BZ] = __dadd_rn(F[BZ], qdiv<KX>(__dsub_rn(gr[4], gl[4]), g.h2x));
            F[EN] = __dadd_rn(F[EN], qdiv<KX>(__dsub_rn(gr[5], gl[5]), g.h2x));
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BY] = __dadd_rn(F[BY], 0.0);
            const double* gy3 = gy2;
            F[MX] = __dadd_rn(F[MX], qdiv<KY>(__dsub_rn(gyn[0], gy3[0]), g.h2y));
            F[MY] = __dadd_rn(F[MY], qdiv<KY>(__dsub_rn(gyn[1], gy3[1]), g.h2y));
            F[MZ] = __dadd_rn(F[MZ], qdiv<KY>(__dsub_rn(gyn[2], gy3[2]), g.h2y));
            F[BX] = __dadd_rn(F[BX], qdiv<KY>(__dsub_rn(gyn[3], gy3[3]), g.h2y));
            F[BZ] = __dadd_rn(F[BZ], qdiv<KY>(__dsub_rn(gyn[4], gy3[4]), g.h2y));
            F[EN] = __dadd_rn(F[EN], qdiv<KY>(__dsub_rn(gyn[5], gy3[5]), g.h2y));
          }
          // non-finite detection (mhd.py:225-231): exponent field all ones
          {
            unsigned ex = 0;
#pragma unroll
            for (int f = 0; f < NF; ++f)
              ex = max(ex, (unsigned)__double2hiint(F[f]) & 0x7ff00000u);
            bad |= (ex == 0x7ff00000u);
          }
          // The epilogue's two divisions (by eps, by theta) take the
          // one-correction path when the divisor's class proves it exact
          // (XB_EPI_K1: one uniform branch per row step into one of four copies).
          auto epilogue = [&](auto KEc, auto KTc) {
            constexpr int KE = decltype(KEc)::value, KT = decltype(KTc)::value;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              const unsigned i = obase + (unsigned)f * plane;
              if (MODE == MODE_RHS) {
                a.out[i] = F[f];
              } else if (MODE == MODE_JVP) {
                const double jv = qdiv<DIV_MK2>(__dsub_rn(F[f], efu[f]), epsd);
                a.out[i] = sfp ? __dsub_rn(__dsub_rn(esf[f], efu[f]), jv) : jv;
                acc0 = __fma_rn(jv, jv, acc0);
              } else {
                // per-launch divisors (eps, theta): exact on either path
                const double w = qdiv<KE>(__dsub_rn(F[f], efu[f]), epsd);
                const double y = ey[f];
                const double yn = __dsub_rn(
                    qdiv<KT>(__dsub_rn(__dmul_rn(dt, w), __dmul_rn(q, y)), thd),
                    __dmul_rn(xim, y));
                yout[i] = yn;
                double pn = 0.0;
                if (pread) {
                  double pb = ep[f];
                  if (XR == XR_NONE && pvirt) pb = __dmul_rn(c0, pb);
                  if (padd) {   // the pending term first
                    pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
                    if (pnorm2) acc2 = __fma_rn(pb, pb, acc2);
                  }
                  pn = __dadd_rn(pb, __dmul_rn(cm, yn));
                  if (pstore) pout[i] = pn;
                }
                if (P2P)
                  push_ghost(push_lo, a.p2p.mirror_lo, push_hi, a.p2p.mirror_hi, f, r - 2, g.ny,
                             g.nx, c_out, yn);
                acc0 = __fma_rn(yn, yn, acc0);
                if (pread) acc1 = __fma_rn(pn, pn, acc1);   // PM_SKIP: no p, no ||p||
              }
            }
          };
          using MK1c = std::integral_constant<int, DIV_MK1>;
          using MK2c = std::integral_constant<int, DIV_MK2>;
          if (XB_EPI_K1 && MODE == MODE_LEJA && epsd.kind == DIV_MK1) {
            if (thd.kind == DIV_MK1) epilogue(MK1c{}, MK1c{});
            else epilogue(MK1c{}, MK2c{});
          } else if (XB_EPI_K1 && MODE == MODE_LEJA && thd.kind == DIV_MK1) {
            epilogue(MK2c{}, MK1c{});
          } else {
            epilogue(MK2c{}, MK2c{});
          }
        }

#pragma unroll
        for (int k = 0; k < NG; ++k) { gy2[k] = gy1[k]; gy1[k] = gyn[k]; }
        if (FYREG) {
#pragma unroll
          for (int k = 0; k < NFY; ++k) { fq3[k] = fq2[k]; fq2[k] = fq1[k]; fq1[k] = fyn[k]; }
        }
        s3 = (s3 == 2) ? 0 : s3 + 1;
        s4 = (s4 + 1) & 3;
      }
      __syncthreads();   // rings are reused by the next unit
    }
  }

  if (bad) atomicOr(a.bad, 1);
  if (MODE == MODE_RHS) return;

  constexpr bool NEED_S2 = (MODE == MODE_LEJA) && (PM == PM_ANY || PM == PM_LOOK);
  const double s0 = block_sum(acc0, red);
  const double s1 = (MODE == MODE_LEJA && PM != PM_SKIP) ? block_sum(acc1, red) : 0.0;
  const double s2 = NEED_S2 ? block_sum(acc2, red) : 0.0;
  if (t == 0) {
    a.partials[3 * bid] = s0;
    a.partials[3 * bid + 1] = s1;
    a.partials[3 * bid + 2] = s2;
    // peer memory: this block's ghost-row stores to the neighbours must be
    // visible system-wide before the last block publishes the epoch
    if (P2P) __threadfence_system();
    else __threadfence();
    const unsigned prev = atomicAdd(a.ticket, 1u);
    am_last = (prev == (unsigned)nblk - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  if (t < 32) {
    const double sy = sum_partials(a.partials, nblk, 3, 0);
    const double sp = (MODE == MODE_LEJA && PM != PM_SKIP) ? sum_partials(a.partials, nblk, 3, 1)
                                                            : 0.0;
    const double sp2 = NEED_S2 ? sum_partials(a.partials, nblk, 3, 2) : 0.0;
    if (t == 0) {
      if (MODE == MODE_JVP && a.pctl) {
        power_after_jvp(a.pctl, sy, *((volatile int*)a.bad));
      } else if (MODE == MODE_JVP) {
        a.result[0] = sqrt(sy);
      } else if (MODE == MODE_LEJA && P2P) {
        // y-strips over peer memory: all-reduce the three sums, then every rank
        // runs the identical control update
        LejaCtl* c = a.ctl;
        const double v[4] = {sy, sp, sp2, *((volatile int*)a.bad) ? 1.0 : 0.0};
        double tot[4];
        const unsigned long long ep = c->epoch + 1;
        c->epoch = ep;
        if (p2p_allreduce4(a.p2p, ep, v, tot))
          leja_finalize(c, tot[0], tot[1], tot[2], tot[3] > 0.0, !zero_dir, cm);
        else
          c->status = LJ_PEER_TIMEOUT;
      } else if (a.ext_sums) {
        // y-strips: publish this rank's partial sums; the control update runs
        // after the cross-rank allreduce (leja_finalize_kernel)
        a.ext_sums[0] = sy;
        a.ext_sums[1] = sp;
        a.ext_sums[2] = sp2;
        a.ext_sums[3] = *((volatile int*)a.bad) ? 1.0 : 0.0;
      } else {
        const int flag = *((volatile int*)a.bad);
        leja_finalize(a.ctl, sy, sp, sp2, flag, !zero_dir, cm, XR == XR_NONE ? a.dual_next : 0);
      }
      if (MODE == MODE_JVP) a.result[1] = sy;   // local sum of squares (y-strips)
      *a.ticket = 0u;
    }
  }
}

template <int MODE, int KX, int KY, int PM = PM_ANY>
__global__ void __launch_bounds__(SW, SW_MINB) stencil_kernel(const StencilArgs a) {
  stencil_body<MODE, KX, KY, XR_NONE, PM>(a, blockIdx.x, gridDim.x);
}

// Fused Leja iteration of one y-strip with the peer-memory exchange.
template <int KX, int KY, int PM = PM_ANY>
__global__ void __launch_bounds__(SW, SW_MINB) leja_peer_kernel(const StencilArgs a) {
  stencil_body<MODE_LEJA, KX, KY, XR_PEER, PM>(a, blockIdx.x, gridDim.x);
}

// P ranks in one cooperative launch on one GPU (tests): blocks
// [r*nblk, (r+1)*nblk) run rank r with args[r]; the ranks' last blocks meet
// in p2p_allreduce3, which the cooperative launch makes safe (co-resident).
template <int KX, int KY, int PM = PM_ANY>
__global__ void __launch_bounds__(SW, SW_MINB) leja_emul_kernel(const StencilArgs* args, int nblk) {
  const int rank = blockIdx.x / nblk;
  stencil_body<MODE_LEJA, KX, KY, XR_EMUL, PM>(args[rank], blockIdx.x - rank * nblk, nblk);
}

// The whole Leja loop of one single-domain phi-action in ONE cooperative
// launch: a term, a grid-wide barrier (y', p' and the control block complete),
// the next term, until the control block leaves RUNNING (converged, blow-up,
// non-finite RHS, 499 terms, or the end of the device coefficient table).
// No host round trip per term: the host enqueues a whole phi-action and
// everything after it without waiting.
template <int KX, int KY>
__global__ void __launch_bounds__(SW, SW_MINB) leja_loop_kernel(const StencilArgs a) {
  cg::grid_group grid = cg::this_grid();
  for (;;) {
    stencil_body<MODE_LEJA, KX, KY, XR_LOOP>(a, blockIdx.x, gridDim.x);
    grid.sync();
    if (((volatile const LejaCtl*)a.ctl)->status != LJ_RUNNING) break;
  }
}

// ---------------------------------------------------------------------------
// Two-role sliding window with a split register file (sm_100a setmaxnreg).
//
// The one-role kernel keeps ~254 registers per column thread, so an SM holds
// two CTAs = 8 warps and the fp64 dependency chains leave the issue slots
// 60% idle.  Here a CTA of 256 threads splits each column's work over two
// warpgroups that work on different rows in the same "tick" and meet at ONE
// __syncthreads() per tick:
//   AB (warpgroup 0, setmaxnreg 160): row r = Y0-2+s: primitives -> PD ring,
//        ideal x- and y-fluxes -> FX / FY rings; then the diffusive fluxes
//        of row r-1 (its own
//        column's PD rows r-2, r-1, r in registers, the x-neighbours of row
//        r-1 from the PD ring written last tick) -> GX ring and the divided
//        GY difference of row r-2 -> DGY ring.  The state / direction loads
//        of row r+1 are issued after that work, so they are in flight across
//        the barrier without adding to the register peak.
//   C  (warpgroup 1, setmaxnreg 96): output row r-3: x-differences of FX and
//        GX, y-differences of FY, the DGY terms in the reference's order (mhd.py:177-178,
//        222-223), the mode epilogue and the norm partials; its epilogue
//        operands for the next row are likewise loaded at the end of a tick.
// Two CTAs per SM (109 KB of rings each, 128 registers per thread at launch)
// = 16 warps and four phase instances in flight instead of two.  Every value
// comes from the same device functions in the same operation order as
// stencil_body, so F, J w, y' and p' are bitwise the one-role kernel's; only
// the order of the per-block norm partial sums differs.
// Ring lifetimes (write tick -> read tick): PD s -> s+1 (2 slots), FX s ->
// s+3 (4), FY s -> s+4 (5), GX s -> s+2 (3), DGY s -> s+1 (2).
// (Round 2 also measured a three-role variant with cp.async.bulk rows: 1.40
// ms per 2048^2 term, commit bd8cda0.)
constexpr int W2_ROLE = 128, W2_THREADS = 2 * W2_ROLE;
constexpr int W2_PD = 2, W2_FX = 4, W2_FY = 5, W2_GX = 3, W2_DGY = 2;
#ifndef XB_W2_AB
#define XB_W2_AB 160   // registers of warpgroup AB (C gets 256 - AB: the launch's 2 x 128)
#endif
#ifndef XB_W2_LOOK
#define XB_W2_LOOK 0   // AB's offset in the terms that read p
#endif
// the even Leja term keeps three epilogue operand rows (F(u), y, p) in C's
// registers across the barrier: give C 8 more there
template <int MODE, int PM>
__host__ __device__ constexpr int w2_reg_ab() { return (MODE == MODE_LEJA && PM != PM_SKIP) ? XB_W2_AB + XB_W2_LOOK : XB_W2_AB; }

struct Ws2Smem {
  double pd[W2_PD][NPD][W2_ROLE];
  double fx[W2_FX][NFX][W2_ROLE];
  double fy[W2_FY][NFY][W2_ROLE];
  double gx[W2_GX][NG][W2_ROLE];
  double dgy[W2_DGY][NG][W2_ROLE];
};

size_t stencil_ws_smem_bytes() { return sizeof(Ws2Smem); }

template <int MODE, int KX, int KY, int PM>
__global__ void __launch_bounds__(W2_THREADS, 2) stencil_ws_kernel(const StencilArgs a) {
  extern __shared__ __align__(16) unsigned char ws_raw[];
  Ws2Smem& S = *reinterpret_cast<Ws2Smem*>(ws_raw);
  __shared__ double red[W2_THREADS / 32];
  __shared__ int am_last;
  const Geom& g = a.g;
  const int tid = threadIdx.x;
  const int role = tid / W2_ROLE;   // 0: AB, 1: C
  const int t = tid - role * W2_ROLE;
  const int bid = blockIdx.x, nblk = gridDim.x;

  // ---- per-launch scalars (as stencil_body)
  double eps = a.eps;
  Divisor epsd = a.epsd;
  Divisor thd = epsd;
  const double* dir = a.dir;
  double* yout = nullptr;
  const double* pin = nullptr;
  double* pout = nullptr;
  double dt = 0.0, q = 0.0, xim = 0.0, cm = 0.0, pcoef = 0.0;
  int ppend = 0, pm_rt = PM_STORE, zero_dir = 0;
  if (MODE == MODE_LEJA) {
    const volatile LejaCtl* c = a.ctl;
    if (c->status != LJ_RUNNING) return;
    const int cur = c->cur, m = c->m;
    eps = c->eps;
    epsd.d = c->epsd.d; epsd.r = c->epsd.r; epsd.kind = c->epsd.kind;
    thd.d = c->thetad.d; thd.r = c->thetad.r; thd.kind = c->thetad.kind;
    zero_dir = c->zero_dir;
    dir = a.ybuf[cur];
    yout = a.ybuf[cur ^ 1];
    const int pc = c->pcur;
    pin = a.pbuf[pc];
    pout = a.pbuf[pc ^ 1];
    ppend = c->ppend;
    pcoef = c->pend_coef;
    pm_rt = c->pmode;
    if (PM != PM_ANY && pm_rt != PM) {
      if (bid == 0 && tid == 0) a.ctl->status = LJ_MODE_ERROR;
      return;
    }
    dt = c->dt;
    q = c->q;
    xim = __ldg(a.xi + (m - 1));
    cm = __ldg(a.coeffs + m);
  }
  if (MODE == MODE_JVP && a.pctl) {
    const PowerCtl* pc = a.pctl;
    if (pc->status != PW_RUNNING) return;
    eps = pc->eps;
    epsd = pc->epsd;
  }
  const int pmode = (PM == PM_ANY) ? pm_rt : PM;
  const bool pread = (pmode != PM_SKIP);
  const bool pstore = (pmode == PM_STORE || pmode == PM_LOOK);
  const bool padd = (PM == PM_LOOK) ? true : (PM == PM_SKIP ? false : (ppend != 0));
  const bool pnorm2 = (pmode == PM_LOOK);
  const unsigned plane = (unsigned)g.plane;

  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  int bad = 0;

  if (MODE == MODE_LEJA && zero_dir) {
    // jvp of a zero vector is exactly zero and costs no RHS call (linearize.py:63-64)
    const long long n = (long long)NF * g.plane;
    for (long long i = (long long)bid * W2_THREADS + tid; i < n; i += (long long)nblk * W2_THREADS) {
      const double y = __ldg(dir + i);
      const double yn = __dsub_rn(__ddiv_rn(__dsub_rn(__dmul_rn(dt, 0.0), __dmul_rn(q, y)), thd.d),
                                  __dmul_rn(xim, y));
      yout[i] = yn;
      double pn = 0.0;
      if (pread) {
        double pb = __ldg(pin + i);
        if (padd) {
          pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
          if (pnorm2) acc2 = __fma_rn(pb, pb, acc2);
        }
        pn = __dadd_rn(pb, __dmul_rn(cm, yn));
        if (pstore) pout[i] = pn;
      }
      acc0 = __fma_rn(yn, yn, acc0);
      acc1 = __fma_rn(pn, pn, acc1);
    }
  } else if (role == 0) {
    // ================================================================ AB
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(w2_reg_ab<MODE, PM>()));
    const double* dsrc = (MODE == MODE_RHS) ? nullptr : dir;
    for (int unit = bid; unit < a.ws_nunits; unit += nblk) {
      const int ux = unit % a.ws_units_x, uy = unit / a.ws_units_x;
      const int X0 = ux * SOUT;
      const int Y0 = uy * a.ws_seg_rows;
      const int Y1 = min(Y0 + a.ws_seg_rows, g.ny);
      const int nrows = Y1 - Y0;
      int cs, flipx;
      col_source(X0 - 2 + t, g, cs, flipx);
      const int tl = max(t - 1, 0), tr = min(t + 1, W2_ROLE - 1);
      const int pf_f = (t >> 3) & 7;
      const int pf_c = min(max(X0 - 2 + (t & 7) * 16, 0), g.nx - 1);
      double pr1[NPD], pr2[NPD], gy1[NG], gy2[NG];
#pragma unroll
      for (int k = 0; k < NPD; ++k) pr1[k] = pr2[k] = 0.0;
#pragma unroll
      for (int k = 0; k < NG; ++k) gy1[k] = gy2[k] = 0.0;
      // state (and direction) of the row the next tick consumes
      double nu[NF], nd[NF];
      int nflip;
      {
        const RowSrc rs = row_source(Y0 - 2, g, a.u, dsrc, g.halo_lo_dir, g.halo_hi_dir);
        nflip = rs.flip;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          nu[f] = __ldg(rs.u + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
          if (MODE != MODE_RHS) nd[f] = __ldg(rs.d + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
        }
      }
      const int nt = nrows + 5;
      for (int s = 0; s < nt; ++s) {
        const int r = Y0 - 2 + s;
        if (s <= nrows + 3) {
          // L2 prefetch of the row loaded two ticks from now: one 128-B line
          // per thread (8 lines per field row, u then the direction)
          {
            const int rp = r + 2;
            if (s + 2 <= nrows + 3 && rp >= 0 && rp < g.ny && (MODE != MODE_RHS || t < 64)) {
              const double* base = (t < 64) ? a.u : dsrc;
              asm volatile("prefetch.global.L2 [%0];" ::"l"(
                  base + ((unsigned)pf_f * plane + (unsigned)rp * (unsigned)g.nx + (unsigned)pf_c)));
            }
          }
          // ---- P1: row r
          double x[NF];
#pragma unroll
          for (int f = 0; f < NF; ++f)
            x[f] = (MODE == MODE_RHS) ? nu[f] : __dadd_rn(nu[f], __dmul_rn(eps, nd[f]));
          if (flipx) { x[MX] = -x[MX]; x[BX] = -x[BX]; }
          if (nflip) { x[MY] = -x[MY]; x[BY] = -x[BY]; }
          Prim p;
          primitives<KX == DIV_IEEE>(x, g, p);
          double pn[NPD];
          pn[PD_VX] = p.vx;
          pn[PD_VY] = p.vy;
          pn[PD_VZ] = p.vz;
          pn[PD_BX] = p.bx;
          pn[PD_BY] = p.by;
          pn[PD_BZ] = p.bz;
          pn[PD_T] = p.temp;
          pn[PD_B2] = p.b2;
#pragma unroll
          for (int k = 0; k < NPD; ++k) S.pd[s % W2_PD][k][t] = pn[k];
          {
            double fv[NFX];
            flux_x<KX == DIV_IEEE>(p, g, fv);
#pragma unroll
            for (int k = 0; k < NFX; ++k) S.fx[s % W2_FX][k][t] = fv[k];
            flux_y<KX == DIV_IEEE>(p, g, fv);
#pragma unroll
            for (int k = 0; k < NFY; ++k) S.fy[s % W2_FY][k][t] = fv[k];
          }
          // ---- P2: diffusive fluxes of row r-1 (x-neighbours from last tick's PD)
          if (diff_on<KX>(g) && s >= 2) {
            const int sp = (s - 1) % W2_PD;
            double xl[NPD], xr[NPD];
#pragma unroll
            for (int k = 0; k < NPD; ++k) {
              xl[k] = S.pd[sp][k][tl];
              xr[k] = S.pd[sp][k][tr];
            }
            double gxv[NG], gyv[NG];
            diffusive_fluxes<KX, KY>(xl, xr, pr2, pn, pr1, g, gxv, gyv);
#pragma unroll
            for (int k = 0; k < NG; ++k) S.gx[s % W2_GX][k][t] = gxv[k];
            if (s >= 4) {
              // +dGY/2dy term of row r-2 (mhd.py:223), divided here
#pragma unroll
              for (int k = 0; k < NG; ++k)
                S.dgy[s % W2_DGY][k][t] = qdiv<KY>(__dsub_rn(gyv[k], gy2[k]), g.h2y);
            }
#pragma unroll
            for (int k = 0; k < NG; ++k) { gy2[k] = gy1[k]; gy1[k] = gyv[k]; }
          }
#pragma unroll
          for (int k = 0; k < NPD; ++k) { pr2[k] = pr1[k]; pr1[k] = pn[k]; }
          // ---- loads of row r+1, in flight across the barrier
          if (s + 1 <= nrows + 3) {
            const RowSrc rs = row_source(r + 1, g, a.u, dsrc, g.halo_lo_dir, g.halo_hi_dir);
            nflip = rs.flip;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              nu[f] = __ldg(rs.u + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
              if (MODE != MODE_RHS) nd[f] = __ldg(rs.d + (rs.off + (unsigned)cs + (unsigned)f * rs.fs));
            }
          }
        }
        __syncthreads();
      }
    }
    asm volatile("setmaxnreg.dec.sync.aligned.u32 128;");
  } else {
    // ================================================================ C
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(256 - w2_reg_ab<MODE, PM>()));
    for (int unit = bid; unit < a.ws_nunits; unit += nblk) {
      const int ux = unit % a.ws_units_x, uy = unit / a.ws_units_x;
      const int X0 = ux * SOUT;
      const int Y0 = uy * a.ws_seg_rows;
      const int Y1 = min(Y0 + a.ws_seg_rows, g.ny);
      const int nrows = Y1 - Y0;
      const int c_out = X0 - 2 + t;
      const bool col_ok = (t >= 2) && (t < W2_ROLE - 2) && (c_out < g.nx);
      const int tl = max(t - 1, 0), tr = min(t + 1, W2_ROLE - 1);
      double efu[NF], ey[NF], ep[NF];
      // F(u) and y of the next output row are loaded at the end of a tick (in
      // flight across the barrier); p, only read by the even terms, at the
      // start of the row's own work after an L2 prefetch one tick earlier
      // (keeps C's register peak within its share)
      // L2 prefetch of an output row's epilogue operands (two ticks ahead):
      // one 128-B line per thread, 8 lines per field row
      const int pf_f = (t >> 3) & 7;
      const int pf_c = min(max(X0 + (t & 7) * 16, 0), g.nx - 1);
      auto prefetch_ops = [&](int row) {
        if (MODE == MODE_RHS || row < 0 || row >= Y1) return;
        const unsigned i = (unsigned)row * (unsigned)g.nx + (unsigned)pf_c + (unsigned)pf_f * plane;
        if (t < 64) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.fu + i));
        } else if (MODE == MODE_LEJA) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(dir + i));
        }
        if (MODE == MODE_LEJA && pread && t < 64)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pin + i));
      };
      auto load_ops = [&](int row) {
        const unsigned ob = (unsigned)row * (unsigned)g.nx + (unsigned)c_out;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const unsigned i = ob + (unsigned)f * plane;
          efu[f] = __ldg(a.fu + i);
          if (MODE == MODE_LEJA) ey[f] = __ldg(dir + i);
        }
      };
      const int nt = nrows + 5;
      for (int s = 0; s < nt; ++s) {
        const int rC = Y0 - 5 + s;
        if (s >= 2) prefetch_ops(rC + 2);
        if (MODE != MODE_RHS && col_ok && s == 4) load_ops(Y0);   // first output row
        if (s >= 5 && col_ok) {
          const unsigned obase = (unsigned)rC * (unsigned)g.nx + (unsigned)c_out;
          if (MODE == MODE_LEJA && pread) {
#pragma unroll
            for (int f = 0; f < NF; ++f) ep[f] = __ldg(pin + obase + (unsigned)f * plane);
          }
          double F[NF];
          {
            const int sx = (s - 3) % W2_FX;
            double aa[NFX], bb[NFX];
#pragma unroll
            for (int k = 0; k < NFX; ++k) { aa[k] = S.fx[sx][k][tr]; bb[k] = S.fx[sx][k][tl]; }
#pragma unroll
            for (int k = 0; k < NFX; ++k)
              F[fx_field(k)] = -qdiv<KX>(__dsub_rn(aa[k], bb[k]), g.h2x);
          }
          F[BX] = -0.0;
          {
            // -(dFY/2dy): FY rows rC+1 and rC-1 of this column (mhd.py:178)
            const int s1 = (s - 2) % W2_FY, s3 = (s - 4) % W2_FY;
#pragma unroll
            for (int k = 0; k < NFY; ++k) {
              const int f = fy_field(k);
              F[f] = __dsub_rn(F[f], qdiv<KY>(__dsub_rn(S.fy[s1][k][t], S.fy[s3][k][t]), g.h2y));
            }
          }
          F[BY] = __dsub_rn(F[BY], 0.0);
          if (diff_on<KX>(g)) {
            const int sgx = (s - 2) % W2_GX, sgy = (s - 1) % W2_DGY;
            double gr[NG], gl[NG];
#pragma unroll
            for (int k = 0; k < NG; ++k) { gr[k] = S.gx[sgx][k][tr]; gl[k] = S.gx[sgx][k][tl]; }
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BX] = __dadd_rn(F[BX], 0.0);
            F[MX] = __dadd_rn(F[MX], qdiv<KX>(__dsub_rn(gr[0], gl[0]), g.h2x));
            F[MY] = __dadd_rn(F[MY], qdiv<KX>(__dsub_rn(gr[1], gl[1]), g.h2x));
            F[MZ] = __dadd_rn(F[MZ], qdiv<KX>(__dsub_rn(gr[2], gl[2]), g.h2x));
            F[BY] = __dadd_rn(F[BY], qdiv<KX>(__dsub_rn(gr[3], gl[3]), g.h2x));
            F[BZ] = __dadd_rn(F[BZ], qdiv<KX>(__dsub_rn(gr[4], gl[4]), g.h2x));
            F[EN] = __dadd_rn(F[EN], qdiv<KX>(__dsub_rn(gr[5], gl[5]), g.h2x));
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BY] = __dadd_rn(F[BY], 0.0);
            F[MX] = __dadd_rn(F[MX], S.dgy[sgy][0][t]);
            F[MY] = __dadd_rn(F[MY], S.dgy[sgy][1][t]);
            F[MZ] = __dadd_rn(F[MZ], S.dgy[sgy][2][t]);
            F[BX] = __dadd_rn(F[BX], S.dgy[sgy][3][t]);
            F[BZ] = __dadd_rn(F[BZ], S.dgy[sgy][4][t]);
            F[EN] = __dadd_rn(F[EN], S.dgy[sgy][5][t]);
          }
          {
            unsigned ex = 0;
#pragma unroll
            for (int f = 0; f < NF; ++f)
              ex = max(ex, (unsigned)__double2hiint(F[f]) & 0x7ff00000u);
            bad |= (ex == 0x7ff00000u);
          }
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const unsigned i = obase + (unsigned)f * plane;
            if (MODE == MODE_RHS) {
              a.out[i] = F[f];
            } else if (MODE == MODE_JVP) {
              const double jv = qdiv<DIV_MK2>(__dsub_rn(F[f], efu[f]), epsd);
              a.out[i] = jv;
              acc0 = __fma_rn(jv, jv, acc0);
            } else {
              const double w = qdiv<DIV_MK2>(__dsub_rn(F[f], efu[f]), epsd);
              const double y = ey[f];
              const double yn = __dsub_rn(
                  qdiv<DIV_MK2>(__dsub_rn(__dmul_rn(dt, w), __dmul_rn(q, y)), thd),
                  __dmul_rn(xim, y));
              yout[i] = yn;
              double pn = 0.0;
              if (pread) {
                double pb = ep[f];
                if (padd) {
                  pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
                  if (pnorm2) acc2 = __fma_rn(pb, pb, acc2);
                }
                pn = __dadd_rn(pb, __dmul_rn(cm, yn));
                if (pstore) pout[i] = pn;
              }
              acc0 = __fma_rn(yn, yn, acc0);
              acc1 = __fma_rn(pn, pn, acc1);
            }
          }
          // epilogue operands of the next output row, in flight across the barrier
          if (MODE != MODE_RHS && rC + 1 < Y1) load_ops(rC + 1);
        }
        __syncthreads();
      }
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 128;");
  }

  if (bad) atomicOr(a.bad, 1);
  if (MODE == MODE_RHS) return;

  // ---- block partials and the last block's reduction / control update
  constexpr bool NEED_S2 = (MODE == MODE_LEJA) && (PM == PM_ANY || PM == PM_LOOK);
  const double s0 = block_sum(acc0, red);
  const double s1 = (MODE == MODE_LEJA && PM != PM_SKIP) ? block_sum(acc1, red) : 0.0;
  const double s2 = NEED_S2 ? block_sum(acc2, red) : 0.0;
  if (tid == 0) {
    a.partials[3 * bid] = s0;
    a.partials[3 * bid + 1] = s1;
    a.partials[3 * bid + 2] = s2;
    __threadfence();
    const unsigned prev = atomicAdd(a.ticket, 1u);
    am_last = (prev == (unsigned)nblk - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  if (tid < 32) {
    const double sy = sum_partials(a.partials, nblk, 3, 0);
    const double sp = (MODE == MODE_LEJA && PM != PM_SKIP) ? sum_partials(a.partials, nblk, 3, 1)
                                                            : 0.0;
    const double sp2 = NEED_S2 ? sum_partials(a.partials, nblk, 3, 2) : 0.0;
    if (tid == 0) {
      if (MODE == MODE_JVP && a.pctl) {
        power_after_jvp(a.pctl, sy, *((volatile int*)a.bad));
      } else if (MODE == MODE_JVP) {
        a.result[0] = sqrt(sy);
      } else if (a.ext_sums) {
        a.ext_sums[0] = sy;
        a.ext_sums[1] = sp;
        a.ext_sums[2] = sp2;
        a.ext_sums[3] = *((volatile int*)a.bad) ? 1.0 : 0.0;
      } else {
        const int flag = *((volatile int*)a.bad);
        leja_finalize(a.ctl, sy, sp, sp2, flag, !zero_dir, cm);
      }
      if (MODE == MODE_JVP) a.result[1] = sy;
      *a.ticket = 0u;
    }
  }
}

// Units of the two-role kernel: column strips of SOUT outputs x y-segments
// over two persistent CTAs per SM; a segment costs 5 warm-up ticks.
void stencil_ws_plan(const Geom& g, int nsm, int& units_x, int& nunits, int& seg_rows,
                     int& grid) {
  units_x = nunits = seg_rows = grid = 0;
  const char* e = std::getenv("XMHD_WS");
  if (!e || std::atoi(e) == 0) return;
  if (g.nx < 2 * W2_ROLE || g.ny < 16) return;
  units_x = (g.nx + SOUT - 1) / SOUT;
  const int slots = 2 * nsm;
  double best = 1e300;
  int best_seg = g.ny;
  for (int s = 1; s <= g.ny; ++s) {
    const int nseg = (g.ny + s - 1) / s;
    const long long units = (long long)units_x * nseg;
    const long long waves = (units + slots - 1) / slots;
    const double cost = (double)waves * (s + 5);
    if (cost < best - 1e-9) { best = cost; best_seg = s; }
  }
  seg_rows = best_seg;
  nunits = units_x * ((g.ny + seg_rows - 1) / seg_rows);
  grid = nunits < slots ? nunits : slots;
}

namespace {

template <int MODE, int KX, int KY, int PM>
cudaError_t launch_ws_one(const StencilArgs& a, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaError_t err = cudaFuncSetAttribute(stencil_ws_kernel<MODE, KX, KY, PM>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)stencil_ws_smem_bytes());
    if (err != cudaSuccess) return err;
    done = true;
  }
  stencil_ws_kernel<MODE, KX, KY, PM><<<a.ws_grid, W2_THREADS, stencil_ws_smem_bytes(), s>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t stencil_smem_bytes() {
  return sizeof(double) * (size_t)SW *
         (RING_PD * NPD + RING_FX * NFX + RING_FY * NFY + RING_GX * NG);
}

// Work decomposition: column strips of SOUT outputs x y-segments; the
// persistent grid is 2 CTAs per SM.  The segment length trades warm-up rows
// (4 per segment) against wave quantisation of the units over the grid.
template <int MODE, int KX, int KY>
cudaError_t set_smem_attr() {
  return cudaFuncSetAttribute(stencil_kernel<MODE, KX, KY>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)stencil_smem_bytes());
}

// Resident CTAs per SM of the fused iteration kernel (registers + shared memory).
int stencil_occupancy() {
  static int occ = 0;
  if (occ) return occ;
  int n = 0;
  if (set_smem_attr<MODE_LEJA, DIV_MUL, DIV_MUL>() == cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &n, stencil_kernel<MODE_LEJA, DIV_MUL, DIV_MUL>, SW, stencil_smem_bytes()) ==
          cudaSuccess &&
      n > 0) {
    occ = n;
  } else {
    cudaGetLastError();
    occ = 2;
  }
  return occ;
}

void stencil_plan(const Geom& g, int nsm, int& units_x, int& nunits, int& seg_rows, int& grid) {
  units_x = (g.nx + SOUT - 1) / SOUT;
  const int slots = stencil_occupancy() * nsm;
  double best = 1e300;
  int best_seg = g.ny;
  for (int s = 1; s <= g.ny; ++s) {
    const int nseg = (g.ny + s - 1) / s;
    const long long units = (long long)units_x * nseg;
    const long long waves = (units + slots - 1) / slots;
    const double cost = (double)waves * (s + 4);   // row steps of the busiest CTA
    if (cost < best - 1e-9) { best = cost; best_seg = s; }
  }
  seg_rows = best_seg;
  nunits = units_x * ((g.ny + seg_rows - 1) / seg_rows);
  grid = nunits < slots ? nunits : slots;
}

namespace {

template <int MODE, int KX, int KY, int PM = PM_ANY>
cudaError_t launch_one(const StencilArgs& a, int grid, cudaStream_t s) {
  static bool attr_done = false;
  const size_t smem = stencil_smem_bytes();
  if (!attr_done) {
    cudaError_t err = cudaFuncSetAttribute(stencil_kernel<MODE, KX, KY, PM>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
    if (err != cudaSuccess) return err;
    attr_done = true;
  }
  stencil_kernel<MODE, KX, KY, PM><<<grid, SW, smem, s>>>(a);
  return cudaGetLastError();
}

// Calls f(KX, KY) with the compile-time division kinds of the geometry.
template <typename F>
cudaError_t with_div_kinds(const Geom& g, F&& f) {
  using M = std::integral_constant<int, DIV_MUL>;
  using K1 = std::integral_constant<int, DIV_MK1>;
  using K2 = std::integral_constant<int, DIV_MK2>;
  using IE = std::integral_constant<int, DIV_IEEE>;
  const int kx = g.h2x.kind, ky = g.h2y.kind;
  // the generic variant (correctly rounded divisions, any mu0, diffusive or
  // not) serves every geometry; the others are compiled for mu0 == 1.0 and a
  // diffusive operator (common.cuh over_mu0, diff_on)
  if (kx == DIV_IEEE || ky == DIV_IEEE || !g.mu0_one || !g.diffusive) return f(IE{}, IE{});
  if (kx == DIV_MUL && ky == DIV_MUL) return f(M{}, M{});
  // a power-of-two divisor is also exact on the one-correction path
  const int x2 = (kx == DIV_MK2), y2 = (ky == DIV_MK2);
  if (x2 && y2) return f(K2{}, K2{});
  if (x2) return f(K2{}, K1{});
  if (y2) return f(K1{}, K2{});
  return f(K1{}, K1{});
}

template <int MODE, int PM = PM_ANY>
cudaError_t launch_mode(const StencilArgs& a, int grid, cudaStream_t s) {
  if (a.ws_grid > 0) {   // warp-specialized TMA kernel (even nx, wide grids)
    return with_div_kinds(a.g, [&](auto X, auto Y) {
      return launch_ws_one<MODE, decltype(X)::value, decltype(Y)::value, PM>(a, s);
    });
  }
  return with_div_kinds(a.g, [&](auto X, auto Y) {
    return launch_one<MODE, decltype(X)::value, decltype(Y)::value, PM>(a, grid, s);
  });
}

template <typename K>
cudaError_t smem_attr_once(K kernel, bool& done) {
  if (done) return cudaSuccess;
  cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)stencil_smem_bytes());
  if (err == cudaSuccess) done = true;
  return err;
}

template <int KX, int KY, int PM>
cudaError_t launch_peer_one(const StencilArgs& a, int grid, cudaStream_t s) {
  static bool done = false;
  cudaError_t err = smem_attr_once(leja_peer_kernel<KX, KY, PM>, done);
  if (err != cudaSuccess) return err;
  leja_peer_kernel<KX, KY, PM><<<grid, SW, stencil_smem_bytes(), s>>>(a);
  return cudaGetLastError();
}

template <int KX, int KY, int PM>
cudaError_t launch_emul_one(const StencilArgs* args_dev, int nranks, int nblk, cudaStream_t s) {
  static bool done = false;
  cudaError_t err = smem_attr_once(leja_emul_kernel<KX, KY, PM>, done);
  if (err != cudaSuccess) return err;
  void* kargs[] = {(void*)&args_dev, (void*)&nblk};
  return cudaLaunchCooperativeKernel((const void*)leja_emul_kernel<KX, KY, PM>,
                                     dim3(nranks * nblk), dim3(SW), kargs, stencil_smem_bytes(),
                                     s);
}

template <int KX, int KY>
cudaError_t launch_loop_one(const StencilArgs& a, int grid, cudaStream_t s) {
  static bool done = false;
  cudaError_t err = smem_attr_once(leja_loop_kernel<KX, KY>, done);
  if (err != cudaSuccess) return err;
  void* kargs[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((const void*)leja_loop_kernel<KX, KY>, dim3(grid), dim3(SW),
                                     kargs, stencil_smem_bytes(), s);
}

}  // namespace

cudaError_t launch_leja_loop(const StencilArgs& a, int grid, cudaStream_t s) {
  return with_div_kinds(a.g, [&](auto X, auto Y) {
    return launch_loop_one<decltype(X)::value, decltype(Y)::value>(a, grid, s);
  });
}

// Co-resident blocks of the loop kernel on the whole device.
int leja_loop_max_blocks(int nsm) {
  int n = 0;
  static bool done = false;
  if (smem_attr_once(leja_loop_kernel<DIV_MUL, DIV_MUL>, done) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, leja_loop_kernel<DIV_MUL, DIV_MUL>, SW,
                                                    stencil_smem_bytes()) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n * nsm;
}

cudaError_t launch_leja_peer(const StencilArgs& a, int grid, int pmode, cudaStream_t s) {
  return with_div_kinds(a.g, [&](auto X, auto Y) {
    constexpr int KX = decltype(X)::value, KY = decltype(Y)::value;
    switch (pmode) {
      case PM_SKIP: return launch_peer_one<KX, KY, PM_SKIP>(a, grid, s);
      case PM_LOOK: return launch_peer_one<KX, KY, PM_LOOK>(a, grid, s);
      default: return launch_peer_one<KX, KY, PM_ANY>(a, grid, s);
    }
  });
}

cudaError_t launch_leja_emul(const StencilArgs* args_dev, const StencilArgs& a0, int nranks,
                             int nblk, int pmode, cudaStream_t s) {
  return with_div_kinds(a0.g, [&](auto X, auto Y) {
    constexpr int KX = decltype(X)::value, KY = decltype(Y)::value;
    switch (pmode) {
      case PM_SKIP: return launch_emul_one<KX, KY, PM_SKIP>(args_dev, nranks, nblk, s);
      case PM_LOOK: return launch_emul_one<KX, KY, PM_LOOK>(args_dev, nranks, nblk, s);
      default: return launch_emul_one<KX, KY, PM_ANY>(args_dev, nranks, nblk, s);
    }
  });
}

// Co-resident blocks of the emulation kernel on the whole device.
int leja_emul_max_blocks(int nsm) {
  int n = 0;
  static bool done = false;
  if (smem_attr_once(leja_emul_kernel<DIV_MUL, DIV_MUL>, done) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, leja_emul_kernel<DIV_MUL, DIV_MUL>, SW,
                                                    stencil_smem_bytes()) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n * nsm;
}

// ---------------------------------------------------------------------------
// Small-grid Leja loop: 2D tiles, all Newton terms in one cooperative launch.
//
// On grids of up to ~1M cells a term of the sliding-window kernel is latency
// bound (a y-segment needs 4 warm-up rows, so a CTA spends 5 dependent row
// steps on one output row).  Here a CTA computes a TX x TY tile in three
// dependent phases over shared memory: (1) x = u + eps*y, primitives and
// ideal fluxes on the tile plus its 2-cell halo, (2) the diffusive fluxes on
// the level-1 ring, (3) the differenced RHS, the FD-JVP and the Newton update
// for the tile.  Every per-cell value is the same IEEE operation sequence as
// in stencil_body (same device functions, same association order), so F bits
// are identical; only the order of the norm sums differs (fixed per grid).
//
// Terms are separated by one grid-wide barrier: each block publishes
// [sum y'^2, sum p'^2, bad] into a parity-double-buffered slot, and after the
// barrier EVERY block sums the slots in the same fixed order and runs the
// reference's control update on its own shared-memory copy of the control
// block (identical in all blocks), so no second barrier or last-block ticket
// is needed.  Block 0 mirrors the control block to global memory.
// Measured and dropped: loading the next tile's phase-1 inputs during phases
// 2-3 of the current one (512^2: 40.3 us/term at 2 blocks/SM, 45.7 at 3 with
// spills, vs 38.2 without).
// Resident tile blocks per SM the register budget targets: 2 (210 registers,
// the shortest chain when every block holds one tile: 8.8 us/term at 128^2)
// or 3 (160 registers, more tiles in flight when blocks loop over several
// tiles: 37.9 vs 41.5 us/term at 512^2; 4 blocks: 38.4).
constexpr int TX = 16, TY = 8, TNT = TX * TY;        // outputs per tile = threads
constexpr int EX = TX + 4, EY = TY + 4, NE = EX * EY;  // tile + 2-cell halo
constexpr int FXW = TX + 2, NFXC = TY * FXW;           // FX / GX: rows [0,TY), cols [-1,TX]
constexpr int FYH = TY + 2, NFYC = FYH * TX;           // FY / GY: rows [-1,TY], cols [0,TX)
constexpr int GBW = TX + 2, NGB = (TY + 2) * GBW;      // level-1 box (corners skipped)

struct TileSmem {
  double pd[NPD][NE];
  double fx[NFX][NFXC];
  double fy[NFY][NFYC];
  double gx[NG][NFXC];
  double gy[NG][NFYC];
};

size_t tile_smem_bytes() { return sizeof(TileSmem); }

namespace {

// Row r (any integer) of the domain seen from a tile: rows beyond the 2-row
// halo only feed outputs outside the grid, so they are clamped into it (the
// loads stay in bounds); the halo itself follows row_source.
__device__ __forceinline__ RowSrc tile_row(int r, const Geom& g, const double* u, const double* d,
                                           const double* hlo_dir, const double* hhi_dir) {
  r = min(max(r, -2), g.ny + 1);
  return row_source(r, g, u, d, hlo_dir, hhi_dir);
}

}  // namespace

template <int KX, int KY, int MINB>
__global__ void __launch_bounds__(MINB == 1 ? 2 * TNT : TNT, MINB)
    leja_tile_loop_kernel(const StencilArgs a) {
  // MINB == 1: 256 threads per tile (grids with at most one tile per SM: the
  // halo phases take one pass instead of two); else 128 threads, MINB blocks/SM
  constexpr int NT = (MINB == 1) ? 2 * TNT : TNT;
  extern __shared__ __align__(16) double smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  __shared__ LejaCtl lc;
  __shared__ double red[4][NT / 32];
  cg::grid_group grid = cg::this_grid();
  const Geom& g = a.g;
  const int t = threadIdx.x;
  const int bid = blockIdx.x, nblk = gridDim.x;
  const int ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY, ntiles = ntx * nty;
  const unsigned plane = (unsigned)g.plane;
  if (t == 0) {
    lc = *a.ctl;
    // small grids are not bandwidth-bound: a fresh call stores p every term
    // (no interpolant schedule, the lean reduction path below)
    if (lc.m == 1 && !lc.ppend) {
      lc.defer = 0;
      lc.pmode = PM_STORE;
    }
  }
  __syncthreads();
  int par = 0;
  for (;;) {
    if (lc.status != LJ_RUNNING) break;
    const int cur = lc.cur, m = lc.m;
    const double eps = lc.eps, dt = lc.dt, q = lc.q;
    const Divisor epsd = lc.epsd, thd = lc.thetad;
    const int zero_dir = lc.zero_dir;
    const double* dir = a.ybuf[cur];
    double* yout = a.ybuf[cur ^ 1];
    const double* pin = a.pbuf[lc.pcur];
    double* pout = a.pbuf[lc.pcur ^ 1];
    const int ppend = lc.ppend;
    const double pcoef = lc.pend_coef;
    const int pmode = lc.pmode;
    const bool pread = (pmode != PM_SKIP), pstore = (pmode == PM_STORE || pmode == PM_LOOK);
    const double xim = __ldg(a.xi + (m - 1));
    const double cm = __ldg(a.coeffs + m);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    int bad = 0;

    if (zero_dir) {
      // jvp of a zero vector is exactly zero and costs no RHS call (linearize.py:63-64)
      const long long n = (long long)NF * g.plane;
      for (long long i = (long long)bid * NT + t; i < n; i += (long long)nblk * NT) {
        const double y = __ldcg(dir + i);
        const double yn = __dsub_rn(__ddiv_rn(__dsub_rn(__dmul_rn(dt, 0.0), __dmul_rn(q, y)), thd.d),
                                    __dmul_rn(xim, y));
        yout[i] = yn;
        acc0 = __fma_rn(yn, yn, acc0);
        if (pread) {
          double pb = __ldcg(pin + i);
          if (ppend) {
            pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
            if (pmode == PM_LOOK) acc2 = __fma_rn(pb, pb, acc2);
          }
          const double pn = __dadd_rn(pb, __dmul_rn(cm, yn));
          if (pstore) pout[i] = pn;
          acc1 = __fma_rn(pn, pn, acc1);
        }
      }
    } else {
      for (int tile = bid; tile < ntiles; tile += nblk) {
        const int X0 = (tile % ntx) * TX, Y0 = (tile / ntx) * TY;
        // output cell of this thread and its epilogue operands (issued first)
        const int oj = t / TX, oi = t - oj * TX;
        const bool is_out = (NT == TNT) || (t < TNT);
        const bool out_ok = is_out && (Y0 + oj < g.ny) && (X0 + oi < g.nx);
        const unsigned obase = out_ok ? (unsigned)(Y0 + oj) * (unsigned)g.nx + (unsigned)(X0 + oi) : 0u;
        double efu[NF], ey[NF], ep[NF];
        if (is_out) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const unsigned i = obase + (unsigned)f * plane;
            efu[f] = __ldg(a.fu + i);
            ey[f] = __ldcg(dir + i);
            if (pread) ep[f] = __ldcg(pin + i);
          }
        }
        // ---- phase 1: primitives and ideal fluxes on the tile + halo
#pragma unroll
        for (int h = 0; h < (NE + NT - 1) / NT; ++h) {
          const int e = t + h * NT;
          if (e < NE) {
            const int ej = e / EX, ei = e - ej * EX;
            const int j = ej - 2, i = ei - 2;
            const RowSrc rs = tile_row(Y0 + j, g, a.u, dir, g.halo_lo_dir, g.halo_hi_dir);
            int cs, flipx;
            col_source(X0 + i, g, cs, flipx);
            double x[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) {
              const unsigned k = rs.off + (unsigned)cs + (unsigned)f * rs.fs;
              x[f] = __dadd_rn(__ldg(rs.u + k), __dmul_rn(eps, __ldcg(rs.d + k)));
            }
            if (flipx) { x[MX] = -x[MX]; x[BX] = -x[BX]; }
            if (rs.flip) { x[MY] = -x[MY]; x[BY] = -x[BY]; }
            Prim p;
            primitives<KX == DIV_IEEE>(x, g, p);
            S.pd[PD_VX][e] = p.vx;
            S.pd[PD_VY][e] = p.vy;
            S.pd[PD_VZ][e] = p.vz;
            S.pd[PD_BX][e] = p.bx;
            S.pd[PD_BY][e] = p.by;
            S.pd[PD_BZ][e] = p.bz;
            S.pd[PD_T][e] = p.temp;
            S.pd[PD_B2][e] = p.b2;
            double fv[NFX];
            if (j >= 0 && j < TY && i >= -1 && i <= TX) {
              flux_x<KX == DIV_IEEE>(p, g, fv);
#pragma unroll
              for (int k = 0; k < NFX; ++k) S.fx[k][j * FXW + i + 1] = fv[k];
            }
            if (j >= -1 && j <= TY && i >= 0 && i < TX) {
              flux_y<KX == DIV_IEEE>(p, g, fv);
#pragma unroll
              for (int k = 0; k < NFY; ++k) S.fy[k][(j + 1) * TX + i] = fv[k];
            }
          }
        }
        __syncthreads();
        // ---- phase 2: diffusive fluxes on the level-1 ring (mhd.py:182-221)
        if (diff_on<KX>(g)) {
#pragma unroll
          for (int h = 0; h < (NGB + NT - 1) / NT; ++h) {
            const int e = t + h * NT;
            if (e < NGB) {
              const int bj = e / GBW, bi = e - bj * GBW;
              const int j = bj - 1, i = bi - 1;
              const bool in_gx = (j >= 0 && j < TY), in_gy = (i >= 0 && i < TX);
              if (in_gx || in_gy) {
                const int c = (j + 2) * EX + (i + 2);
                double xl[NPD], xr[NPD], yd[NPD], yu[NPD], own[NPD];
#pragma unroll
                for (int k = 0; k < NPD; ++k) {
                  xl[k] = S.pd[k][c - 1];
                  xr[k] = S.pd[k][c + 1];
                  yd[k] = S.pd[k][c - EX];
                  yu[k] = S.pd[k][c + EX];
                  own[k] = S.pd[k][c];
                }
                double gxv[NG], gyv[NG];
                diffusive_fluxes<KX, KY>(xl, xr, yd, yu, own, g, gxv, gyv);
                if (in_gx) {
#pragma unroll
                  for (int k = 0; k < NG; ++k) S.gx[k][j * FXW + i + 1] = gxv[k];
                }
                if (in_gy) {
#pragma unroll
                  for (int k = 0; k < NG; ++k) S.gy[k][(j + 1) * TX + i] = gyv[k];
                }
              }
            }
          }
        }
        __syncthreads();
        // ---- phase 3: output cell (oj, oi): RHS in the reference's order + Newton update
        if (out_ok) {
          const int cx = oj * FXW + oi + 1;         // FX / GX index of the cell
          const int cy = (oj + 1) * TX + oi;        // FY / GY index of the cell
          double F[NF];
#pragma unroll
          for (int k = 0; k < NFX; ++k)
            F[fx_field(k)] = -qdiv<KX>(__dsub_rn(S.fx[k][cx + 1], S.fx[k][cx - 1]), g.h2x);
          F[BX] = -0.0;
#pragma unroll
          for (int k = 0; k < NFY; ++k) {
            const int f = fy_field(k);
            F[f] = __dsub_rn(F[f], qdiv<KY>(__dsub_rn(S.fy[k][cy + TX], S.fy[k][cy - TX]), g.h2y));
          }
          F[BY] = __dsub_rn(F[BY], 0.0);
          if (diff_on<KX>(g)) {
            double gr[NG], gl[NG], gu[NG], gd[NG];
#pragma unroll
            for (int k = 0; k < NG; ++k) {
              gr[k] = S.gx[k][cx + 1];
              gl[k] = S.gx[k][cx - 1];
              gu[k] = S.gy[k][cy + TX];
              gd[k] = S.gy[k][cy - TX];
            }
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BX] = __dadd_rn(F[BX], 0.0);
            F[MX] = __dadd_rn(F[MX], qdiv<KX>(__dsub_rn(gr[0], gl[0]), g.h2x));
            F[MY] = __dadd_rn(F[MY], qdiv<KX>(__dsub_rn(gr[1], gl[1]), g.h2x));
            F[MZ] = __dadd_rn(F[MZ], qdiv<KX>(__dsub_rn(gr[2], gl[2]), g.h2x));
            F[BY] = __dadd_rn(F[BY], qdiv<KX>(__dsub_rn(gr[3], gl[3]), g.h2x));
            F[BZ] = __dadd_rn(F[BZ], qdiv<KX>(__dsub_rn(gr[4], gl[4]), g.h2x));
            F[EN] = __dadd_rn(F[EN], qdiv<KX>(__dsub_rn(gr[5], gl[5]), g.h2x));
            F[RHO] = __dadd_rn(F[RHO], 0.0);
            F[BY] = __dadd_rn(F[BY], 0.0);
            F[MX] = __dadd_rn(F[MX], qdiv<KY>(__dsub_rn(gu[0], gd[0]), g.h2y));
            F[MY] = __dadd_rn(F[MY], qdiv<KY>(__dsub_rn(gu[1], gd[1]), g.h2y));
            F[MZ] = __dadd_rn(F[MZ], qdiv<KY>(__dsub_rn(gu[2], gd[2]), g.h2y));
            F[BX] = __dadd_rn(F[BX], qdiv<KY>(__dsub_rn(gu[3], gd[3]), g.h2y));
            F[BZ] = __dadd_rn(F[BZ], qdiv<KY>(__dsub_rn(gu[4], gd[4]), g.h2y));
            F[EN] = __dadd_rn(F[EN], qdiv<KY>(__dsub_rn(gu[5], gd[5]), g.h2y));
          }
          unsigned ex = 0;
#pragma unroll
          for (int f = 0; f < NF; ++f) ex = max(ex, (unsigned)__double2hiint(F[f]) & 0x7ff00000u);
          bad |= (ex == 0x7ff00000u);
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const unsigned i = obase + (unsigned)f * plane;
            const double w = qdiv<DIV_MK2>(__dsub_rn(F[f], efu[f]), epsd);
            const double y = ey[f];
            const double yn = __dsub_rn(
                qdiv<DIV_MK2>(__dsub_rn(__dmul_rn(dt, w), __dmul_rn(q, y)), thd),
                __dmul_rn(xim, y));
            yout[i] = yn;
            acc0 = __fma_rn(yn, yn, acc0);
            if (pread) {
              double pb = ep[f];
              if (ppend) {
                pb = __dadd_rn(pb, __dmul_rn(pcoef, y));
                if (pmode == PM_LOOK) acc2 = __fma_rn(pb, pb, acc2);
              }
              const double pn = __dadd_rn(pb, __dmul_rn(cm, yn));
              if (pstore) pout[i] = pn;
              acc1 = __fma_rn(pn, pn, acc1);
            }
          }
        }
        __syncthreads();   // shared tiles are rewritten by the next tile
      }
    }

    // ---- term end: publish [sum y'^2, sum p'^2, sum pending p^2, bad], barrier,
    // every block reduces
    {
      double v[4] = {acc0, acc1, acc2, bad ? 1.0 : 0.0};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
      const int w = t >> 5, l = t & 31;
      if (l == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) red[k][w] = v[k];
      }
      __syncthreads();
      if (t == 0) {
        double* slot = a.partials + ((size_t)par * nblk + bid) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double sk = 0.0;
          for (int j = 0; j < NT / 32; ++j) sk += red[k][j];
          slot[k] = sk;
        }
      }
    }
    grid.sync();
    if (t < 32) {
      // the four sums in one pass over the slots (fixed order: lanes stride
      // the blocks, then one shuffle tree per sum)
      const double* base = a.partials + (size_t)par * nblk * 4;
      double r4[4] = {0.0, 0.0, 0.0, 0.0};
      for (int b = t; b < nblk; b += 32) {
        const double2 lo = __ldcg(reinterpret_cast<const double2*>(base + 4 * b));
        const double2 hi = __ldcg(reinterpret_cast<const double2*>(base + 4 * b + 2));
        r4[0] += lo.x;
        r4[1] += lo.y;
        r4[2] += hi.x;
        r4[3] += hi.y;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r4[k] += __shfl_xor_sync(0xffffffffu, r4[k], o);
      const double sy = r4[0], sp = r4[1], sp2 = r4[2], sb = r4[3];
      if (t == 0) {
        leja_finalize(&lc, sy, sp, sp2, sb > 0.0, !zero_dir, cm);
        if (bid == 0) *a.ctl = lc;
      }
    }
    __syncthreads();
    par ^= 1;
  }
}

namespace {

template <int KX, int KY, int MINB>
cudaError_t launch_tile_loop_one(const StencilArgs& a, int grid, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaError_t err = cudaFuncSetAttribute(leja_tile_loop_kernel<KX, KY, MINB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)tile_smem_bytes());
    if (err != cudaSuccess) return err;
    done = true;
  }
  void* kargs[] = {(void*)&a};
  return cudaLaunchCooperativeKernel((const void*)leja_tile_loop_kernel<KX, KY, MINB>, dim3(grid),
                                     dim3(MINB == 1 ? 2 * TNT : TNT), kargs, tile_smem_bytes(), s);
}

template <int MINB>
int tile_blocks_per_sm() {
  int n = 0;
  if (cudaFuncSetAttribute(leja_tile_loop_kernel<DIV_MUL, DIV_MUL, MINB>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tile_smem_bytes()) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &n, leja_tile_loop_kernel<DIV_MUL, DIV_MUL, MINB>, MINB == 1 ? 2 * TNT : TNT,
          tile_smem_bytes()) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // namespace

// minb: 1 (256 threads per tile), 2 or 3 (128 threads; leja_tile_loop_grid's choice).
cudaError_t launch_leja_tile_loop(const StencilArgs& a, int grid, int minb, cudaStream_t s) {
  return with_div_kinds(a.g, [&](auto X, auto Y) {
    constexpr int KX = decltype(X)::value, KY = decltype(Y)::value;
    if (minb == 1) return launch_tile_loop_one<KX, KY, 1>(a, grid, s);
    if (minb == 3) return launch_tile_loop_one<KX, KY, 3>(a, grid, s);
    return launch_tile_loop_one<KX, KY, 2>(a, grid, s);
  });
}

// Grid of the tile loop (one block per tile, capped at the co-resident blocks)
// and its occupancy variant: 2 blocks / SM when every block holds one tile,
// else 3 (more tiles in flight).  0 when the kernel cannot be resident.
int leja_tile_loop_grid(const Geom& g, int nsm, int* minb) {
  const long long ntiles = (long long)((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
  const int n2 = tile_blocks_per_sm<2>();
  int mb = 2, n = n2;
  const char* force = std::getenv("XMHD_TILE_MINB");   // A/B knob: 1, 2 or 3
  const int fmb = force ? std::atoi(force) : 0;
  const int n1 = (fmb == 0 || fmb == 1) ? tile_blocks_per_sm<1>() : 0;
  if (fmb == 3) {
    const int n3 = tile_blocks_per_sm<3>();
    if (n3 > 0) { mb = 3; n = n3; }
  } else if ((fmb == 1 || (fmb == 0 && ntiles <= (long long)nsm)) && n1 > 0) {
    mb = 1;   // every tile on its own SM: 256 threads per tile
    n = n1;
  } else if (fmb == 0 && ntiles > (long long)n2 * nsm) {
    const int n3 = tile_blocks_per_sm<3>();
    if (n3 > n2) { mb = 3; n = n3; }
  }
  if (n < 1) return 0;
  *minb = mb;
  const long long cap = (long long)n * nsm;
  return (int)(ntiles < cap ? ntiles : cap);
}

// One Newton term with the kernel variant compiled for its interpolant mode
// (leja_pmode of the term: lookahead pairs on one domain).
cudaError_t launch_leja_term(const StencilArgs& a, int grid, int pmode, cudaStream_t s) {
  switch (pmode) {
    case PM_SKIP: return launch_mode<MODE_LEJA, PM_SKIP>(a, grid, s);
    case PM_LOOK: return launch_mode<MODE_LEJA, PM_LOOK>(a, grid, s);
    case PM_STORE: return launch_mode<MODE_LEJA, PM_STORE>(a, grid, s);
    default: return launch_mode<MODE_LEJA>(a, grid, s);
  }
}

cudaError_t launch_stencil(int mode, const StencilArgs& a, int grid, cudaStream_t s) {
  switch (mode) {
    case MODE_RHS: return launch_mode<MODE_RHS>(a, grid, s);
    case MODE_JVP: return launch_mode<MODE_JVP>(a, grid, s);
    default: return launch_mode<MODE_LEJA>(a, grid, s);
  }
}

}  // namespace xb
