// Host C++ port of the phi_l divided-difference routine (phi.py:99-144) that
// feeds the Leja Newton coefficients (leja.py:84-100).
//
// Bitwise contract with the NumPy routine: every element-wise step is one IEEE
// operation in the same order (compiled with -ffp-contract=off, no fast-math),
// the substep count uses the same libm log2/ceil, and the bidiagonal matvec
// computes out[i] = RN(RN(d[i]*w[i]) + RN(e*w[i-1])) exactly like
// `out = diag*w; out[1:] += sub*w[:-1]`, then `/ k` and `new += term`.
// The element loop is SIMD-vectorised (per-element IEEE ops, no reassociation);
// target_clones picks AVX-512 / AVX2 / baseline at load time.
#include <cmath>
#include <cstring>
#include <vector>

#include "xmhd_b200.h"

namespace {

// One Taylor term of one substep: term <- (diag*term + sub*shift(term)) / k,
// acc <- acc + term.  `prev` holds the previous term (read-only here).
__attribute__((target_clones("avx512f", "avx2", "default")))
void taylor_term(int dim, const double* __restrict diag, double sub, double dk,
                 const double* __restrict prev, double* __restrict next,
                 double* __restrict acc) {
  next[0] = (diag[0] * prev[0]) / dk;
  acc[0] = acc[0] + next[0];
  for (int i = 1; i < dim; ++i) {
    const double a = diag[i] * prev[i];
    const double b = sub * prev[i - 1];
    const double t = (a + b) / dk;
    next[i] = t;
    acc[i] = acc[i] + t;
  }
}

}  // namespace

extern "C" int xmhd_phi_divided_diffs(int l, const double* nodes, int n, double subdiag,
                                      double* out) {
  if (l < 0 || n < 1 || !nodes || !out) return XMHD_BADARG;
  const int dim = l + n;
  std::vector<double> ext(dim, 0.0);
  for (int i = 0; i < n; ++i) ext[l + i] = nodes[i];
  const int terms = 60;
  // scale = max(np.max(np.abs(ext)), abs(subdiag), 1e-30)   (Python max order)
  double amax = std::fabs(ext[0]);
  for (int i = 1; i < dim; ++i) {
    const double a = std::fabs(ext[i]);
    if (a > amax || a != a) amax = a;
  }
  double scale = amax;
  if (std::fabs(subdiag) > scale) scale = std::fabs(subdiag);
  if (1e-30 > scale) scale = 1e-30;
  int s = 0;
  const int s1 = (int)std::ceil(std::log2(scale));
  const int s2 = (int)std::ceil(std::log2((double)(dim + terms) / (double)terms));
  if (s1 > s) s = s1;
  if (s2 > s) s = s2;
  const double p2 = std::ldexp(1.0, s);  // 2.0 ** s
  std::vector<double> diag(dim);
  for (int i = 0; i < dim; ++i) diag[i] = ext[i] / p2;
  const double sub = subdiag / p2;

  std::vector<double> col(dim, 0.0), t0(dim), t1(dim), acc(dim);
  col[0] = 1.0;
  const long long nsub = 1LL << s;
  for (long long it = 0; it < nsub; ++it) {
    std::memcpy(t0.data(), col.data(), sizeof(double) * dim);
    std::memcpy(acc.data(), col.data(), sizeof(double) * dim);
    double* prev = t0.data();
    double* next = t1.data();
    for (int k = 1; k < terms; ++k) {
      taylor_term(dim, diag.data(), sub, (double)k, prev, next, acc.data());
      double* sw = prev;
      prev = next;
      next = sw;
    }
    col.swap(acc);
  }
  for (int i = 0; i < n; ++i) out[i] = col[l + i];
  return XMHD_OK;
}

// _newton_coeffs without the cache (leja.py:94-96): the divided differences of
// phi_l(q + theta*xi) at the first `count` Leja points, divided by theta**l
// (Python float ** int is C pow).
extern "C" int xmhd_newton_coeffs(int l, double q, double theta, const double* xi, int count,
                                  double* out) {
  if (l < 0 || l > 4 || count < 1 || count > 500 || !xi || !out || !(theta > 0.0))
    return XMHD_BADARG;
  std::vector<double> nodes(count);
  for (int i = 0; i < count; ++i) nodes[i] = q + theta * xi[i];
  const int rc = xmhd_phi_divided_diffs(l, nodes.data(), count, theta, out);
  if (rc) return rc;
  const double s = std::pow(theta, (double)l);
  for (int i = 0; i < count; ++i) out[i] = out[i] / s;
  return XMHD_OK;
}

// The 500-entry table one apply_phi_leja call of an uncached (l, q, theta)
// indexes (leja.py:119-130): term m < 64 reads the 64-chunk, m < 128 the
// 128-chunk (recomputed, not extended), m < 256 the 256-chunk, else the
// 500-chunk.  xmhd_leja takes it as its coefficient table.
extern "C" int xmhd_leja_schedule(int l, double q, double theta, const double* xi, double* out) {
  if (!out) return XMHD_BADARG;
  std::vector<double> chunk(500);
  int lo = 0;
  for (int size : {64, 128, 256, 500}) {
    const int rc = xmhd_newton_coeffs(l, q, theta, xi, size, chunk.data());
    if (rc) return rc;
    for (int i = lo; i < size; ++i) out[i] = chunk[i];
    lo = size;
  }
  return XMHD_OK;
}
