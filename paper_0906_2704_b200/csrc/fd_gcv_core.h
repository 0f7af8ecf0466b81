// gcv_minimize's selection logic (reference src/regularize.cpp:144-214),
// written once as __host__ __device__ code: the sm_100a kernels run it per
// item on the GPU, and the C-ABI exports the same code on the host
// (fd_gcv_minimize_host) so the CPU test suite pins it against the reference.
#pragma once

#include <math.h>

#ifdef __CUDACC__
#define FD_HD __host__ __device__
#else
#define FD_HD
#endif

namespace fdb {

struct GcvPick {
  int best_k;
  int tied;
  double mu_tie;
  double lo, hi;
};

// First minimum (std::min_element), 1e-12 relative tie test with the
// geometric midpoint of the tied grid values (regularize.cpp:172-185), and the
// golden-section bracket [mu_{k-1}, mu_{k+1}] clamped at the ends (325-326).
FD_HD inline GcvPick gcv_pick(const double* mus, const double* logmus, const double* vals,
                              int count) {
  GcvPick p;
  int bk = 0;
  double best = vals[0];
  for (int k = 1; k < count; ++k)
    if (vals[k] < best) {
      best = vals[k];
      bk = k;
    }
  int ntied = 0;
  double mean_log = 0.0;
  for (int k = 0; k < count; ++k) {
    const bool tie = best == 0.0 ? vals[k] == 0.0 : vals[k] <= best + 1e-12 * fabs(best);
    if (tie) {
      ++ntied;
      mean_log += logmus[k];
    }
  }
  p.best_k = bk;
  p.tied = ntied > 1;
  p.mu_tie = p.tied ? exp(mean_log / (double)ntied) : 0.0;
  p.lo = mus[bk > 0 ? bk - 1 : 0];
  p.hi = mus[bk + 1 < count ? bk + 1 : count - 1];
  return p;
}

// Golden-section refinement in log(mu) (regularize.cpp:187-213), verbatim.
#ifdef __CUDACC__
#pragma nv_exec_check_disable
#endif
template <class GF>
FD_HD inline double gcv_golden(const double* mus, int count, int best_k, double best, GF& G) {
  const double lo = mus[best_k > 0 ? best_k - 1 : 0];
  const double hi = mus[best_k + 1 < count ? best_k + 1 : count - 1];
  double a = log(lo), b = log(hi);
  const double invphi = 0.6180339887498949;
  double x1 = b - invphi * (b - a);
  double x2 = a + invphi * (b - a);
  double f1 = G(exp(x1));
  double f2 = G(exp(x2));
  while (exp(b - a) - 1.0 > 1e-3) {
    if (f1 <= f2) {
      b = x2;
      x2 = x1;
      f2 = f1;
      x1 = b - invphi * (b - a);
      f1 = G(exp(x1));
    } else {
      a = x1;
      x1 = x2;
      f1 = f2;
      x2 = a + invphi * (b - a);
      f2 = G(exp(x2));
    }
  }
  const double refined = exp(0.5 * (a + b));
  return G(refined) <= best ? refined : mus[best_k];
}

// Number of Taylor moments J so that every golden-section point in
// [lo, hi] = [mu_{k-1}, mu_{k+1}] is evaluated to ~1e-17 relative:
// ratio = sqrt(hi/lo) - 1 = e^{Delta} - 1, Delta the grid's log spacing;
// need (J+1) ratio^J < 1e-17.  Returns 0 when the series would need > 48
// terms (very coarse grids), in which case the caller evaluates directly.
// the term counts the moment kernels are instantiated for (launch_moments):
// 4, 8, every J in 12..20, then 24..48 in steps of 4
FD_HD inline bool gcv_moment_count_supported(int J) {
  return J >= 4 && J <= 48 && ((J >= 12 && J <= 20) || J % 4 == 0);
}

FD_HD inline int gcv_moment_terms(double mu_min, double mu_max, int count) {
  const double delta = (log(mu_max) - log(mu_min)) / (double)(count - 1);
  const double ratio = exp(delta) - 1.0;
  if (!(ratio < 0.45)) return 0;
  // every J in 12..20 (the configs' grids land there: 13 at 512 points over
  // 1e-8..1, 17 at 256, 20 at 128 over 1e-6..1), multiples of 4 elsewhere --
  // the moment kernels are instantiated for exactly these counts
  for (int J = 4; J <= 48; J += (J >= 12 && J < 20) ? 1 : 4)
    if ((J + 1) * pow(ratio, (double)J) < 1e-17) return J;
  return 0;
}

}  // namespace fdb
