// TEST INFRASTRUCTURE ONLY (oracle/). Never linked into the product library.
//
// A flat extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src/*.cpp (see oracle/Makefile). It lets the
// Python tests, the golden-vector generator and bench.py's reference arm call
// the reference's own public API through ctypes:
//   build_operator / build_operator_2d     operators.cpp:293-301, multidim.cpp:309-322
//   SpectralBasis::analyze / synthesize    operators.cpp:181-201
//   tensor_apply                           multidim.cpp:172-198
//   blur_apply(_2d)                        operators.cpp:319-322, multidim.cpp:324-327
//   smoothing_eigenvalues(_2d)             regularize.cpp:19-47, multidim.cpp:329-356
//   tikhonov_solve(_2d), gcv_value(_2d)    regularize.cpp:73-142, multidim.cpp:358-415
//   gcv_minimize, gcv_select(_2d)          regularize.cpp:144-247, multidim.cpp:417-442
//   deblur(_2d)                            pipeline.cpp:147-165
//   sweep_mu                               pipeline.cpp:55-115
//   add_noise, convolve_valid(_2d)         operators.cpp:332-358, pipeline.cpp:15-51
// Status codes follow the CLI mapping (fastdeblur.cpp:442-451):
// 0 ok, 2 ValidationError, 3 DegenerateError, 1 anything else.
#include <atomic>
#include <cmath>
#include <complex>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fastdeblur/boundary.hpp"
#include "fastdeblur/errors.hpp"
#include "fastdeblur/multidim.hpp"
#include "fastdeblur/operators.hpp"
#include "fastdeblur/pipeline.hpp"
#include "fastdeblur/regularize.hpp"

namespace fd = fastdeblur;
using fd::cplx;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const fd::ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const fd::DegenerateError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

fd::BoundaryCondition bc_of(int bc) {
  switch (bc) {
    case 0: return fd::BoundaryCondition::periodic;
    case 1: return fd::BoundaryCondition::reflective;
    case 2: return fd::BoundaryCondition::antireflective;
    case 3: return fd::BoundaryCondition::hoc_cosine;
    case 4: return fd::BoundaryCondition::hoc_fourier;
  }
  throw fd::ValidationError("unknown bc code");
}

fd::Psf psf_of(const double* w, int len) {
  return fd::make_psf(std::vector<double>(w, w + len), /*normalize=*/true);
}

// smoother: 0 identity, 1 laplacian, 2 caller-supplied eigenvalues (custom)
fd::SmoothingOperator smoother_1d(int kind, const double* custom, const fd::BlurOperator& op) {
  if (kind == 2) {
    fd::SmoothingOperator L;
    L.kind = fd::SmootherKind::identity;
    const int n = fd::operator_order(op);
    L.eigenvalues.assign(custom, custom + n);
    return L;
  }
  return fd::smoothing_eigenvalues(kind == 0 ? fd::SmootherKind::identity
                                             : fd::SmootherKind::laplacian,
                                   op);
}

void split(const std::vector<cplx>& v, double* re, double* im) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    re[i] = v[i].real();
    if (im) im[i] = v[i].imag();
  }
}

// 2D operator: eig_mode 0 = the reference's own build_operator_2d
// (eigenvalues_2d three-step scheme); eig_mode 1 = aggregate initialisation
// with the outer product of the marginal 1D eigenvalues (equal to
// eigenvalues_2d for separable masks, test_multidim.cpp:106-123).
fd::BlurOperator2D op2d(const double* psf2, int rows, int cols, int n1, int n2, int bc,
                        int eig_mode) {
  const fd::Psf2D p = fd::make_psf2d(std::vector<double>(psf2, psf2 + rows * cols), rows,
                                     cols, /*normalize=*/true);
  const fd::BoundaryCondition b = bc_of(bc);
  if (eig_mode == 0) return fd::build_operator_2d(p, n1, n2, b);
  const fd::Psf a1 = fd::marginal_sum_columns(p);
  const fd::Psf a2 = fd::marginal_sum_rows(p);
  if (fd::is_complex_basis(b)) {
    const auto d1 = fd::operator_eigenvalues<cplx>(a1, n1, b);
    const auto d2 = fd::operator_eigenvalues<cplx>(a2, n2, b);
    std::vector<cplx> d(static_cast<std::size_t>(n1) * n2);
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n2; ++j) d[static_cast<std::size_t>(i) * n2 + j] = d1[i] * d2[j];
    return fd::ComplexBlurOperator2D{b, n1, n2, std::move(d), p,
                                     fd::SpectralBasis<cplx>(b, n1),
                                     fd::SpectralBasis<cplx>(b, n2)};
  }
  const auto d1 = fd::operator_eigenvalues<double>(a1, n1, b);
  const auto d2 = fd::operator_eigenvalues<double>(a2, n2, b);
  std::vector<double> d(static_cast<std::size_t>(n1) * n2);
  for (int i = 0; i < n1; ++i)
    for (int j = 0; j < n2; ++j) d[static_cast<std::size_t>(i) * n2 + j] = d1[i] * d2[j];
  return fd::RealBlurOperator2D{b, n1, n2, std::move(d), p, fd::SpectralBasis<double>(b, n1),
                                fd::SpectralBasis<double>(b, n2)};
}

fd::SmoothingOperator2D smoother_2d(int kind, const double* custom, const fd::BlurOperator2D& op,
                                    std::size_t total) {
  if (kind == 2) {
    fd::SmoothingOperator2D L;
    L.kind = fd::SmootherKind::identity;
    L.eigenvalues.assign(custom, custom + total);
    return L;
  }
  return fd::smoothing_eigenvalues_2d(
      kind == 0 ? fd::SmootherKind::identity : fd::SmootherKind::laplacian, op);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_eigenvalues_1d(const double* psf, int len, int n, int bc, double* re, double* im) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    std::visit(
        [&](const auto& o) {
          for (int i = 0; i < n; ++i) {
            const cplx d(o.eigenvalues[i]);
            re[i] = d.real();
            im[i] = d.imag();
          }
        },
        op);
  });
}

int ref_smoother_1d(const double* psf, int len, int n, int bc, int kind, double* s) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    const auto L = smoother_1d(kind, nullptr, op);
    std::copy(L.eigenvalues.begin(), L.eigenvalues.end(), s);
  });
}

// dir 0 = analyze (T^-1), 1 = synthesize (T). im arrays used for complex bases.
int ref_basis_apply_1d(int bc, int n, int dir, const double* in_re, const double* in_im,
                       double* out_re, double* out_im) {
  return guarded([&] {
    const fd::BoundaryCondition b = bc_of(bc);
    if (fd::is_complex_basis(b)) {
      fd::SpectralBasis<cplx> basis(b, n);
      std::vector<cplx> x(static_cast<std::size_t>(n));
      for (int i = 0; i < n; ++i) x[i] = cplx(in_re[i], in_im ? in_im[i] : 0.0);
      split(dir == 0 ? basis.analyze(x) : basis.synthesize(x), out_re, out_im);
    } else {
      fd::SpectralBasis<double> basis(b, n);
      std::vector<double> x(in_re, in_re + n);
      const auto y = dir == 0 ? basis.analyze(x) : basis.synthesize(x);
      std::copy(y.begin(), y.end(), out_re);
      if (out_im) std::fill(out_im, out_im + n, 0.0);
    }
  });
}

// Structured-transform internals (boundary.hpp:44-60) for bases 0 AR, 1 HC, 2 HF.
int ref_transform_fields(int basis, int n, double* q, double* alpha, double* v, double* w,
                         double* row_a, double* row_b, double* c_a, double* c_b, double* cap) {
  return guarded([&] {
    const fd::BoundaryBasis bb = basis == 0   ? fd::BoundaryBasis::antireflective
                                 : basis == 1 ? fd::BoundaryBasis::hoc_cosine
                                              : fd::BoundaryBasis::hoc_fourier;
    auto dump = [&](const auto& t) {
      std::copy(t.q.begin(), t.q.end(), q);
      *alpha = t.alpha;
      const int m = n - 2;
      for (int i = 0; i < m; ++i) {
        const cplx vi(t.v[i]), wi(t.w[i]), ra(t.row_a[i]), rb(t.row_b[i]), ca(t.c_a[i]),
            cb(t.c_b[i]);
        v[2 * i] = vi.real(), v[2 * i + 1] = vi.imag();
        w[2 * i] = wi.real(), w[2 * i + 1] = wi.imag();
        row_a[2 * i] = ra.real(), row_a[2 * i + 1] = ra.imag();
        row_b[2 * i] = rb.real(), row_b[2 * i + 1] = rb.imag();
        c_a[2 * i] = ca.real(), c_a[2 * i + 1] = ca.imag();
        c_b[2 * i] = cb.real(), c_b[2 * i + 1] = cb.imag();
      }
      for (int k = 0; k < 4; ++k) {
        const cplx c(t.capacitance[k]);
        cap[2 * k] = c.real(), cap[2 * k + 1] = c.imag();
      }
    };
    if (bb == fd::BoundaryBasis::hoc_fourier)
      dump(fd::build_fourier_transform(n));
    else
      dump(fd::build_real_transform(bb, n));
  });
}

int ref_matvec_1d(const double* psf, int len, int n, int bc, const double* f, double* out,
                  double* imag_residue) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    const auto y = fd::blur_apply(op, std::span<const double>(f, n), imag_residue);
    std::copy(y.begin(), y.end(), out);
  });
}

// sweep_mu (pipeline.cpp:55-115): curve (mu, G, rre) and summary
// {min_rre, mu_opt, mu_gcv, rre_gcv}; truth may be null (NaN rre fields).
int ref_sweep_mu_1d(const double* psf, int len, int n, int bc, int smoother,
                    const double* s_custom, const double* g, const double* truth, double mu_min,
                    double mu_max, int count, double* mus, double* G, double* rre,
                    double* summary) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    const auto L = smoother_1d(smoother, s_custom, op);
    fd::GcvSearch s;
    s.mu_min = mu_min;
    s.mu_max = mu_max;
    s.count = count;
    const fd::BcSweep sw =
        fd::sweep_mu(op, L, std::span<const double>(g, n),
                     truth ? std::span<const double>(truth, n) : std::span<const double>(), s);
    for (size_t k = 0; k < sw.curve.size(); ++k) {
      mus[k] = sw.curve[k].mu;
      G[k] = sw.curve[k].gcv;
      rre[k] = sw.curve[k].rre;
    }
    summary[0] = sw.min_rre;
    summary[1] = sw.mu_opt;
    summary[2] = sw.mu_gcv;
    summary[3] = sw.rre_gcv;
  });
}

int ref_gcv_value_1d(const double* psf, int len, int n, int bc, int smoother,
                     const double* s_custom, const double* g, double mu, double* G) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    const auto L = smoother_1d(smoother, s_custom, op);
    *G = fd::gcv_value(op, L, std::span<const double>(g, n), mu);
  });
}

// deblur (pipeline.cpp:147-155) for `batch` independent signals sharing one
// operator; `threads` > 1 runs an outer pool over signals (a harness
// addition; the reference itself has no batch entry point).
// curve_G (optional) receives batch*count grid values of G.
int ref_deblur_1d(const double* psf, int len, int n, int bc, int smoother,
                  const double* s_custom, int use_gcv, double fixed_mu, double mu_min,
                  double mu_max, int count, long batch, const double* g, double* out,
                  double* mu_used, double* curve_G, double* imag_residue, int threads) {
  return guarded([&] {
    const fd::BlurOperator op = fd::build_operator(psf_of(psf, len), n, bc_of(bc));
    const auto L = smoother_1d(smoother, s_custom, op);
    const fd::GcvSearch search{mu_min, mu_max, count};
    const fd::MuChoice choice{use_gcv != 0, fixed_mu};
    std::atomic<long> next{0};
    std::atomic<int> status{0};
    std::string first_err;
    auto work = [&] {
      for (;;) {
        const long b = next.fetch_add(1);
        if (b >= batch || status.load() != 0) return;
        const int st = guarded([&] {
          const auto rep = fd::deblur(op, L, std::span<const double>(g + b * n, n), choice,
                                      {}, curve_G != nullptr, search);
          std::copy(rep.restored.begin(), rep.restored.end(), out + b * n);
          if (mu_used) mu_used[b] = rep.mu_used;
          if (imag_residue) imag_residue[b] = rep.imag_residue;
          if (curve_G)
            for (int k = 0; k < count && k < static_cast<int>(rep.gcv_curve.size()); ++k)
              curve_G[b * count + k] = rep.gcv_curve[k].second;
        });
        if (st != 0) {
          int expected = 0;
          if (status.compare_exchange_strong(expected, st)) first_err = g_err;
        }
      }
    };
    if (threads <= 1) {
      work();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) pool.emplace_back(work);
      for (auto& t : pool) t.join();
    }
    if (status.load() == 2) throw fd::ValidationError(first_err);
    if (status.load() == 3) throw fd::DegenerateError(first_err);
    if (status.load() != 0) throw fd::Error(first_err);
  });
}

typedef double (*ref_gcv_fn)(double mu, void* ctx);

// gcv_minimize (regularize.cpp:144-214) driven by an arbitrary G callback;
// used to pin the product's host-side selection logic.
int ref_gcv_minimize(ref_gcv_fn G, void* ctx, double mu_min, double mu_max, int count,
                     double* mu, double* curve_G) {
  return guarded([&] {
    const auto r = fd::gcv_minimize([&](double x) { return G(x, ctx); },
                                    fd::GcvSearch{mu_min, mu_max, count});
    *mu = r.mu;
    if (curve_G)
      for (std::size_t k = 0; k < r.curve.size(); ++k) curve_G[k] = r.curve[k].second;
  });
}

int ref_add_noise(const double* g, long n, double level, unsigned long long seed, double* out) {
  return guarded([&] {
    const auto y = fd::add_noise(std::span<const double>(g, n), level, seed);
    std::copy(y.begin(), y.end(), out);
  });
}

int ref_convolve_valid(const double* ext, long len_ext, const double* psf, int len,
                       double* out) {
  return guarded([&] {
    const auto y = fd::convolve_valid(std::span<const double>(ext, len_ext), psf_of(psf, len));
    std::copy(y.begin(), y.end(), out);
  });
}

int ref_convolve_valid_2d(const double* ext, int rows, int cols, const double* psf2, int pr,
                          int pc, double* out) {
  return guarded([&] {
    const fd::Psf2D p = fd::make_psf2d(std::vector<double>(psf2, psf2 + pr * pc), pr, pc, true);
    const auto y = fd::convolve_valid_2d(
        std::span<const double>(ext, static_cast<std::size_t>(rows) * cols), rows, cols, p);
    std::copy(y.begin(), y.end(), out);
  });
}

int ref_eigenvalues_2d(const double* psf2, int rows, int cols, int n1, int n2, int bc,
                       int eig_mode, double* re, double* im) {
  return guarded([&] {
    const auto op = op2d(psf2, rows, cols, n1, n2, bc, eig_mode);
    std::visit(
        [&](const auto& o) {
          for (std::size_t i = 0; i < o.eigenvalues.size(); ++i) {
            const cplx d(o.eigenvalues[i]);
            re[i] = d.real();
            im[i] = d.imag();
          }
        },
        op);
  });
}

// tensor_apply (multidim.cpp:172-198): dir 0 = analyze, 1 = synthesize.
int ref_tensor_apply(int bc, int n1, int n2, int dir, const double* in_re, const double* in_im,
                     double* out_re, double* out_im) {
  return guarded([&] {
    const fd::BoundaryCondition b = bc_of(bc);
    const std::size_t total = static_cast<std::size_t>(n1) * n2;
    const fd::Direction d = dir == 0 ? fd::Direction::inverse : fd::Direction::forward;
    if (fd::is_complex_basis(b)) {
      fd::SpectralBasis<cplx> r(b, n1), c(b, n2);
      std::vector<cplx> x(total);
      for (std::size_t i = 0; i < total; ++i) x[i] = cplx(in_re[i], in_im ? in_im[i] : 0.0);
      split(fd::tensor_apply<cplx>(r, c, x, d), out_re, out_im);
    } else {
      fd::SpectralBasis<double> r(b, n1), c(b, n2);
      std::vector<double> x(in_re, in_re + total);
      const auto y = fd::tensor_apply<double>(r, c, x, d);
      std::copy(y.begin(), y.end(), out_re);
      if (out_im) std::fill(out_im, out_im + total, 0.0);
    }
  });
}

int ref_matvec_2d(const double* psf2, int rows, int cols, int n1, int n2, int bc, int eig_mode,
                  const double* f, double* out, double* imag_residue) {
  return guarded([&] {
    const auto op = op2d(psf2, rows, cols, n1, n2, bc, eig_mode);
    const std::size_t total = static_cast<std::size_t>(n1) * n2;
    const auto y = fd::blur_apply_2d(op, std::span<const double>(f, total), imag_residue);
    std::copy(y.begin(), y.end(), out);
  });
}

int ref_gcv_value_2d(const double* psf2, int rows, int cols, int n1, int n2, int bc,
                     int eig_mode, int smoother, const double* s_custom, const double* g,
                     double mu, double* G) {
  return guarded([&] {
    const auto op = op2d(psf2, rows, cols, n1, n2, bc, eig_mode);
    const std::size_t total = static_cast<std::size_t>(n1) * n2;
    const auto L = smoother_2d(smoother, s_custom, op, total);
    *G = fd::gcv_value_2d(op, L, std::span<const double>(g, total), mu);
  });
}

// deblur_2d (pipeline.cpp:157-165) for `batch` images sharing one operator.
int ref_deblur_2d(const double* psf2, int rows, int cols, int n1, int n2, int bc, int eig_mode,
                  int smoother, const double* s_custom, int use_gcv, double fixed_mu,
                  double mu_min, double mu_max, int count, long batch, const double* g,
                  double* out, double* mu_used, double* curve_G, double* imag_residue,
                  int threads) {
  return guarded([&] {
    const auto op = op2d(psf2, rows, cols, n1, n2, bc, eig_mode);
    const std::size_t total = static_cast<std::size_t>(n1) * n2;
    const auto L = smoother_2d(smoother, s_custom, op, total);
    const fd::GcvSearch search{mu_min, mu_max, count};
    const fd::MuChoice choice{use_gcv != 0, fixed_mu};
    std::atomic<long> next{0};
    std::atomic<int> status{0};
    std::string first_err;
    auto work = [&] {
      for (;;) {
        const long b = next.fetch_add(1);
        if (b >= batch || status.load() != 0) return;
        const int st = guarded([&] {
          const auto rep = fd::deblur_2d(op, L, std::span<const double>(g + b * total, total),
                                         choice, {}, curve_G != nullptr, search);
          std::copy(rep.restored.begin(), rep.restored.end(), out + b * total);
          if (mu_used) mu_used[b] = rep.mu_used;
          if (imag_residue) imag_residue[b] = rep.imag_residue;
          if (curve_G)
            for (int k = 0; k < count && k < static_cast<int>(rep.gcv_curve.size()); ++k)
              curve_G[b * count + k] = rep.gcv_curve[k].second;
        });
        if (st != 0) {
          int expected = 0;
          if (status.compare_exchange_strong(expected, st)) first_err = g_err;
        }
      }
    };
    if (threads <= 1) {
      work();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) pool.emplace_back(work);
      for (auto& t : pool) t.join();
    }
    if (status.load() == 2) throw fd::ValidationError(first_err);
    if (status.load() == 3) throw fd::DegenerateError(first_err);
    if (status.load() != 0) throw fd::Error(first_err);
  });
}

}  // extern "C"
