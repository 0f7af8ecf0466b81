// Internal structures shared by the sm_100a kernels (fd_kernels.cu) and the
// C-ABI / host orchestration (fd_capi.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fdb {

// BoundaryCondition codes (reference operators.hpp:15-21).
// Extension codes 5, 6: higher-order Fourier borders of degree d = 1 and 3
// (oracle/fdoracle.py HoTransform), not in the reference.
enum Bc : int { BC_PERIODIC = 0, BC_REFLECTIVE = 1, BC_ANTIREFLECTIVE = 2, BC_HOC_COSINE = 3,
                BC_HOC_FOURIER = 4, BC_HOC_FOURIER_D1 = 5, BC_HOC_FOURIER_D3 = 6 };

// border widths (k_left, k_right) of the higher-order codes
__host__ __device__ __forceinline__ int ho_kl(int bc) {
  return bc == BC_HOC_FOURIER_D1 ? 1 : bc == BC_HOC_FOURIER_D3 ? 2 : 0;
}
__host__ __device__ __forceinline__ int ho_kr(int bc) { return bc == BC_HOC_FOURIER_D3 ? 1 : 0; }
__host__ __device__ __forceinline__ bool is_ho_bc(int bc) {
  return bc == BC_HOC_FOURIER_D1 || bc == BC_HOC_FOURIER_D3;
}
constexpr int kHoMax = 3;  // largest border rank (d = 3)
// Interior trigonometric transform of an axis (boundary.cpp:35-43, operators.cpp:181-201).
enum Interior : int { IK_COS = 0, IK_FOURIER = 1, IK_SINE = 2 };
// Smoother kinds (regularize.hpp:15) + the first-difference extension.
enum Smoother : int { SM_IDENTITY = 0, SM_LAPLACIAN = 1, SM_FIRST_DIFFERENCE = 2, SM_CUSTOM = 3 };

// Tables for one length-L DFT evaluated by Bluestein's chirp-z convolution on
// a power-of-two FFT of size M >= 2L-1 held in shared memory.
struct FftTables {
  int L, M, logM;
  const double2* chirp;  // L entries  e^{-i pi j^2 / L}
  const double2* bhat;   // M entries  DIF_M(b)/M (in the DIF output order)
  const double2* tw;     // M/2 entries e^{-2 pi i j / M}
};

// One transform axis: T_X of order n (boundary.hpp:44-60) or a plain trig
// basis (periodic: F^H / F, reflective: C^T / C).  All vectors are complex
// (imag = 0 for the real bases) and live in device memory.
struct AxisDev {
  int n, m;        // order and interior length (m = n-2 when bordered)
  int kind;        // Interior
  int bordered;    // antireflective / hoc-cosine / hoc-fourier
  int correction;  // rank-2 SMW correction (false for antireflective)
  int cplx;        // complex basis (periodic, hoc-fourier)
  FftTables fft;          // full-length interior DFT (complex lines, line pairs)
  // Half-length real path: a real line of even length R (R = m, or 2(m+1) for
  // the DST-I odd extension) as a complex DFT of length R/2 (fd_kernels.cuh,
  // k_ranalyze / k_rsynth); rhalf = 0 when R is odd.
  int rhalf;
  FftTables hfft;         // DFT of length R/2
  const double2* rtw;     // R/2 entries e^{-2 pi i k/R}
  const double2* dct_tw;  // m entries e^{-i pi k/(2m)} (IK_COS)
  const double* q;        // n, boundary column (unit norm, q[n-1] = 0)
  double alpha;           // 1/q[0]
  const double2 *v, *w, *row_a, *row_b, *c_a, *c_b;  // m each
  const double *vr, *wr;  // real bases: Re v, Re w (m each; the real-line kernels' tables)
  double2 cav[4];         // ca_v, ca_w, cb_v, cb_w
  double2 cap[4];         // capacitance I + [c rows][v w], row-major
  // Real-line kernels (k_ranalyze / k_rsynth) never touch v, w, row_a/b,
  // c_a/b or q: for real data the correction is folded into the interior
  // transform (see k_ranalyze), using
  //   row_a = X^T c_a, row_b = X^T c_b  -- unit impulses at interior ia, ib
  //                                        (values ra1, rb1; checked at build),
  //   c_a . u = (X^H u)[top_i],  c_b . u = (X^H u)[bot_i],
  //   q_e = (q_gb - (e q_s + q_o))^2 q_inv   (qmode 1), (1 - e q_s) q_inv (qmode 0),
  // and the real parts of the 2x2 capacitance system (exactly real for real
  // data; the imaginary parts of the hoc-fourier tables are rounding noise).
  int ia, ib, top_i, bot_i, qmode;
  double ra1, rb1, q0;
  double q_gb, q_s, q_o, q_inv;
  // q over the interior as polynomials in the interior index s:
  //   q[s+1] = (qa1 - q_s s)^k q_inv,  q[n-2-s] = (qa2 + q_s s)^k q_inv,  k = 2 (qmode 1)
  //   or 1 (qmode 0), so a border combination a q[s+1] + b q[n-2-s] is one
  //   quadratic per line (border_poly).
  double qa1, qa2;
  // per-axis constants of the trig transforms (trig.cpp:116-180), host-computed
  double inv_sqrt_m, dct_s0, dct_s1, dst_scale;
  double cavr[4], capr[4];
  // inverse of the 2x2 capacitance (host, extended precision; see build_axis)
  double capi[4];
  // Interior coefficient e = i + kl (kl = 1 for the rank-2 borders).
  int kl;
  // Higher-order borders (hob = 1; bordered = correction = 0): k = kl + kr
  // polynomial columns P (P[l*n + i], unit norm) around the Fourier interior
  // of length m = n - k (oracle HoTransform).  Border row bord[l] is the
  // 2 pi-periodic image of interior sample wrap[l], so
  //   analyze     a = sinv (y[bord] - y[kl + wrap]),  b = F (y_I - P_I a)
  //   synthesize  y_I = F^H b + P_I a,  y[bord] = (F^H b)[wrap] + P[bord] a
  // with coefficient l of a stored at element l (l < kl) or m + l (l >= kl).
  int hob, kr, hk;
  // closed form of the border columns for the pair kernels (fd_pair.cuh):
  //   P[l][e] = L_{l+1}(t_e) ho_s[l],  t_e = ho_ta e + ho_tb  (Legendre)
  double ho_ta, ho_tb, ho_s[kHoMax];
  const double* P;
  // direct mixed-radix DFT of the interior (fd_mixed.cuh) when m is a product
  // of 3, 5, 7, 9, 11, 13 (mstages > 0): radices in stage order, the twiddle
  // table e^{-2 pi i t/m} (t < m) and the output permutation
  int mstages, mrad[6];
  const double2* mtw;
  const int* mperm;
  // Rader (fd_rader.cuh) when m is an odd prime and m - 1 factors into 2..31:
  // the mixed-radix plan above is for length m - 1; g^n table, output
  // positions, DFT(b)/(m-1) in the DIF output order
  int rader;
  const int* rgidx;
  const int* ropos;
  const double2* rbhat;
  // cosine lines whose half length h is a prime with smooth h - 1 (fd_cdirect.cuh):
  // Rader over N = h - 1 with the plan in mrad / mtw; sample j -> slot
  // cd_ilog[j], frequency k -> slot cd_opos[k] (h entries each), DFT(b)/N
  int cdir;
  const int* cd_ilog;
  const int* cd_opos;
  const double2* cd_bhat;
  double sinv[kHoMax * kHoMax];
  int bord[kHoMax], wrap[kHoMax];
};

// Geometry of a set of lines (rows or columns of a batch of arrays).
// Element e of line l lives at  (l / per_item) * item_stride
//                              + (l % per_item) * line_stride + e * elem_stride
// (strides in elements of the array's own type).
struct Lines {
  long long item_stride;
  long long line_stride;
  long long elem_stride;
  int per_item;
  int count;
};

__host__ __device__ __forceinline__ long long line_offset(const Lines& g, int l) {
  if (g.per_item == 1) return (long long)l * g.item_stride;
  return (long long)(l / g.per_item) * g.item_stride + (long long)(l % g.per_item) * g.line_stride;
}

// Per-coefficient spectral data for the filter / matvec scale / GCV.
//   mode 1: 1D vectors indexed by the element (d[e], s[e]);
//   mode 2: separable 2D  d = dA[i] * dB[j],  s = sA[i] + sB[j] (laplacian) or 1;
//   mode 3: full 2D arrays d[i*n2 + j], s[i*n2 + j].
// For 2D, (i, j) are recovered from (line, element) by the pass direction.
struct Spectral {
  int mode;
  int smooth_sum;        // separable: 1 = s_ij = sA[i] + sB[j]; 0 = identity (s = 1)
  int n2;                // row length of the 2D array
  int col_pass;          // 1: line = column j, element = row i; 0: line = row i, element = j
  const double2* dA;
  const double2* dB;
  const double* sA;
  const double* sB;
  // half-spectrum layout of a real image in a complex basis (see HalfRows):
  // stored row r is full row r (r < hr_split) or r + hr_off
  int hr_split, hr_off;
};

// Half-spectrum row layout of the 2D coefficients of a REAL image in a complex
// (Fourier-interior) basis.  After the column pass the coefficient rows are
// Hermitian in the row index: row kl + k = conj(row kl + m1 - k) for interior
// k (the border rows are real), and the row transform preserves the pairing
// (row kl + m1 - k of the result = conj of row kl + k with the columns
// reflected).  Only the rows 0 .. hs-1 (borders + interior k <= h1) and the
// kr right border rows are stored: H = hs + kr rows.
struct HalfRows {
  int n1, kl, kr, m1, h1, hs, H;
  __host__ __device__ int pos(int e) const {  // stored row of full row e, or -1
    if (e < hs) return e;
    if (e >= n1 - kr) return e - (n1 - kr) + hs;
    return -1;
  }
  __host__ __device__ int mirror(int e) const { return 2 * kl + m1 - e; }
};
__host__ __device__ inline HalfRows make_half_rows(int n1, int kl, int kr) {
  HalfRows h;
  h.n1 = n1;
  h.kl = kl;
  h.kr = kr;
  h.m1 = n1 - kl - kr;
  h.h1 = h.m1 / 2;
  h.hs = kl + h.h1 + 1;
  h.H = h.hs + kr;
  return h;
}

struct GcvGrid {
  int count;             // K
  const double* mus;     // K grid values (host std::exp, regularize.cpp:154-156)
  const double* logmus;  // log of each grid value (tie geometric mean)
};

}  // namespace fdb
