// sm_100a kernels of the transform + filter + GCV restoration path.
//
// Reference functions restated here (paths under /root/reference/proj/core):
//   transform_apply_inverse (analyze)       src/boundary.cpp:253-289
//   transform_apply (synthesize)            src/boundary.cpp:225-250
//   cosine_apply / fourier_apply / sine_apply  src/trig.cpp:116-180
//   SpectralBasis::analyze / synthesize     src/operators.cpp:181-201
//   tensor_apply (2D: column pass, row pass) src/multidim.cpp:172-198
//   apply_tikhonov_filter                   include/fastdeblur/regularize.hpp:42-58
//   gcv_from_coeffs                         include/fastdeblur/regularize.hpp:63-81
//   gcv_minimize                            src/regularize.cpp:144-214
//   operator_eigenvalues / eigenvalues_2d   src/operators.cpp:238-286, src/multidim.cpp:208-272
//   smoothing_eigenvalues(_2d)              src/regularize.cpp:19-38, src/multidim.cpp:329-356
//
// Every line transform is one CTA: the interior trigonometric transform runs
// in shared memory (fd_fft.cuh), two real lines share one complex FFT, and the
// rank-2 border (dot products, 2x2 capacitance solve, axpy) is fused into the
// load / store loops, so a line is read once and written once.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fd_fft.cuh"
#include "fd_gcv_core.h"
#include "fd_internal.h"

namespace fdb {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ldc(const void* base, bool cplx, long long idx) {
  if (cplx) return __ldg(reinterpret_cast<const double2*>(base) + idx);
  return make_double2(__ldg(reinterpret_cast<const double*>(base) + idx), 0.0);
}

__device__ __forceinline__ void stc(void* base, bool cplx, long long idx, double2 v) {
  if (cplx)
    reinterpret_cast<double2*>(base)[idx] = v;
  else
    reinterpret_cast<double*>(base)[idx] = v.x;
}

// element index of interior coefficient i
__device__ __forceinline__ int interior_elem(const AxisDev& ax, int i) { return i + ax.kl; }

// spectral values (d, s) of coefficient e of line l
__device__ __forceinline__ void spectral_at(const Spectral& sp, const Lines& g, int l, int e,
                                            double2& d, double& s) {
  if (sp.mode == 1) {
    d = __ldg(&sp.dA[e]);
    s = sp.sA ? __ldg(&sp.sA[e]) : 1.0;
    return;
  }
  const int li = l % g.per_item;
  const int i = sp.col_pass ? e : (li < sp.hr_split ? li : li + sp.hr_off);
  const int j = sp.col_pass ? li : e;
  if (sp.mode == 2) {
    d = cmul(__ldg(&sp.dA[i]), __ldg(&sp.dB[j]));
    s = sp.smooth_sum ? __ldg(&sp.sA[i]) + __ldg(&sp.sB[j]) : 1.0;
  } else {
    const long long idx = (long long)i * sp.n2 + j;
    d = __ldg(&sp.dA[idx]);
    s = sp.sA ? __ldg(&sp.sA[idx]) : 1.0;
  }
}

// ---------------------------------------------------------------------------
// setup kernels
// ---------------------------------------------------------------------------
// chirp c_j = e^{-i pi j^2/L}, twiddles e^{-2 pi i j/M}, Bluestein kernel b,
// DCT quarter-wave twiddles e^{-i pi k/(2m)} (trig.cpp:73-87).
__global__ void k_init_tables(int L, int M, double2* chirp, double2* tw, double2* b, int mdct,
                              double2* dct_tw) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < M; j += stride) {
    if (j < L) {
      const long long q = (j * j) % (2LL * L);
      double s, c;
      sincospi(-(double)q / (double)L, &s, &c);
      chirp[j] = make_double2(c, s);
    }
    if (j < M / 2) {
      double s, c;
      sincospi(-2.0 * (double)j / (double)M, &s, &c);
      tw[j] = make_double2(c, s);
    }
    // b_j = conj(c_|j|) on the circle of length M
    long long jj = -1;
    if (j < L)
      jj = j;
    else if (j > M - L)
      jj = M - j;
    if (jj >= 0) {
      const long long q = (jj * jj) % (2LL * L);
      double s, c;
      sincospi((double)q / (double)L, &s, &c);
      b[j] = make_double2(c, s);
    } else {
      b[j] = make_double2(0.0, 0.0);
    }
    if (j < mdct) {
      double s, c;
      sincospi(-(double)j / (2.0 * mdct), &s, &c);
      dct_tw[j] = make_double2(c, s);
    }
  }
}

// real-FFT twiddles e^{-2 pi i k/R}, k < R/2
__global__ void k_init_rtw(int R, double2* rtw) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < R / 2; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)R, &s, &c);
    rtw[k] = make_double2(c, s);
  }
}

// bhat = DIF_M(b)/M, left in DIF (digit-reversed) order.  part < 0: the whole
// transform in shared memory; part 0/1: half p of a split DIF for M beyond
// shared memory (first stage lower = b_lo + b_hi, upper = (b_lo - b_hi) W^t,
// then a local DIF of size M/2), writing bhat[p M/2, (p+1) M/2).
__global__ void __launch_bounds__(512) k_bhat(FftTables T, const double2* __restrict__ b,
                                              double2* bhat, int part) {
  extern __shared__ double2 sm[];
  const int Mloc = part < 0 ? T.M : T.M / 2;
  const int logMloc = part < 0 ? T.logM : T.logM - 1;
  const TwSm tw = load_twiddles(sm + pidx(Mloc) + 1, T);
  __syncthreads();
  for (int j = threadIdx.x; j < Mloc; j += blockDim.x) {
    double2 v;
    if (part < 0) {
      v = b[j];
    } else {
      const double2 lo = b[j], hi = b[j + Mloc];
      v = part == 0 ? cadd(lo, hi) : cmul(csub(lo, hi), tw(j));
    }
    sm[pidx(j)] = v;
  }
  __syncthreads();
  fft_dif_local(sm, Mloc, logMloc, T.M, tw);
  const double inv = 1.0 / (double)T.M;
  const int off = part < 0 ? 0 : part * Mloc;
  for (int j = threadIdx.x; j < Mloc; j += blockDim.x)
    bhat[off + bhat_store_index(j, logMloc)] = cscale(sm[pidx(j)], inv);
}

// bhat for M beyond shared memory: the same DIF in a global buffer x of
// pidx(M) + 1 slots (one CTA; setup only)
__global__ void __launch_bounds__(512) k_bhat_long(FftTables T, const double2* __restrict__ b,
                                                   double2* bhat, double2* x) {
  extern __shared__ double2 sm[];
  const TwSm tw = load_twiddles(sm, T);
  for (int j = threadIdx.x; j < T.M; j += blockDim.x) x[pidx(j)] = b[j];
  __syncthreads();
  fft_dif_local(x, T.M, T.logM, T.M, tw);
  const double inv = 1.0 / (double)T.M;
  for (int j = threadIdx.x; j < T.M; j += blockDim.x)
    bhat[bhat_store_index(j, T.logM)] = cscale(x[pidx(j)], inv);
}

// symbol z(t) = sum_j h_j e^{ijt} (psf.cpp:39-52)
__device__ double2 symbol_eval(const double* __restrict__ h, int m, int symmetric, double t) {
  if (symmetric) {
    double z = h[m];
    for (int j = 1; j <= m; ++j) z += 2.0 * h[m + j] * cos(j * t);
    return make_double2(z, 0.0);
  }
  double zr = h[m], zi = 0.0;
  for (int j = 1; j <= m; ++j) {
    double s, c;
    sincos(j * t, &s, &c);
    // h_j (c + i s) + h_{-j} (c - i s)
    zr += h[m + j] * c + h[m - j] * c;
    zi += h[m + j] * s - h[m - j] * s;
  }
  return make_double2(zr, zi);
}

// node_i of eigenvalue_grid (operators.cpp:130-161), operation order mirrored
__device__ __forceinline__ double eig_node(int bc, int n, int i) {
  const double kPi = 3.14159265358979323846;
  switch (bc) {
    case BC_PERIODIC: return 2.0 * kPi * i / n;
    case BC_REFLECTIVE: return kPi * i / n;
    case BC_ANTIREFLECTIVE: return i < n - 1 ? kPi * i / (n - 1) : 0.0;
    case BC_HOC_COSINE: return (i >= 1 && i < n - 1) ? kPi * (i - 1) / (n - 2) : 0.0;
    case BC_HOC_FOURIER_D1:
    case BC_HOC_FOURIER_D3: {  // extension: 2 pi j / m on the interior, 0 on the borders
      const int kl = ho_kl(bc), m = n - kl - ho_kr(bc);
      return (i >= kl && i < kl + m) ? 2.0 * kPi * (i - kl) / m : 0.0;
    }
    default: return (i >= 1 && i < n - 1) ? 2.0 * kPi * (i - 1) / (n - 2) : 0.0;
  }
}

// 1D eigenvalues d (operators.cpp:238-286): symbol at the interior nodes,
// boundary eigenvalues of corrected operators pinned to exactly 1.
__global__ void k_eigenvalues_1d(const double* __restrict__ h, int m, int symmetric, int bc,
                                 int n, double2* d) {
  const double kPi = 3.14159265358979323846;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double t;
    bool pinned = false;
    switch (bc) {
      case BC_PERIODIC: t = 2.0 * kPi * i / n; break;  // exp_grid_symbol(len=n)
      case BC_REFLECTIVE: t = i * kPi / n; break;       // cos_grid_symbol(denom=n)
      case BC_ANTIREFLECTIVE:
        pinned = (i == 0 || i == n - 1);
        t = i * kPi / (n - 1);
        break;
      case BC_HOC_COSINE:
        pinned = (i == 0 || i == n - 1);
        t = (i - 1) * kPi / (n - 2);
        break;
      case BC_HOC_FOURIER_D1:
      case BC_HOC_FOURIER_D3: {  // extension (oracle operator_eigenvalues)
        const int kl = ho_kl(bc), m = n - kl - ho_kr(bc);
        pinned = (i < kl || i >= kl + m);
        t = 2.0 * kPi * (i - kl) / m;
        break;
      }
      default:
        pinned = (i == 0 || i == n - 1);
        t = 2.0 * kPi * (i - 1) / (n - 2);
        break;
    }
    double2 z = pinned ? make_double2(1.0, 0.0) : symbol_eval(h, m, symmetric, t);
    if (bc != BC_PERIODIC && bc != BC_HOC_FOURIER && !is_ho_bc(bc))
      z.y = 0.0;  // real bases keep .real()
    d[i] = z;
  }
}

// smoother eigenvalues on the node grid (regularize.cpp:19-38)
__global__ void k_smoother_1d(int kind, int bc, int n, double* s) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (kind == SM_IDENTITY) {
      s[i] = 1.0;
    } else {
      const double v = 2.0 - 2.0 * cos(eig_node(bc, n, i));
      s[i] = kind == SM_FIRST_DIFFERENCE ? sqrt(v) : v;
    }
  }
}

// r_e = |d_e|^2 / s_e^2 (+inf where s = 0) for the GCV kernels; sigma = 1/(r+mu)
// equals s^2/(|d|^2 + mu s^2) of regularize.hpp:71 (to rounding).
__global__ void k_gcv_ratio(const double2* __restrict__ d, const double* __restrict__ s, int n,
                            double* r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 di = d[i];
    const double si = s[i];
    const double d2 = di.x * di.x + di.y * di.y;
    r[i] = si == 0.0 ? INFINITY : d2 / (si * si);
  }
}

// 2D interior eigenvalues d_ij = sum_{p,q} h_pq e^{i(p t1_i + q t2_j)} as
// E1 (H E2): first T[p][j] = sum_q h_pq e^{i q t2_j}, then d_ij.
__global__ void k_eig2d_stage1(const double* __restrict__ h, int m1, int m2, int bc, int n2,
                               double2* T) {
  const int cols = 2 * m2 + 1, rows = 2 * m1 + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)rows * n2;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(idx / n2), j = (int)(idx % n2);
    const double t2 = eig_node(bc, n2, j);
    double re = 0.0, im = 0.0;
    for (int q = -m2; q <= m2; ++q) {
      double s, c;
      sincos(q * t2, &s, &c);
      const double w = h[p * cols + (q + m2)];
      re += w * c;
      im += w * s;
    }
    T[idx] = make_double2(re, im);
  }
}

__global__ void k_eig2d_stage2(const double2* __restrict__ T, int m1, int bc, int n1, int n2,
                               int cplx, double2* d) {
  const int rows = 2 * m1 + 1;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n1 * n2;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n2), j = (int)(idx % n2);
    const double t1 = eig_node(bc, n1, i);
    double2 z = make_double2(0.0, 0.0);
    for (int p = 0; p < rows; ++p) {
      double s, c;
      sincos((p - m1) * t1, &s, &c);
      z = cadd(z, cmul(make_double2(c, s), T[(long long)p * n2 + j]));
    }
    if (!cplx) z.y = 0.0;
    d[idx] = z;
  }
}

// edges from the marginal 1D eigenvalues, corners 1 (multidim.cpp:248-271)
__global__ void k_eig2d_edges(const double2* __restrict__ d1, const double2* __restrict__ d2,
                              int n1, int n2, double2* d) {
  const int tot = 2 * n1 + 2 * n2;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
    if (t < n1) {
      d[(long long)t * n2] = d1[t];
    } else if (t < 2 * n1) {
      const int i = t - n1;
      d[(long long)i * n2 + n2 - 1] = d1[i];
    } else if (t < 2 * n1 + n2) {
      const int j = t - 2 * n1;
      d[j] = d2[j];
    } else {
      const int j = t - 2 * n1 - n2;
      d[(long long)(n1 - 1) * n2 + j] = d2[j];
    }
  }
}

__global__ void k_eig2d_corners(int n1, int n2, double2* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double2 one = make_double2(1.0, 0.0);
    d[0] = one;
    d[n2 - 1] = one;
    d[(long long)(n1 - 1) * n2] = one;
    d[(long long)(n1 - 1) * n2 + n2 - 1] = one;
  }
}

// higher-order borders (extension): the same scheme with kl + kr border lines
// per axis -- border columns from d1, border rows from d2, crossings 1
__global__ void k_eig2d_ho_border(const double2* __restrict__ d1, const double2* __restrict__ d2,
                                  int n1, int n2, int kl, int kr, double2* d) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n1 * n2;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n2), j = (int)(idx % n2);
    const bool bi = i < kl || i >= n1 - kr, bj = j < kl || j >= n2 - kr;
    if (bi && bj)
      d[idx] = make_double2(1.0, 0.0);
    else if (bj)
      d[idx] = d1[i];
    else if (bi)
      d[idx] = d2[j];
  }
}

__global__ void k_smoother_2d(int kind, const double* __restrict__ s1,
                              const double* __restrict__ s2, int n1, int n2, double* s) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n1 * n2;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / n2), j = (int)(idx % n2);
    s[idx] = kind == SM_IDENTITY ? 1.0 : s1[i] + s2[j];
  }
}

// ---------------------------------------------------------------------------
// analyze: out = T_X^{-1} in along each line (transform_apply_inverse,
// boundary.cpp:253-289; plain C / F for reflective / periodic).
// Real input lines are packed in pairs into one complex FFT.
// ---------------------------------------------------------------------------
// ---- higher-order borders (extension; AxisDev::hob) ----
// a = sinv (y[bord] - y[kl + wrap]) of one line: k <= 3 samples, solved by
// every thread (no block synchronisation)
template <class LD>
__device__ __forceinline__ void ho_amplitudes(const AxisDev& ax, LD ld, double2 (&a)[kHoMax]) {
  double2 r[kHoMax];
#pragma unroll
  for (int l = 0; l < kHoMax; ++l)
    r[l] = l < ax.hk ? csub(ld(ax.bord[l]), ld(ax.kl + ax.wrap[l])) : czero();
#pragma unroll
  for (int l = 0; l < kHoMax; ++l) {
    double2 v = czero();
#pragma unroll
    for (int q = 0; q < kHoMax; ++q) {
      const double sv = ax.sinv[l * kHoMax + q];
      v.x += sv * r[q].x;
      v.y += sv * r[q].y;
    }
    a[l] = v;
  }
}

// (P a)_e: the border columns' contribution at element e
__device__ __forceinline__ double2 ho_poly(const AxisDev& ax, const double2 (&a)[kHoMax], int e) {
  double2 v = czero();
#pragma unroll
  for (int l = 0; l < kHoMax; ++l)
    if (l < ax.hk) {
      const double p = __ldg(&ax.P[(long long)l * ax.n + e]);
      v.x += a[l].x * p;
      v.y += a[l].y * p;
    }
  return v;
}

// element of border coefficient l: [a_0 .. a_{kl-1}, interior, a_kl .. a_{k-1}]
__device__ __forceinline__ int ho_coef_elem(const AxisDev& ax, int l) {
  return l < ax.kl ? l : ax.m + l;
}

struct LineIO {
  const void* in;
  void* out;
  Lines gi, go;
  int in_cplx, out_cplx;
  // optional GCV weights of 1D analyze (k_ranalyze): w[l * wstride + i] = |ghat|^2,
  // Hermitian pairs pre-summed for complex bases (reduced index order of
  // build_pairs in fd_capi.cu)
  double* wout;
  long long wstride;
  long long wn;  // weights actually written; [wn, wstride) is zero-filled
  int pack;      // Fourier lines of real data stored Hermitian-packed (k_ranalyze)
  int chirp_smem;  // real-line kernels: copy the Bluestein chirp to shared memory
  float* wout32;    // optional TF32 split of wout in screen tiles (fd_tc.cuh): hi
  float* wout32lo;  // and lo parts
  // fp32 storage variant (BASELINE config 3): the analyze input / synthesis
  // output are float (float2 when complex); arithmetic stays fp64.  Only the
  // generic kernels k_analyze / k_synth take these (launch_* route them).
  int in_f32, out_f32;
  // half-spectrum rows (HalfRows): the column analysis writes only the stored
  // rows; the column synthesis reads them and mirrors the rest (conj)
  int half;
  HalfRows hr;
  // long lines (full-length transform beyond shared memory): the generic
  // kernels k_analyze<0> / k_synth<0> run their Bluestein passes in a global
  // (L2-resident) buffer of pidx(M) + 1 slots per CTA; blk0 offsets the line
  // index so a bounded scratch serves any line count (launch_long)
  double2* xscr;
  int blk0;
};


__device__ __forceinline__ double2 ld_in(const LineIO& io, long long idx) {
  if (io.in_f32) {
    if (io.in_cplx) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(io.in) + idx);
      return make_double2(v.x, v.y);
    }
    return make_double2((double)__ldg(reinterpret_cast<const float*>(io.in) + idx), 0.0);
  }
  return ldc(io.in, io.in_cplx, idx);
}
// coefficient store of the analysis (element e of the line at `base`); in the
// half-spectrum layout element e goes to its stored row, or is dropped
__device__ __forceinline__ void st_coef(const LineIO& io, long long base, int e, double2 v) {
  if (io.half) {
    e = io.hr.pos(e);
    if (e < 0) return;
  }
  stc(io.out, io.out_cplx, base + (long long)e * io.go.elem_stride, v);
}

__device__ __forceinline__ void st_out(const LineIO& io, long long idx, double2 v) {
  if (io.out_f32) {
    if (io.out_cplx)
      reinterpret_cast<float2*>(io.out)[idx] = make_float2((float)v.x, (float)v.y);
    else
      reinterpret_cast<float*>(io.out)[idx] = (float)v.x;
    return;
  }
  stc(io.out, io.out_cplx, idx, v);
}

// LOGM > 0: size-specialised Bluestein core (bluestein_t; blockDim = line_threads(M))
// resident threads per SM the generic line kernels are compiled for (register cap 65536 / kLineOcc);
// 768 (80 registers, 1.5 KB of spills) measured 15 % slower on config 3 (r02)
#ifndef FD_LINE_OCC
#define FD_LINE_OCC 512
#endif
constexpr int kLineOcc = FD_LINE_OCC;
template <int LOGM>
constexpr int kLineNT = (1 << LOGM) / 16 < 64 ? 64 : ((1 << LOGM) / 16 > 512 ? 512 : (1 << LOGM) / 16);
template <int LOGM>
__global__ void __launch_bounds__(LOGM > 0 ? kLineNT<LOGM> : 512, LOGM > 0 ? kLineOcc / kLineNT<LOGM> : 1) k_analyze(AxisDev ax, LineIO io) {
  extern __shared__ double2 sm[];
  const int M = ax.fft.M;
  const bool xg = LOGM == 0 && io.xscr != nullptr;
  double2* x = xg ? io.xscr + (long long)blockIdx.x * (pidx(M) + 1) : sm;
  double2* aux = xg ? sm : sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(aux, ax.fft);
  double* red = reinterpret_cast<double*>(aux + tw_slots(ax.fft.logM));
  double2* bc = reinterpret_cast<double2*>(red + 32 * 8);

  const bool pair = !io.in_cplx;
  const int blk = blockIdx.x + io.blk0;
  const int l0 = pair ? 2 * blk : blk;
  if (l0 >= io.gi.count) return;
  const bool has1 = pair && (l0 + 1 < io.gi.count);
  const long long oi0 = line_offset(io.gi, l0);
  const long long oi1 = has1 ? line_offset(io.gi, l0 + 1) : oi0;
  const long long es = io.gi.elem_stride;
  const int n = ax.n, m = ax.m, L = ax.fft.L;
  const double2* chirp = ax.fft.chirp;

  auto ld0 = [&](int e) { return ld_in(io, oi0 + e * es); };
  auto ld1 = [&](int e) { return has1 ? ld_in(io, oi1 + e * es) : czero(); };

  double2 y00 = czero(), yn0 = czero(), y01 = czero(), yn1 = czero();
  if (ax.bordered) {
    y00 = ld0(0);
    yn0 = ld0(n - 1);
    y01 = ld1(0);
    yn1 = ld1(n - 1);
  }
  double2 ha0[kHoMax], ha1[kHoMax];
  if (ax.hob) {
    ho_amplitudes(ax, ld0, ha0);
    ho_amplitudes(ax, ld1, ha1);
  }

  // ---- load (with chirp premultiply) + border dot products ----
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // ra0, rb0, ra1, rb1 (re, im)
  const bool dots = ax.bordered && ax.correction;
  if (ax.kind == IK_COS) {
    const int half = (m + 1) / 2;
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double2 val = czero();
      if (j < m) {
        const int src = j < half ? 2 * j : 2 * (m - 1 - j) + 1;  // trig.cpp:139-141
        const int e = interior_elem(ax, src);
        const double a = ld0(e).x, b = ld1(e).x;
        val = cmul(make_double2(a, b), __ldg(&chirp[j]));
        if (dots) {
          const double ra = __ldg(&ax.row_a[src]).x, rb = __ldg(&ax.row_b[src]).x;
          acc[0] += ra * a;
          acc[2] += rb * a;
          acc[4] += ra * b;
          acc[6] += rb * b;
        }
      }
      x[pidx(j)] = val;
    }
  } else if (ax.kind == IK_FOURIER) {
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double2 val = czero();
      if (j < m) {
        const int e = interior_elem(ax, j);
        if (pair) {
          double a = ld0(e).x, b = ld1(e).x;
          if (ax.hob) {  // fold the border: F (y_I - P_I a)
            a -= ho_poly(ax, ha0, e).x;
            b -= ho_poly(ax, ha1, e).x;
          }
          val = cmul(make_double2(a, b), __ldg(&chirp[j]));
          if (dots) {
            const double2 ra = __ldg(&ax.row_a[j]), rb = __ldg(&ax.row_b[j]);
            acc[0] += ra.x * a, acc[1] += ra.y * a;
            acc[2] += rb.x * a, acc[3] += rb.y * a;
            acc[4] += ra.x * b, acc[5] += ra.y * b;
            acc[6] += rb.x * b, acc[7] += rb.y * b;
          }
        } else {
          double2 z = ld0(e);
          if (ax.hob) z = csub(z, ho_poly(ax, ha0, e));
          val = cmul(z, __ldg(&chirp[j]));
          if (dots) {
            const double2 ra = cmul(__ldg(&ax.row_a[j]), z), rb = cmul(__ldg(&ax.row_b[j]), z);
            acc[0] += ra.x, acc[1] += ra.y;
            acc[2] += rb.x, acc[3] += rb.y;
          }
        }
      }
      x[pidx(j)] = val;
    }
  } else {  // IK_SINE: odd extension (0, u, 0, -rev u) of length 2(m+1) (trig.cpp:165-174)
    for (int p = threadIdx.x; p < M; p += blockDim.x) {
      double2 val = czero();
      if (p < L && p != 0 && p != m + 1) {
        double a, b;
        if (p <= m) {
          const int e = interior_elem(ax, p - 1);
          a = ld0(e).x, b = ld1(e).x;
        } else {
          const int e = interior_elem(ax, L - 1 - p);
          a = -ld0(e).x, b = -ld1(e).x;
        }
        val = cmul(make_double2(a, b), __ldg(&chirp[p]));
      }
      x[pidx(p)] = val;
    }
  }
  if (dots) block_sum<8>(acc, red);

  // ---- SMW capacitance solve (boundary.cpp:278-286) ----
  if (threadIdx.x == 0) {
    double2 beta[4] = {czero(), czero(), czero(), czero()};
    if (dots) {
      const double* ci = ax.capi;  // real capacitance^-1 (exactly real: see build_axis)
      for (int t = 0; t < (pair ? 2 : 1); ++t) {
        const double2 y0 = t == 0 ? y00 : y01, yn = t == 0 ? yn0 : yn1;
        double2 ra = cadd(cmul(ax.cav[0], y0), cmul(ax.cav[1], yn));
        double2 rb = cadd(cmul(ax.cav[2], y0), cmul(ax.cav[3], yn));
        ra = cadd(ra, make_double2(acc[4 * t + 0], acc[4 * t + 1]));
        rb = cadd(rb, make_double2(acc[4 * t + 2], acc[4 * t + 3]));
        beta[2 * t] = cadd(cscale(ra, ci[0]), cscale(rb, ci[1]));
        beta[2 * t + 1] = cadd(cscale(ra, ci[2]), cscale(rb, ci[3]));
        if (!ax.cplx) {
          beta[2 * t].y = 0.0;
          beta[2 * t + 1].y = 0.0;
        }
      }
    }
    for (int k = 0; k < 4; ++k) bc[k] = beta[k];
  }
  __syncthreads();

  if constexpr (LOGM > 0)
    bluestein_t<LOGM, kLineNT<LOGM>>(x, ax.fft, tw, ax.fft.M);
  else
    bluestein_core(x, ax.fft, tw, ax.fft.M);

  const double2 b00 = bc[0], b10 = bc[1], b01 = bc[2], b11 = bc[3];
  const long long oo0 = line_offset(io.go, l0);
  const long long oo1 = has1 ? line_offset(io.go, l0 + 1) : oo0;

  // ---- post-process, border update, store ----
  const double inv_sqrt_m = 1.0 / sqrt((double)m);
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    double2 xi0, xi1 = czero();
    if (ax.kind == IK_SINE) {
      const double sc = -0.5 * sqrt(2.0 / ((double)m + 1.0));
      const double2 Z = cmul(x[pidx(k + 1)], __ldg(&chirp[k + 1]));
      xi0 = make_double2(sc * Z.y, 0.0);
      xi1 = make_double2(-sc * Z.x, 0.0);
    } else {
      const double2 Zk = cmul(x[pidx(k)], __ldg(&chirp[k]));
      if (pair) {
        const int kc = k == 0 ? 0 : m - k;
        const double2 Zc = cconj(cmul(x[pidx(kc)], __ldg(&chirp[kc])));
        const double2 U0 = cscale(cadd(Zk, Zc), 0.5);
        const double2 D = csub(Zk, Zc);
        const double2 U1 = make_double2(0.5 * D.y, -0.5 * D.x);
        if (ax.kind == IK_COS) {
          const double2 t = __ldg(&ax.dct_tw[k]);
          const double sk = k == 0 ? sqrt(1.0 / (double)m) : sqrt(2.0 / (double)m);
          xi0 = make_double2(sk * (t.x * U0.x - t.y * U0.y), 0.0);
          xi1 = make_double2(sk * (t.x * U1.x - t.y * U1.y), 0.0);
        } else {
          xi0 = cscale(U0, inv_sqrt_m);
          xi1 = cscale(U1, inv_sqrt_m);
        }
      } else {
        xi0 = cscale(Zk, inv_sqrt_m);
      }
    }
    const int e = interior_elem(ax, k);
    if (ax.bordered) {
      const double2 v = __ldg(&ax.v[k]), w = __ldg(&ax.w[k]);
      if (ax.cplx) {
        double2 o = cadd(cadd(cmul(y00, v), xi0), cmul(yn0, w));
        if (dots) o = csub(o, cadd(cmul(b00, v), cmul(b10, w)));
        st_coef(io, oo0, e, o);
        if (has1) {
          double2 o1 = cadd(cadd(cmul(y01, v), xi1), cmul(yn1, w));
          if (dots) o1 = csub(o1, cadd(cmul(b01, v), cmul(b11, w)));
          st_coef(io, oo1, e, o1);
        }
      } else {
        double o = y00.x * v.x + xi0.x + yn0.x * w.x;
        if (dots) o -= b00.x * v.x + b10.x * w.x;
        st_coef(io, oo0, e, make_double2(o, 0.0));
        if (has1) {
          double o1 = y01.x * v.x + xi1.x + yn1.x * w.x;
          if (dots) o1 -= b01.x * v.x + b11.x * w.x;
          st_coef(io, oo1, e, make_double2(o1, 0.0));
        }
      }
    } else {
      st_coef(io, oo0, e, xi0);
      if (has1) st_coef(io, oo1, e, xi1);
    }
  }
  if (ax.hob && threadIdx.x == 0) {
    for (int l = 0; l < ax.hk; ++l) {
      const int le = ho_coef_elem(ax, l);
      st_coef(io, oo0, le, pair ? make_double2(ha0[l].x, 0.0) : ha0[l]);
      if (has1) st_coef(io, oo1, le, make_double2(ha1[l].x, 0.0));
    }
  }
  if (ax.bordered && threadIdx.x == 0) {
    const double al = ax.alpha;
    for (int t = 0; t < (has1 ? 2 : 1); ++t) {
      const double2 y0 = t == 0 ? y00 : y01, yn = t == 0 ? yn0 : yn1;
      const double2 b0 = t == 0 ? b00 : b01, b1 = t == 0 ? b10 : b11;
      double2 o0 = cscale(y0, al), on = cscale(yn, al);
      if (dots) {
        o0 = csub(o0, cscale(b0, al));
        on = csub(on, cscale(b1, al));
      }
      const long long oo = t == 0 ? oo0 : oo1;
      st_coef(io, oo, 0, o0);
      st_coef(io, oo, n - 1, on);
    }
  }
}

// ---------------------------------------------------------------------------
// synthesize: out = T_X c (transform_apply, boundary.cpp:225-250), optionally
// with the Tikhonov filter (mode 1, regularize.hpp:42-58) or the eigenvalue
// scale of the matvec (mode 2, operators.cpp:207-232) fused into the load.
// Real bases: pairs of real lines.  Complex bases: one complex line per CTA;
// real outputs keep Re and report sum(Im^2) per line (operators.cpp:222-229).
// ---------------------------------------------------------------------------
struct SynthArgs {
  int mode;              // 0 plain, 1 filter, 2 scale by d
  Spectral sp;
  const double* mu_item; // per item (filter)
  double* resid2;        // per line sum Im^2 (complex basis, real output), or null
};

// coefficient c of element e of line l after the synthesis mode's scaling
// (apply_tikhonov_filter, regularize.hpp:42-58, for mode 1)
// (mu: the line's regularisation parameter, read once per line by the caller)
__device__ __forceinline__ double2 coeff_filter(const AxisDev& ax, const SynthArgs& sa,
                                                const Lines& g, int l, int e, double2 c,
                                                double mu) {
  if (sa.mode == 0) return c;
  double2 d;
  double s;
  spectral_at(sa.sp, g, l, e, d, s);
  if (sa.mode == 2) return ax.cplx ? cmul(c, d) : make_double2(c.x * d.x, 0.0);
  if (ax.cplx) {
    const double den = (d.x * d.x + d.y * d.y) + mu * s * s;
    return cmul(c, make_double2(d.x / den, -d.y / den));
  }
  const double f = d.x / (d.x * d.x + mu * s * s);
  return make_double2(c.x * f, 0.0);
}

// 1/x for positive normal x: MUFU reciprocal seed + two Newton steps (<= 1 ulp)
__device__ __forceinline__ double rcp_pos(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// coeff_filter of the real-line synthesis: the two quotients conj(d)/den share
// one reciprocal (within 1 ulp of the reference's two divisions)
__device__ __forceinline__ double2 coeff_filter_fast(const AxisDev& ax, const SynthArgs& sa,
                                                     const Lines& g, int l, int e, double2 c,
                                                     double mu) {
  if (sa.mode != 1) return coeff_filter(ax, sa, g, l, e, c, mu);
  double2 d;
  double s;
  spectral_at(sa.sp, g, l, e, d, s);
  if (ax.cplx) {
    const double r = rcp_pos((d.x * d.x + d.y * d.y) + mu * s * s);
    return cmul(c, make_double2(d.x * r, -d.y * r));
  }
  return make_double2(c.x * (d.x * rcp_pos(d.x * d.x + mu * s * s)), 0.0);
}

__device__ __forceinline__ double line_mu(const SynthArgs& sa, const Lines& g, int l) {
  return sa.mode == 1 ? __ldg(&sa.mu_item[l / g.per_item]) : 0.0;
}

__device__ __forceinline__ double2 coeff_at(const AxisDev& ax, const LineIO& io,
                                            const SynthArgs& sa, int l, long long off, int e) {
  double2 c;
  if (io.half) {  // stored row, or the conjugate of the mirrored stored row
    const int p = io.hr.pos(e);
    c = p >= 0 ? ldc(io.in, io.in_cplx, off + (long long)p * io.gi.elem_stride)
               : cconj(ldc(io.in, io.in_cplx,
                           off + (long long)io.hr.pos(io.hr.mirror(e)) * io.gi.elem_stride));
  } else {
    c = ldc(io.in, io.in_cplx, off + e * io.gi.elem_stride);
  }
  // one reciprocal instead of the filter's two divisions (<= 1 ulp, as the real-line kernels)
  return coeff_filter_fast(ax, sa, io.gi, l, e, c, line_mu(sa, io.gi, l));
}

template <int LOGM>
__global__ void __launch_bounds__(LOGM > 0 ? kLineNT<LOGM> : 512, LOGM > 0 ? kLineOcc / kLineNT<LOGM> : 1) k_synth(AxisDev ax, LineIO io,
                                                                        SynthArgs sa) {
  extern __shared__ double2 sm[];
  const int M = ax.fft.M;
  const bool xg = LOGM == 0 && io.xscr != nullptr;
  double2* x = xg ? io.xscr + (long long)blockIdx.x * (pidx(M) + 1) : sm;
  double2* aux = xg ? sm : sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(aux, ax.fft);
  double* red = reinterpret_cast<double*>(aux + tw_slots(ax.fft.logM));

  // Real bases: real coefficients, two lines per FFT.  Complex bases with a
  // real output and no residue request: the real part of T_X c only depends
  // on the Hermitian part of the interior coefficients (F^H of the
  // anti-Hermitian part is purely imaginary), so two lines share one FFT as
  // z = herm(c0) + i herm(c1).
  const bool hpack = ax.cplx && !io.out_cplx && sa.resid2 == nullptr;
  const bool pair = !ax.cplx || hpack;
  const int blk = blockIdx.x + io.blk0;
  const int l0 = pair ? 2 * blk : blk;
  if (l0 >= io.gi.count) return;
  const bool has1 = pair && (l0 + 1 < io.gi.count);
  const long long oi0 = line_offset(io.gi, l0);
  const long long oi1 = has1 ? line_offset(io.gi, l0 + 1) : oi0;
  const int n = ax.n, m = ax.m, L = ax.fft.L;
  const double2* chirp = ax.fft.chirp;

  auto c0 = [&](int e) { return coeff_at(ax, io, sa, l0, oi0, e); };
  auto c1 = [&](int e) { return has1 ? coeff_at(ax, io, sa, l0 + 1, oi1, e) : czero(); };

  double2 u00 = czero(), un0 = czero(), u01 = czero(), un1 = czero();
  if (ax.bordered) {
    u00 = c0(0);
    un0 = c0(n - 1);
    u01 = c1(0);
    un1 = c1(n - 1);
  }
  double2 ua0[kHoMax], ua1[kHoMax];  // border amplitudes a (filtered)
  if (ax.hob) {
#pragma unroll
    for (int l = 0; l < kHoMax; ++l) {
      ua0[l] = l < ax.hk ? c0(ho_coef_elem(ax, l)) : czero();
      ua1[l] = l < ax.hk ? c1(ho_coef_elem(ax, l)) : czero();
    }
  }
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // top0, bottom0, top1, bottom1 (re, im)
  const bool dots = ax.bordered && ax.correction;

  if (ax.kind == IK_COS) {
    // C^T u (trig.cpp:147-158): buf_k = s_k u_k tw_k, Re FFT(buf) reordered.
    // Two lines: Re FFT(buf) = FFT(herm(buf)), herm(b)_k = (b_k + conj b_{-k})/2.
    const double s0 = sqrt(1.0 / (double)m), s = sqrt(2.0 / (double)m);
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double2 val = czero();
      if (j < m) {
        const int jc = j == 0 ? 0 : m - j;
        const int e = interior_elem(ax, j), ec = interior_elem(ax, jc);
        const double2 tj = __ldg(&ax.dct_tw[j]), tc = __ldg(&ax.dct_tw[jc]);
        const double sj = j == 0 ? s0 : s, sc = jc == 0 ? s0 : s;
        const double a = c0(e).x, ac = c0(ec).x;
        const double b = c1(e).x, bcv = c1(ec).x;
        const double ta = sj * a, tac = sc * ac, tb = sj * b, tbc = sc * bcv;
        const double2 h0 = make_double2(0.5 * (ta * tj.x + tac * tc.x), 0.5 * (ta * tj.y - tac * tc.y));
        const double2 h1 = make_double2(0.5 * (tb * tj.x + tbc * tc.x), 0.5 * (tb * tj.y - tbc * tc.y));
        val = cmul(make_double2(h0.x - h1.y, h0.y + h1.x), __ldg(&chirp[j]));
        if (dots) {
          const double ca = __ldg(&ax.c_a[j]).x, cb = __ldg(&ax.c_b[j]).x;
          acc[0] += ca * a;
          acc[2] += cb * a;
          acc[4] += ca * b;
          acc[6] += cb * b;
        }
      }
      x[pidx(j)] = val;
    }
  } else if (ax.kind == IK_SINE) {  // Q is an involution (boundary.cpp:35-43)
    for (int p = threadIdx.x; p < M; p += blockDim.x) {
      double2 val = czero();
      if (p < L && p != 0 && p != m + 1) {
        double a, b;
        if (p <= m) {
          const int e = interior_elem(ax, p - 1);
          a = c0(e).x, b = c1(e).x;
        } else {
          const int e = interior_elem(ax, L - 1 - p);
          a = -c0(e).x, b = -c1(e).x;
        }
        val = cmul(make_double2(a, b), __ldg(&chirp[p]));
      }
      x[pidx(p)] = val;
    }
  } else if (hpack) {  // IK_FOURIER, two Hermitian-projected lines per FFT
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double2 val = czero();
      if (j < m) {
        const int jc = j == 0 ? 0 : m - j;
        const int e = interior_elem(ax, j), ec = interior_elem(ax, jc);
        const double2 z0 = c0(e), z1 = c1(e);
        double2 h0 = z0, h1 = z1;
        if (!io.half) {  // half-spectrum columns are exactly Hermitian already
          h0 = cscale(cadd(z0, cconj(c0(ec))), 0.5);
          h1 = cscale(cadd(z1, cconj(c1(ec))), 0.5);
        }
        const double2 z = make_double2(h0.x - h1.y, h0.y + h1.x);
        val = cmul(cconj(z), __ldg(&chirp[j]));
        if (dots) {
          const double2 ca = __ldg(&ax.c_a[j]), cb = __ldg(&ax.c_b[j]);
          const double2 t0 = cmul(ca, z0), b0 = cmul(cb, z0);
          const double2 t1 = cmul(ca, z1), b1 = cmul(cb, z1);
          acc[0] += t0.x, acc[1] += t0.y, acc[2] += b0.x, acc[3] += b0.y;
          acc[4] += t1.x, acc[5] += t1.y, acc[6] += b1.x, acc[7] += b1.y;
        }
      }
      x[pidx(j)] = val;
    }
  } else {  // IK_FOURIER: F^H v = conj(F conj(v)) (trig.cpp:116-124)
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      double2 val = czero();
      if (j < m) {
        const double2 z = c0(interior_elem(ax, j));
        val = cmul(cconj(z), __ldg(&chirp[j]));
        if (dots) {
          const double2 t = cmul(__ldg(&ax.c_a[j]), z), bt = cmul(__ldg(&ax.c_b[j]), z);
          acc[0] += t.x, acc[1] += t.y;
          acc[2] += bt.x, acc[3] += bt.y;
        }
      }
      x[pidx(j)] = val;
    }
  }
  if (dots) block_sum<8>(acc, red);
  __syncthreads();

  if constexpr (LOGM > 0)
    bluestein_t<LOGM, kLineNT<LOGM>>(x, ax.fft, tw, ax.fft.M);
  else
    bluestein_core(x, ax.fft, tw, ax.fft.M);

  const long long oo0 = line_offset(io.go, l0);
  const long long oo1 = has1 ? line_offset(io.go, l0 + 1) : oo0;
  const long long eso = io.go.elem_stride;
  const double inv_sqrt_m = 1.0 / sqrt((double)m);
  double im2 = 0.0;
  for (int p = threadIdx.x; p < m; p += blockDim.x) {
    double2 in0, in1 = czero();
    if (ax.kind == IK_COS) {
      const int idx = (p & 1) ? m - 1 - (p >> 1) : (p >> 1);  // trig.cpp:154-157
      const double2 Z = cmul(x[pidx(idx)], __ldg(&chirp[idx]));
      in0 = make_double2(Z.x, 0.0);
      in1 = make_double2(Z.y, 0.0);
    } else if (ax.kind == IK_SINE) {
      const double sc = -0.5 * sqrt(2.0 / ((double)m + 1.0));
      const double2 Z = cmul(x[pidx(p + 1)], __ldg(&chirp[p + 1]));
      in0 = make_double2(sc * Z.y, 0.0);
      in1 = make_double2(-sc * Z.x, 0.0);
    } else if (hpack) {
      const double2 Z = cconj(cmul(x[pidx(p)], __ldg(&chirp[p])));
      in0 = make_double2(Z.x * inv_sqrt_m, 0.0);
      in1 = make_double2(Z.y * inv_sqrt_m, 0.0);
    } else {
      in0 = cscale(cconj(cmul(x[pidx(p)], __ldg(&chirp[p]))), inv_sqrt_m);
    }
    const int e = interior_elem(ax, p);
    if (ax.hob) {
      // y_I = F^H b + P_I a; border rows whose 2 pi image is p: (F^H b)_p + P_B a
      if (ax.cplx && !hpack) {
        const double2 o = cadd(in0, ho_poly(ax, ua0, e));
        st_out(io, oo0 + e * eso, o);
        im2 += o.y * o.y;
        for (int l = 0; l < ax.hk; ++l)
          if (ax.wrap[l] == p) {
            const double2 ob = cadd(in0, ho_poly(ax, ua0, ax.bord[l]));
            st_out(io, oo0 + ax.bord[l] * eso, ob);
            im2 += ob.y * ob.y;
          }
      } else {
        st_out(io, oo0 + e * eso, make_double2(in0.x + ho_poly(ax, ua0, e).x, 0.0));
        if (has1)
          st_out(io, oo1 + e * eso,
              make_double2(in1.x + ho_poly(ax, ua1, e).x, 0.0));
        for (int l = 0; l < ax.hk; ++l)
          if (ax.wrap[l] == p) {
            const int eb = ax.bord[l];
            st_out(io, oo0 + eb * eso,
                make_double2(in0.x + ho_poly(ax, ua0, eb).x, 0.0));
            if (has1)
              st_out(io, oo1 + eb * eso,
                  make_double2(in1.x + ho_poly(ax, ua1, eb).x, 0.0));
          }
      }
    } else if (ax.bordered) {
      const double qi = __ldg(&ax.q[e]), qr = __ldg(&ax.q[n - 1 - e]);
      if (ax.cplx && !hpack) {
        const double2 o = cadd(cadd(cscale(u00, qi), in0), cscale(un0, qr));
        st_out(io, oo0 + e * eso, o);
        im2 += o.y * o.y;
      } else {
        const double o = qi * u00.x + in0.x + qr * un0.x;
        st_out(io, oo0 + e * eso, make_double2(o, 0.0));
        if (has1) {
          const double o1 = qi * u01.x + in1.x + qr * un1.x;
          st_out(io, oo1 + e * eso, make_double2(o1, 0.0));
        }
      }
    } else {
      st_out(io, oo0 + e * eso, in0);
      if (!hpack) im2 += in0.y * in0.y;
      if (has1) st_out(io, oo1 + e * eso, in1);
    }
  }
  if (ax.bordered && threadIdx.x == 0) {
    const double q0 = ax.q[0];
    for (int t = 0; t < (has1 ? 2 : 1); ++t) {
      const double2 u0 = t == 0 ? u00 : u01, un = t == 0 ? un0 : un1;
      const double2 top = make_double2(acc[4 * t + 0], acc[4 * t + 1]);
      const double2 bot = make_double2(acc[4 * t + 2], acc[4 * t + 3]);
      const double2 o0 = cadd(cscale(u0, q0), top);
      const double2 on = cadd(bot, cscale(un, q0));
      const long long oo = t == 0 ? oo0 : oo1;
      st_out(io, oo, o0);
      st_out(io, oo + (long long)(n - 1) * eso, on);
      if (ax.cplx && !hpack) im2 += o0.y * o0.y + on.y * on.y;
    }
  }
  if (ax.cplx && sa.resid2 != nullptr) {
    double v[1] = {im2};
    block_sum<1>(v, red);
    if (threadIdx.x == 0) sa.resid2[l0] = v[0];
  }
}

// ---------------------------------------------------------------------------
// Real lines through the half-length complex DFT (one line per CTA).
//   R2C (analyze):  X = DFT_R(x), x real, R even, h = R/2:
//     z_j = x_{2j} + i x_{2j+1},  Z = DFT_h(z),
//     E_k = (Z_k + conj Z_{-k})/2,  O_k = -i (Z_k - conj Z_{-k})/2,
//     X_k = E_k + W_R^k O_k,  X_{k+h} = E_k - W_R^k O_k.
//   C2R (synthesize):  x_j = sum_q X_q e^{+2 pi i jq/R} for Hermitian X:
//     Zin_k = (X_k + X_{k+h}) + i (X_k - X_{k+h}) W_R^{-k},  z = IDFT_h(Zin),
//     x_{2j} = Re z_j,  x_{2j+1} = Im z_j.
// A real line of even length is exactly the interleaved complex buffer z, so
// the Bluestein size drops from M >= 2R-1 to M >= R-1 (4096 at n = 4096): a
// 70 KB buffer, several CTAs per SM.  The interior kinds map on this as
//   cosine (DCT-II / III, trig.cpp:126-160): Makhoul reorder + quarter-wave twiddle,
//     DCT-III via Re DFT(buf) = C2R(herm(conj buf));
//   Fourier (F / F^H, real data): R2C / C2R of length m (Re F^H c = F^H herm(c));
//   sine (DST-I, trig.cpp:162-180): R2C of the odd extension, R = 2(m+1).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk global -> shared copy (TMA engine, UBLKCP), completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch of [src, src + bytes) into L2 (TMA engine, no completion);
// src and bytes 16-byte aligned
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
}
}  // namespace fdb
#include "fd_tc.cuh"
namespace fdb {

__device__ __forceinline__ int makhoul_src(int p, int m, int half) {
  return p < half ? 2 * p : 2 * (m - 1 - p) + 1;  // trig.cpp:139-141
}

// Two-level table of a twiddle sequence t_k (k < len) in shared memory:
// t_k = hi[k >> 6] * lo[k & 63] (both exact entries of the global table).
struct Tw2 {
  const double2* lo;
  const double2* hi;
  __device__ __forceinline__ double2 operator()(int k) const {
    return cmul(hi[k >> 6], lo[k & 63]);
  }
};
__host__ __device__ __forceinline__ int tw2_slots(int len) {
  return len > 0 ? 64 + ((len + 63) >> 6) : 0;
}
__device__ __forceinline__ Tw2 load_tw2(double2* slots, const double2* tab, int len) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x)
    if (i < len) slots[i] = tab[i];
  const int nhi = (len + 63) >> 6;
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) slots[64 + i] = tab[i << 6];
  return Tw2{slots, slots + 64};
}

// boundary column q_e (boundary.cpp:162-217) in registers
__device__ __forceinline__ double q_at(const AxisDev& ax, int e) {
  if (ax.qmode == 0) return (1.0 - e * ax.q_s) * ax.q_inv;
  const double t = ax.q_gb - fma((double)e, ax.q_s, ax.q_o);
  return t * t * ax.q_inv;
}

// a q[s+1] + b q[n-2-s] over the interior index s, in the factored form
//   q[s+1] = k (qa1 - q_s s)^p,  q[n-2-s] = k (qa2 + q_s s)^p   (p = 2, or 1 for qmode 0).
// The amplitudes are O(n |y|) (alpha (y_0 - beta_0)), while q decays to ~0 at
// the far end: expanded into monomials of s the terms cancel there and leave
// an absolute error eps |a| q_0 on EVERY sample -- white noise on the
// transform's input that the Tikhonov gain amplifies (measured: restoration
// error 4x the reference's in 1D, 40x in 2D at n = 4096).  The factored form
// keeps each term relatively accurate, like the reference's q[e] * u products
// (boundary.cpp:225-250, 253-289).
struct BorderPoly {
  double ak, bk, qa1, qa2, qs;
  int lin;
  __device__ __forceinline__ double operator()(int s) const {
    const double t = (double)s;
    const double t1 = fma(-qs, t, qa1), t2 = fma(qs, t, qa2);
    if (lin) return fma(ak, t1, bk * t2);
    return fma(ak * t1, t1, (bk * t2) * t2);
  }
};
__device__ __forceinline__ BorderPoly border_poly(const AxisDev& ax, double a, double b) {
  BorderPoly p;
  p.ak = a * ax.q_inv;
  p.bk = b * ax.q_inv;
  p.qa1 = ax.qa1;
  p.qa2 = ax.qa2;
  p.qs = ax.q_s;
  p.lin = ax.qmode == 0;
  return p;
}

// Border terms of T_X^{-1} y for a real line (transform_apply_inverse,
// boundary.cpp:253-289).  row_a / row_b are unit impulses, so the two dot
// products are two samples and every thread solves the 2x2 system itself.
// The interior coefficients are  xi + (y0 - b0) v + (yn - b1) w  with the
// tables v = -alpha X qhat, w = -alpha X J qhat, exactly the reference's form.
// (Round 1 folded the border into the transform input instead:
//   y0 v + xi + yn w - (b0 v + b1 w) = X (x - o0 qhat - on J qhat),
// algebraically the same and table-free, but the folded polynomial is up to
// ~n alpha times larger than the data, so the transform's rounding error --
// proportional to its input -- lands on every frequency instead of following
// the decay of v and w: restorations at n = 4096 differed from the reference
// by 6e-10 in 2D even with numpy's FFT in place of ours, 25x the spread
// between the reference and its numpy restatement; DESIGN 4.)
struct Fold {
  double o0, on;  // border coefficients alpha (y_0 - beta_0), alpha (y_{n-1} - beta_1)
  double c0, c1;  // y_0 - beta_0, y_{n-1} - beta_1: the factors of v and w
};
template <class LD>
__device__ __forceinline__ Fold fold_terms(const AxisDev& ax, LD ld) {
  Fold f{0.0, 0.0, 0.0, 0.0};
  if (!ax.bordered) return f;
  const double y0 = ld(0), yn = ld(ax.n - 1);
  double b0 = 0.0, b1 = 0.0;
  if (ax.correction) {
    const double xa = ld(ax.ia + 1), xb = ld(ax.ib + 1);
    const double ra = (ax.cavr[0] * y0 + ax.cavr[1] * yn) + ax.ra1 * xa;
    const double rb = (ax.cavr[2] * y0 + ax.cavr[3] * yn) + ax.rb1 * xb;
    const double* ci = ax.capi;  // capacitance^-1 (boundary.cpp:278-286 solves by Cramer's rule)
    b0 = ci[0] * ra + ci[1] * rb;
    b1 = ci[2] * ra + ci[3] * rb;
  }
  const double al = ax.alpha;
  f.o0 = al * y0 - b0 * al;
  f.on = al * yn - b1 * al;
  f.c0 = y0 - b0;
  f.c1 = yn - b1;
  return f;
}

// smem of the real-line kernels: buffer, FFT twiddles, rtw and DCT tables,
// then one mbarrier
__host__ __device__ __forceinline__ int rline_slots(const AxisDev& ax, int Mloc) {
  return pidx(Mloc) + 1 + kTwSlots + tw2_slots(ax.hfft.L) +
         (ax.kind == IK_COS ? tw2_slots(ax.m) : 0);
}

// Input staging of the real-line kernels: the n doubles of the NEXT line are
// bulk-copied (TMA engine) into the upper part of the FFT buffer, which is
// free from the end of the convolution until the next line's first DIF pass
// (the load phase writes only [0, h) and that pass reads the rest as zero).
// A line is staged when its row is contiguous and 16-byte aligned.
struct Stage {
  double* buf;     // smem, >= n doubles
  uint64_t* bar;   // mbarrier
  bool on;         // kernel-level: layout allows staging
  uint32_t phase;
};
__device__ __forceinline__ bool stage_line(const Stage& s, const LineIO& io, int l, int n) {
  if (!s.on || l >= io.gi.count) return false;
  const double* src = reinterpret_cast<const double*>(io.in) + line_offset(io.gi, l);
  return (reinterpret_cast<uintptr_t>(src) & 15) == 0;
}
// thread 0: start the copy of line l (after a barrier that ends all reads of
// the region through the generic proxy)
__device__ __forceinline__ void stage_issue(Stage& s, const LineIO& io, int l, int n) {
  if (!stage_line(s, io, l, n)) return;
  const double* src = reinterpret_cast<const double*>(io.in) + line_offset(io.gi, l);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(s.bar, (uint32_t)n * 8);
  bulk_g2s(s.buf, src, (uint32_t)n * 8, s.bar);
}
__device__ __forceinline__ Stage stage_init(double2* x, int h, int Mloc, double2* after, int n,
                                            const LineIO& io, bool big) {
  Stage s;
  s.buf = reinterpret_cast<double*>(x + pidx(h) + 1);
  s.bar = reinterpret_cast<uint64_t*>(after);
  s.phase = 0;
  s.on = !big && io.gi.elem_stride == 1 && (n & 1) == 0 &&
         2LL * (pidx(Mloc) - pidx(h)) >= (long long)n;
  if (threadIdx.x == 0 && s.on) {
    mbar_init(s.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  return s;
}

// scr != null: split-convolution mode for M beyond shared memory
// (bluestein_half), persistent over lines, 2h complex of per-CTA scratch.
// io.pack (Fourier interior): the line is stored Hermitian-packed in n doubles
//   [border0, border_n-1] [X_0, X_h] X_1 .. X_{h-1}   (double2 slots; the
//   border slot only when bordered) -- the coefficients of real data in this
//   basis are exactly Hermitian once the border is folded in.
// Optional phase timing of the real-line kernels (build with -DFD_PHASE_CLOCKS):
// thread 0 of every CTA adds the SM clocks of [line start, load done),
// [load done, convolution done), [convolution done, line done) and the
// staging wait at the line start, per kernel.
#ifdef FD_PHASE_CLOCKS
__device__ unsigned long long g_phase_clocks[2][4];
#define FD_CLK(v) long long clk_##v = clock64()
#define FD_CLK_SET(v) clk_##v = clock64()
#define FD_CLK_ADD(k, i, a, b) \
  if (threadIdx.x == 0) \
  atomicAdd(&g_phase_clocks[k][i], (unsigned long long)((clk_##b) - (clk_##a)))
#else
#define FD_CLK(v)
#define FD_CLK_SET(v)
#define FD_CLK_ADD(k, i, a, b)
#endif

// LOGM > 0: size-specialised Bluestein core (bluestein_t), blockDim = FftShape<LOGM>::NT
template <int LOGM>
__global__ void __launch_bounds__(256, 2) k_ranalyze(AxisDev ax, LineIO io, double2* scr) {
  extern __shared__ double2 sm[];
  const FftTables& T = ax.hfft;
  const int M = T.M, h = T.L;
  const bool big = scr != nullptr;
  const int Mloc = big ? M / 2 : M;
  double2* x = sm;
  double2* slots = sm + pidx(Mloc) + 1;
  const TwSm tw = load_twiddles(slots, T);
  const Tw2 rtw = load_tw2(slots + kTwSlots, ax.rtw, h);
  Tw2 dtw{nullptr, nullptr};
  if (ax.kind == IK_COS) dtw = load_tw2(slots + kTwSlots + tw2_slots(h), ax.dct_tw, ax.m);
  const bool pk = io.pack && ax.kind == IK_FOURIER;
  double2* scrA = big ? scr + (long long)blockIdx.x * 2 * h : nullptr;
  double2* scrY = big ? scrA + h : nullptr;
  Stage stg = stage_init(x, h, Mloc, sm + rline_slots(ax, Mloc), ax.n, io, big);
  const double2* chirp = T.chirp;
  if (io.chirp_smem) {  // persistent CTA: the chirp once per CTA in shared memory
    double2* cs = sm + rline_slots(ax, Mloc) + 1;
    for (int j = threadIdx.x; j < h; j += blockDim.x) cs[j] = T.chirp[j];
    chirp = cs;
  }
  auto chirp_at = [&](int j) { return io.chirp_smem ? chirp[j] : __ldg(&chirp[j]); };
  __syncthreads();
  if (threadIdx.x == 0) stage_issue(stg, io, blockIdx.x, ax.n);
  for (int l = blockIdx.x; l < io.gi.count; l += gridDim.x) {
  const long long oi = line_offset(io.gi, l), es = io.gi.elem_stride;
  const int n = ax.n, m = ax.m;
  const double* in = reinterpret_cast<const double*>(io.in);
  FD_CLK(c0);
  const bool st = stage_line(stg, io, l, n);
  if (st) {
    mbar_wait(stg.bar, stg.phase);
    stg.phase ^= 1;
  }
  FD_CLK(cw);
  FD_CLK_ADD(0, 3, c0, cw);
  const double* sin_ = stg.buf;
  const double* gin = in + oi;
  Fold fd;
  // the load phase, instantiated for the staged (shared) and the global source
  auto load_phase = [&](auto ld) {
  fd = fold_terms(ax, ld);
  // interior sample s
  auto xin = [&](int s) { return ld(interior_elem(ax, s)); };
  const int half = (m + 1) / 2;
#pragma unroll 4
  for (int j = threadIdx.x; j < h; j += blockDim.x) {
    const int p0 = 2 * j, p1 = 2 * j + 1;
    double a, b;
    if (ax.kind == IK_SINE) {
      const int R = 2 * (m + 1);
      auto ext = [&](int p) -> double {
        if (p == 0 || p == m + 1) return 0.0;
        if (p <= m) return xin(p - 1);
        return -xin(R - 1 - p);
      };
      a = ext(p0);
      b = ext(p1);
    } else {
      a = xin(ax.kind == IK_COS ? makhoul_src(p0, m, half) : p0);
      b = xin(ax.kind == IK_COS ? makhoul_src(p1, m, half) : p1);
    }
    x[pidx(j)] = cmul(make_double2(a, b), chirp_at(j));
  }
  };
  if (st)
    load_phase([&](int e) { return sin_[e]; });
  else if (es == 1)
    load_phase([&](int e) { return __ldg(gin + e); });
  else
    load_phase([&](int e) { return __ldg(gin + (long long)e * es); });
  __syncthreads();

  FD_CLK(c1);
  FD_CLK(c2);
  if (!big) {
    if constexpr (LOGM > 0)
      bluestein_t<LOGM, 0, true>(x, T, tw, h);
    else
      bluestein_core<true>(x, T, tw, h);
    // the post phase reads [0, h) only: stage the next line behind it
    if (threadIdx.x == 0) stage_issue(stg, io, l + gridDim.x, n);
    FD_CLK_SET(c2);
    FD_CLK_ADD(0, 0, c0, c1);
    FD_CLK_ADD(0, 1, c1, c2);
  } else {
    for (int j = threadIdx.x; j < h; j += blockDim.x) scrA[j] = x[pidx(j)];
    bluestein_half<true>(x, T, tw, 1, h);  // x = a (.) W, convolved: y1
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
      scrY[j] = x[pidx(j)];
      x[pidx(j)] = scrA[j];
    }
    __syncthreads();
    bluestein_half<true>(x, T, tw, 0, h);  // y0
  }
  // Z_k = (a * b)_k c_k; in split mode the lower half of the last DIT stage
  auto zv = [&](int k) {
    const double2 y = big ? cadd(x[pidx(k)], cmulc(scrY[k], tw(k))) : x[pidx(k)];
    return cmul(y, chirp_at(k));
  };

  const long long oo = line_offset(io.go, l), eso = io.go.elem_stride;
  double2* P = reinterpret_cast<double2*>(reinterpret_cast<double*>(io.out) + oo);
  const int off = ax.bordered ? 1 : 0;
  const double inv_sqrt_m = ax.inv_sqrt_m;
  const double s0 = ax.dct_s0, s1 = ax.dct_s1;
  double* wl = io.wout ? io.wout + (long long)l * io.wstride : nullptr;
  const long long nkb32 = io.wstride >> 5;
  auto wset = [&](long long i, double v) {  // GCV weight (and its TF32 split for the screen)
    wl[i] = v;
    if (io.wout32) {
      float hi, lo;
      tf32_split(v, hi, lo);
      const long long t = tc_tile_index(l, i, kTcBM, nkb32);
      io.wout32[t] = hi;
      io.wout32lo[t] = lo;
    }
  };
  if (wl)
    for (long long i = io.wn + threadIdx.x; i < io.wstride; i += blockDim.x) wset(i, 0.0);
  // + (y0 - b0) v_i + (yn - b1) w_i on interior coefficient i (boundary.cpp:271-287)
  const double c0 = fd.c0, c1 = fd.c1;
  const bool brd = ax.bordered != 0;
  auto corr = [&](int i, double2 o) {
    if (!brd) return o;
    if (ax.cplx) {
      const double2 v = __ldg(&ax.v[i]), w = __ldg(&ax.w[i]);
      o.x += c0 * v.x + c1 * w.x;
      o.y += c0 * v.y + c1 * w.y;
    } else {
      o.x += c0 * __ldg(&ax.vr[i]) + c1 * __ldg(&ax.wr[i]);
    }
    return o;
  };
  auto emit = [&](int i, double2 o) {
    const int e = interior_elem(ax, i);
    o = corr(i, o);
    stc(io.out, io.out_cplx, oo + e * eso, o);
    if (wl && !ax.cplx) wset(e, o.x * o.x);
  };
  auto nrm = [](double2 a) { return a.x * a.x + a.y * a.y; };
  if (ax.kind == IK_FOURIER) {
    // groups {k, h-k}: both Hermitian partners of each coefficient come out of
    // the same pair (Z_k, Z_{h-k}), so the GCV weights |g_k|^2 + |g_{m-k}|^2
    // are formed in registers
    for (int k = threadIdx.x; k <= h / 2; k += blockDim.x) {
      const int kp = k == 0 ? 0 : h - k;
      const double2 Zk = zv(k);
      const double2 Zp = zv(kp);
      const double2 E = cscale(cadd(Zk, cconj(Zp)), 0.5);
      const double2 D = csub(Zk, cconj(Zp));
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
      const double2 WO = cmul(rtw(k), O);
      const double2 ok = corr(k, cscale(cadd(E, WO), inv_sqrt_m));
      const double2 okh = corr(k + h, cscale(csub(E, WO), inv_sqrt_m));
      const double2 WOp = cmul(rtw(kp), cconj(O));
      const double2 okp = corr(kp, cscale(cadd(cconj(E), WOp), inv_sqrt_m));
      const double2 okph = corr(kp + h, cscale(csub(cconj(E), WOp), inv_sqrt_m));
      if (pk) {
        if (k == 0) {
          P[off] = make_double2(ok.x, okh.x);
        } else {
          P[off + k] = ok;
          if (kp != k) P[off + kp] = okp;
        }
      } else {  // already corrected: plain stores
        auto put = [&](int i, double2 o) {
          stc(io.out, io.out_cplx, oo + interior_elem(ax, i) * eso, o);
        };
        put(k, ok);
        put(k + h, okh);
        if (kp != k) {
          put(kp, okp);
          put(kp + h, okph);
        }
      }
      if (wl) {
        if (k == 0) {  // singleton group {0}: self pairs 0 and h
          wset(off, nrm(ok));
          wset(off + h, nrm(okh));
        } else if (kp != k) {
          wset(off + k, nrm(ok) + nrm(okph));   // pair (k, m-k = kp+h)
          wset(off + kp, nrm(okp) + nrm(okh));  // pair (kp, m-kp = k+h)
        } else {
          wset(off + k, nrm(ok) + nrm(okh));  // k = h/2: pair (k, k+h)
        }
      }
    }
  } else {
    for (int k = threadIdx.x; k < h; k += blockDim.x) {
      const int kc = k == 0 ? 0 : h - k;
      const double2 Zk = zv(k);
      const double2 Zc = cconj(zv(kc));
      const double2 E = cscale(cadd(Zk, Zc), 0.5);
      const double2 D = csub(Zk, Zc);
      const double2 WO = cmul(rtw(k), make_double2(0.5 * D.y, -0.5 * D.x));
      const double2 X0 = cadd(E, WO), X1 = csub(E, WO);  // X_k, X_{k+h}
      if (ax.kind == IK_SINE) {
        if (k >= 1) emit(k - 1, make_double2(ax.dst_scale * X0.y, 0.0));
      } else {
        const double2 t0 = dtw(k), t1 = dtw(k + h);
        emit(k, make_double2((k == 0 ? s0 : s1) * (t0.x * X0.x - t0.y * X0.y), 0.0));
        emit(k + h, make_double2(s1 * (t1.x * X1.x - t1.y * X1.y), 0.0));
      }
    }
  }
  if (ax.bordered && threadIdx.x == 0) {
    const double2 o0 = make_double2(fd.o0, 0.0), on = make_double2(fd.on, 0.0);
    if (pk) {
      P[0] = make_double2(fd.o0, fd.on);
    } else {
      stc(io.out, io.out_cplx, oo, o0);
      stc(io.out, io.out_cplx, oo + (long long)(n - 1) * eso, on);
    }
    if (wl) {
      wset(0, fd.o0 * fd.o0);
      wset(ax.cplx ? h + 2 : n - 1, fd.on * fd.on);
    }
  }
  __syncthreads();  // x and the scratch are reused by the next line
#ifdef FD_PHASE_CLOCKS
  if (!big) {
    FD_CLK(c3);
    FD_CLK_ADD(0, 2, c2, c3);
  }
#endif
  }
}

// Real output of T_X c (transform_apply, boundary.cpp:225-250) with the
// filter of the restoration fused into the coefficient loads.  The two border
// dots c_a . c_mid, c_b . c_mid are samples of the interior synthesis
// (top_i, bot_i), written by the thread that produces them.
// scr != null: split-convolution mode (see k_ranalyze); io.pack: packed input.
// LOGM > 0: size-specialised Bluestein core (bluestein_t), blockDim = FftShape<LOGM>::NT
template <int LOGM>
__global__ void __launch_bounds__(256, 2) k_rsynth(AxisDev ax, LineIO io, SynthArgs sa,
                                                   double2* scr) {
  extern __shared__ double2 sm[];
  const FftTables& T = ax.hfft;
  const int M = T.M, h = T.L;
  const bool big = scr != nullptr;
  const int Mloc = big ? M / 2 : M;
  double2* x = sm;
  double2* slots = sm + pidx(Mloc) + 1;
  const TwSm tw = load_twiddles(slots, T);
  const Tw2 rtw = load_tw2(slots + kTwSlots, ax.rtw, h);
  Tw2 dtw{nullptr, nullptr};
  if (ax.kind == IK_COS) dtw = load_tw2(slots + kTwSlots + tw2_slots(h), ax.dct_tw, ax.m);
  const bool pk = io.pack && ax.kind == IK_FOURIER;
  double2* scrA = big ? scr + (long long)blockIdx.x * 2 * h : nullptr;
  double2* scrY = big ? scrA + h : nullptr;
  // staging needs real (or packed) input lines of n doubles
  Stage stg = stage_init(x, h, Mloc, sm + rline_slots(ax, Mloc), ax.n, io,
                         big || (io.in_cplx && !pk));
  const double2* chirp = T.chirp;
  if (io.chirp_smem) {  // persistent CTA: the chirp once per CTA in shared memory
    double2* cs = sm + rline_slots(ax, Mloc) + 1;
    for (int j = threadIdx.x; j < h; j += blockDim.x) cs[j] = T.chirp[j];
    chirp = cs;
  }
  auto chirp_at = [&](int j) { return io.chirp_smem ? chirp[j] : __ldg(&chirp[j]); };
  __syncthreads();
  if (threadIdx.x == 0) stage_issue(stg, io, blockIdx.x, ax.n);
  for (int l = blockIdx.x; l < io.gi.count; l += gridDim.x) {
  const long long oi = line_offset(io.gi, l);
  const int n = ax.n, m = ax.m;
  FD_CLK(c0);
  const bool st = stage_line(stg, io, l, n);
  if (st) {
    mbar_wait(stg.bar, stg.phase);
    stg.phase ^= 1;
  }
  FD_CLK(cw);
  FD_CLK_ADD(1, 3, c0, cw);
  const double mu = line_mu(sa, io.gi, l);
  auto filt = [&](int e, double2 c) { return coeff_filter_fast(ax, sa, io.gi, l, e, c, mu); };
  auto cf = [&](int e) {
    return filt(e, st ? make_double2(stg.buf[e], 0.0)
                      : ldc(io.in, io.in_cplx, oi + e * io.gi.elem_stride));
  };
  const double2* Pin =
      st ? reinterpret_cast<const double2*>(stg.buf)
         : reinterpret_cast<const double2*>(reinterpret_cast<const double*>(io.in) + oi);
  auto ldp = [&](int i) { return st ? Pin[i] : __ldg(Pin + i); };
  const int off = ax.bordered ? 1 : 0;
  double u0 = 0.0, un = 0.0;
  if (ax.bordered) {
    if (pk) {
      const double2 b = ldp(0);
      u0 = filt(0, make_double2(b.x, 0.0)).x;
      un = filt(n - 1, make_double2(b.y, 0.0)).x;
    } else {
      u0 = cf(0).x;
      un = cf(n - 1).x;
    }
  }
  if (ax.kind == IK_SINE) {  // Q c_mid: R2C of the odd extension (Q is an involution)
    const int R = 2 * (m + 1);
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
      auto ext = [&](int p) -> double {
        if (p == 0 || p == m + 1) return 0.0;
        if (p <= m) return cf(interior_elem(ax, p - 1)).x;
        return -cf(interior_elem(ax, R - 1 - p)).x;
      };
      x[pidx(j)] = cmul(make_double2(ext(2 * j), ext(2 * j + 1)), chirp_at(j));
    }
  } else {
    // cosine works on conj(buf_i) = s_i c_i conj(tw_i) (DCT-III, trig.cpp:147-158)
    const double s0 = ax.dct_s0, s1 = ax.dct_s1;
    auto val_at = [&](int i) {
      const double2 c = cf(interior_elem(ax, i));
      if (ax.kind == IK_COS) {
        const double2 t = dtw(i);
        const double ts = (i == 0 ? s0 : s1) * c.x;
        return make_double2(ts * t.x, -(ts * t.y));
      }
      return c;
    };
    // C2R pre-pass over the closed index groups {k, h-k}: X = herm(c),
    // Zin_k = (X_k + X_{k+h}) + i (X_k - X_{k+h}) W^{-k}; Bluestein input conj(Zin) c_k.
    // Each coefficient is read exactly once, straight from global memory.
    auto zin = [&](int kk, double2 Xa, double2 Xb) {
      const double2 Od = cmulc(csub(Xa, Xb), rtw(kk));
      const double2 Ev = cadd(Xa, Xb);
      return make_double2(Ev.x - Od.y, Ev.y + Od.x);
    };
    // Fast path (packed Fourier line, 1D filter of a complex basis, h / 2 < 4
    // blockDim): straight-line batches of two groups, the coefficient pairs and
    // the spectral values of a batch all requested before the first is used.
    // The generic loop below runs group after group behind the filter's mode
    // branches, one cache round trip each (see k_msynth).
    const bool fastpk = pk && sa.mode == 1 && sa.sp.mode == 1 && ax.cplx &&
                        h / 2 < 4 * (int)blockDim.x;
    if (fastpk) {
      const double2* dA = sa.sp.dA;
      const double* sA = sa.sp.sA;
      const int kl = ax.kl;
      auto fil = [&](double2 d, double sv) {  // conj(d) / (|d|^2 + mu s^2)
        const double r = rcp_pos((d.x * d.x + d.y * d.y) + mu * sv * sv);
        return make_double2(d.x * r, -d.y * r);
      };
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        double2 ck[2], cp[2], dk[2], dp[2];
        double sk[2], sp[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int kq = threadIdx.x + (2 * b + u) * blockDim.x;
          const int k = kq <= h / 2 ? kq : h / 2;
          const int kp = k == 0 ? 0 : h - k;
          // k = 0: the packed pair (X_0, X_h), two real coefficients at e = kl, kl + h
          ck[u] = ldp(off + k);
          cp[u] = ldp(off + kp);
          dk[u] = __ldg(dA + kl + k);
          sk[u] = sA ? __ldg(sA + kl + k) : 1.0;
          const int ep = k == 0 ? kl + h : kl + kp;
          dp[u] = __ldg(dA + ep);
          sp[u] = sA ? __ldg(sA + ep) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = threadIdx.x + (2 * b + u) * blockDim.x;
          if (k > h / 2) continue;
          const int kp = k == 0 ? 0 : h - k;
          double2 Xk, Xkh, Xp, Xph;
          if (k == 0) {
            Xk = Xp = cmul(make_double2(ck[u].x, 0.0), fil(dk[u], sk[u]));
            Xkh = Xph = cmul(make_double2(ck[u].y, 0.0), fil(dp[u], sp[u]));
          } else {
            const double2 fk = cmul(ck[u], fil(dk[u], sk[u]));
            const double2 fp = kp != k ? cmul(cp[u], fil(dp[u], sp[u])) : fk;
            Xk = fk;
            Xp = fp;
            Xkh = cconj(fp);  // m - (k+h) = kp
            Xph = cconj(fk);
          }
          x[pidx(k)] = cmul(cconj(zin(k, Xk, Xkh)), chirp_at(k));
          if (kp != k) x[pidx(kp)] = cmul(cconj(zin(kp, Xp, Xph)), chirp_at(kp));
        }
      }
    } else
    for (int k = threadIdx.x; k <= h / 2; k += blockDim.x) {
      const int kp = k == 0 ? 0 : h - k;
      double2 Xk, Xkh, Xp, Xph;  // X at k, k+h, kp, kp+h
      if (pk) {  // exactly Hermitian: X_{m-q} = conj X_q
        if (k == 0) {
          const double2 b = ldp(off);
          Xk = Xp = filt(interior_elem(ax, 0), make_double2(b.x, 0.0));
          Xkh = Xph = filt(interior_elem(ax, h), make_double2(b.y, 0.0));
        } else {
          const double2 fk = filt(interior_elem(ax, k), ldp(off + k));
          const double2 fp = kp != k ? filt(interior_elem(ax, kp), ldp(off + kp)) : fk;
          Xk = fk;
          Xp = fp;
          Xkh = cconj(fp);  // m - (k+h) = kp
          Xph = cconj(fk);
        }
      } else {
        // herm(q) = (v_q + conj v_{m-q})/2: m-k = kp+h, m-(k+h) = kp (k = 0: 0 and h)
        const double2 vk = val_at(k), vkh = val_at(k + h);
        const double2 vp = kp != k ? val_at(kp) : vk, vph = kp != k ? val_at(kp + h) : vkh;
        Xk = cscale(cadd(vk, cconj(k == 0 ? vk : vph)), 0.5);
        Xkh = cscale(cadd(vkh, cconj(k == 0 ? vkh : vp)), 0.5);
        Xp = cscale(cadd(vp, cconj(k == 0 ? vp : vkh)), 0.5);
        Xph = cscale(cadd(vph, cconj(k == 0 ? vph : vk)), 0.5);
      }
      x[pidx(k)] = cmul(cconj(zin(k, Xk, Xkh)), chirp_at(k));
      if (kp != k) x[pidx(kp)] = cmul(cconj(zin(kp, Xp, Xph)), chirp_at(kp));
    }
  }
  __syncthreads();

  FD_CLK(c1);
  FD_CLK(c2);
  if (!big) {
    if constexpr (LOGM > 0)
      bluestein_t<LOGM, 0, true>(x, T, tw, h);
    else
      bluestein_core<true>(x, T, tw, h);
    if (threadIdx.x == 0) stage_issue(stg, io, l + gridDim.x, n);
    FD_CLK_SET(c2);
    FD_CLK_ADD(1, 0, c0, c1);
    FD_CLK_ADD(1, 1, c1, c2);
  } else {
    for (int j = threadIdx.x; j < h; j += blockDim.x) scrA[j] = x[pidx(j)];
    bluestein_half<true>(x, T, tw, 1, h);
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
      scrY[j] = x[pidx(j)];
      x[pidx(j)] = scrA[j];
    }
    __syncthreads();
    bluestein_half<true>(x, T, tw, 0, h);
  }
  auto zv = [&](int k) {
    const double2 y = big ? cadd(x[pidx(k)], cmulc(scrY[k], tw(k))) : x[pidx(k)];
    return cmul(y, chirp_at(k));
  };

  const long long oo = line_offset(io.go, l), eso = io.go.elem_stride;
  double* out = reinterpret_cast<double*>(io.out);
  const BorderPoly bp = border_poly(ax, u0, un);  // q[e] u0 + q[n-1-e] un, e = p + 1
  auto put = [&](int p, double val) {  // interior position p of the output line
    const int e = interior_elem(ax, p);
    double o = val;
    if (ax.bordered) o = val + bp(p);
    out[oo + e * eso] = o;
  };
  // interior synthesis sample p (before the border terms), read back from x
  auto interior_at = [&](int p) {
    if (ax.kind == IK_COS) {  // inverse of the Makhoul placement below
      const int half = (m + 1) / 2;
      const int sp = (p % 2 == 0) ? p / 2 : m - 1 - (p - 1) / 2;
      (void)half;
      const double2 z = cconj(zv(sp >> 1));
      return (sp & 1) ? z.y : z.x;
    }
    const double2 z = cconj(zv(p >> 1));
    return ((p & 1) ? z.y : z.x) * ax.inv_sqrt_m;
  };
  if (ax.kind == IK_SINE) {
    const double sc = ax.dst_scale;
    for (int k = 1 + threadIdx.x; k < h; k += blockDim.x) {
      const int kc = h - k;
      const double2 Zk = zv(k);
      const double2 Zc = cconj(zv(kc));
      const double2 E = cscale(cadd(Zk, Zc), 0.5);
      const double2 D = csub(Zk, Zc);
      const double2 WO = cmul(rtw(k), make_double2(0.5 * D.y, -0.5 * D.x));
      put(k - 1, sc * (E.y + WO.y));
    }
  } else {
    const double inv_sqrt_m = ax.inv_sqrt_m;
    const int half = (m + 1) / 2;
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
      const double2 z = cconj(zv(j));
      if (ax.kind == IK_COS) {  // spec[p] -> out[2p] (p < half) or out[2(m-1-p)+1]
        const int p0 = 2 * j, p1 = 2 * j + 1;
        put(p0 < half ? 2 * p0 : 2 * (m - 1 - p0) + 1, z.x);
        put(p1 < half ? 2 * p1 : 2 * (m - 1 - p1) + 1, z.y);
      } else {
        put(2 * j, z.x * inv_sqrt_m);
        put(2 * j + 1, z.y * inv_sqrt_m);
      }
    }
  }
  if (ax.bordered && threadIdx.x == 0) {
    // out_0 = q_0 u_0 + c_a . c,  out_{n-1} = c_b . c + q_0 u_{n-1}; the dots are
    // the interior synthesis at top_i / bot_i (zero without correction)
    const double top = ax.correction ? interior_at(ax.top_i) : 0.0;
    const double bot = ax.correction ? interior_at(ax.bot_i) : 0.0;
    out[oo] = ax.q0 * u0 + top;
    out[oo + (long long)(n - 1) * eso] = bot + ax.q0 * un;
  }
  __syncthreads();  // x and the scratch are reused by the next line
#ifdef FD_PHASE_CLOCKS
  if (!big) {
    FD_CLK(c3);
    FD_CLK_ADD(1, 2, c2, c3);
  }
#endif
  }
}

// ---------------------------------------------------------------------------
// GCV grid: for every item and grid value mu_k,
//   num_k = sum_e sigma_e^2 |ghat_e|^2,  den_k = sum_e sigma_e,
//   sigma_e = 1/(r_e + mu_k)   (r_e = |d_e|^2/s_e^2; s_e = 0 contributes 0)
// (gcv_from_coeffs, regularize.hpp:63-81).  One warp owns SG items and one
// element chunk; lane k-block owns KC consecutive grid values, whose
// reciprocals share one division (Montgomery batch inversion).  All loads
// are warp-uniform broadcasts.  Partial sums land in
// partial[item][chunk][2][K] and are reduced in a fixed order afterwards.
// ---------------------------------------------------------------------------
struct GcvData {
  const void* ghat;      // item-major coefficients, `stride` per item
  int cplx;
  long long N;           // GCV elements per item
  long long stride;      // coefficients per item in ghat
  int items;
  const double* r1d;     // 1D ratio vector (length N), or null for 2D
  const int2* pair;      // optional: element e sums |ghat|^2 at pair[e].x and pair[e].y (>= 0)
  const double* wred;    // optional: precomputed weights w[item * wstride + e] (k_ranalyze wout)
  long long wstride;
  Spectral sp;           // 2D: mode 2 (separable) or 3 (full); sp.n2 = row length
  // half-spectrum layout (HalfRows): stored rows [hm_lo, hm_hi) stand for
  // themselves and their conjugate partner rows (multiplicity 2)
  int hm_lo, hm_hi;
};

// (row, column) of 2D element e; 32-bit division whenever the item has fewer
// than 2^31 elements (the 64-bit one is ~5x the instructions, and every GCV
// pass over a single large image pays it per element)
__device__ __forceinline__ void gcv_row_col(const GcvData& g, long long e, int& i, int& j) {
  if (g.N <= 0x7fffffffLL) {
    const unsigned ee = (unsigned)e, n2 = (unsigned)g.sp.n2;
    const unsigned q = ee / n2;
    i = (int)q;
    j = (int)(ee - q * n2);
  } else {
    i = (int)(e / g.sp.n2);
    j = (int)(e % g.sp.n2);
  }
}

__device__ __forceinline__ double gcv_ratio(const GcvData& g, long long e) {
  if (g.r1d) return __ldg(&g.r1d[e]);
  int i, j;
  gcv_row_col(g, e, i, j);
  if (i >= g.sp.hr_split) i += g.sp.hr_off;
  double2 d;
  double s;
  if (g.sp.mode == 2) {
    d = cmul(__ldg(&g.sp.dA[i]), __ldg(&g.sp.dB[j]));
    s = g.sp.smooth_sum ? __ldg(&g.sp.sA[i]) + __ldg(&g.sp.sB[j]) : 1.0;
  } else {
    const long long idx = (long long)i * g.sp.n2 + j;
    d = __ldg(&g.sp.dA[idx]);
    s = __ldg(&g.sp.sA[idx]);
  }
  if (s == 0.0) return INFINITY;
  return (d.x * d.x + d.y * d.y) / (s * s);
}

__device__ __forceinline__ double gcv_w1(const GcvData& g, long long idx) {
  if (g.cplx) {
    const double2 c = __ldg(reinterpret_cast<const double2*>(g.ghat) + idx);
    return c.x * c.x + c.y * c.y;
  }
  const double c = __ldg(reinterpret_cast<const double*>(g.ghat) + idx);
  return c * c;
}

// |ghat_e|^2, or the sum over a Hermitian pair (e, R-e) of a real signal's
// coefficients in a complex basis: both share r_e (d_{R-e} = conj d_e,
// s_{R-e} = s_e), so sigma^2 w summed over the pair is one term.
// multiplicity of element e in sum_e sigma_e (2 for a Hermitian pair)
__device__ __forceinline__ double gcv_mult(const GcvData& g, long long e) {
  if (g.hm_hi > g.hm_lo) {
    int r, c;
    gcv_row_col(g, e, r, c);
    return (r >= g.hm_lo && r < g.hm_hi) ? 2.0 : 1.0;
  }
  return (g.pair && __ldg(&g.pair[e]).y >= 0) ? 2.0 : 1.0;
}

// L2 bulk prefetch of one item's compact weight row (wstride doubles, a
// multiple of 32: 16-byte aligned and sized)
__device__ __forceinline__ void gcv_prefetch_row(const GcvData& g, int item) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g.wred + (long long)item * g.wstride),
               "r"((uint32_t)(g.wstride * 8))
               : "memory");
}

__device__ __forceinline__ double gcv_w(const GcvData& g, int item, long long e) {
  if (g.wred) return __ldg(&g.wred[(long long)item * g.wstride + e]);
  const long long base = (long long)item * g.stride;
  if (g.pair) {
    const int2 p = __ldg(&g.pair[e]);
    const double w = gcv_w1(g, base + p.x);
    return p.y >= 0 ? w + gcv_w1(g, base + p.y) : w;
  }
  if (g.hm_hi > g.hm_lo) return gcv_mult(g, e) * gcv_w1(g, base + e);
  return gcv_w1(g, base + e);
}


// Single items / small batches: one warp per (item, element chunk); each lane
// owns KC grid values.  Elements stream in tiles of 32 -- lane t loads and
// forms (r, w) of element e0+t (coalesced, one division per element) -- and
// are broadcast by shuffle; each lane's KC reciprocals share one reciprocal
// (batch inversion).
template <int KC>
__global__ void __launch_bounds__(256) k_gcv_grid(GcvData g, GcvGrid grid, long long chunk,
                                                  int nch, int kblock0, double* partial) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= g.items * nch) return;
  const int item = warp_global / nch, ch = warp_global % nch;
  const int K = grid.count;
  const int k0 = kblock0 + lane * KC;
  double mu[KC], num[KC], den[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    mu[k] = (k0 + k < K) ? grid.mus[k0 + k] : 1.0;
    num[k] = den[k] = 0.0;
  }
  const long long e0 = (long long)ch * chunk;
  const long long e1 = min(g.N, e0 + chunk);
  for (long long et = e0; et < e1; et += 32) {
    const long long e = et + lane;
    double rl = INFINITY, wl = 0.0, ml = 1.0;
    if (e < e1) {
      rl = gcv_ratio(g, e);
      wl = gcv_w(g, item, e);
      ml = gcv_mult(g, e);
    }
    const int cnt = (int)min(32LL, e1 - et);
    for (int t = 0; t < cnt; ++t) {
      const double r = __shfl_sync(0xffffffffu, rl, t);
      const double w = __shfl_sync(0xffffffffu, wl, t);
      const double mult = __shfl_sync(0xffffffffu, ml, t);
      if (!(r < 1e30)) {
        if (isinf(r)) continue;  // s = 0: sigma = 0
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const double s = 1.0 / (r + mu[k]);
          den[k] = fma(mult, s, den[k]);
          num[k] = fma(s * s, w, num[k]);
        }
        continue;
      }
      double xk[KC], pre[KC], sig[KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) xk[k] = r + mu[k];
      pre[0] = xk[0];
#pragma unroll
      for (int k = 1; k < KC; ++k) pre[k] = pre[k - 1] * xk[k];
      double inv = rcp_pos(pre[KC - 1]);
#pragma unroll
      for (int k = KC - 1; k >= 1; --k) {
        sig[k] = inv * pre[k - 1];
        inv *= xk[k];
      }
      sig[0] = inv;
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        den[k] = fma(mult, sig[k], den[k]);
        num[k] = fma(sig[k] * sig[k], w, num[k]);
      }
    }
  }
  double* base = partial + ((long long)item * nch + ch) * 2 * K;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    if (k0 + k < K) {
      base[k0 + k] = num[k];
      base[K + k0 + k] = den[k];
    }
  }
}

// ---------------------------------------------------------------------------
// GCV grid for batches sharing one operator, as a register-tiled fp64 GEMM
// (SURVEY H3(a)): num[b][k] = sum_e w[b][e] * sigma[e][k]^2.  Per element
// chunk of 32, the CTA generates sigma^2 for its 32*NJ grid values once in
// shared memory (one reciprocal per 4 elements by batch inversion) and every
// thread accumulates an 8-signal x NJ-mu micro-tile from shared memory, so
// sigma generation is amortised over 64 signals instead of repeated per
// signal.  den[k] = sum_e sigma is item independent and produced by the same
// pass.  Grid: x = signal blocks of 64, y = element ranges.
// ---------------------------------------------------------------------------
template <int NJ>
__global__ void __launch_bounds__(256) k_gcv_gemm(GcvData g, GcvGrid grid, int kb0,
                                                  long long echunk, int nch, double* partial) {
  constexpr int BS = 64, E = 32, BK = 32 * NJ, GP = 256 / BK;
  extern __shared__ double gsm[];
  double* Wt = gsm;              // [BS][E]
  double* Sg = gsm + BS * E;     // [E][BK]
  double* Rt = Sg + E * BK;      // [E]
  double* Mt = Rt + E;           // [E] multiplicities
  double* Dn = Mt + E;           // [256] den partials
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int item0 = blockIdx.x * BS;
  const int er = blockIdx.y;
  const long long eb = (long long)er * echunk;
  const long long ee = min(g.N, eb + echunk);
  const int K = grid.count;
  const int kk = tid % BK, part = tid / BK;
  const double mu = (kb0 + kk < K) ? grid.mus[kb0 + kk] : 1.0;
  double acc[8][NJ];
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[s][j] = 0.0;
  double den = 0.0;
  // software pipeline: the next tile's global loads are in flight while this
  // tile's sigma^2 generation and micro-GEMM run
  constexpr int NQ = BS * E / 256;
  double wreg[NQ];
  double rreg = INFINITY, mreg = 1.0;
  auto fetch = [&](long long e0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int idx = tid + 256 * q;
      const int sidx = idx >> 5, e = idx & 31;
      const int item = item0 + sidx;
      wreg[q] = (item < g.items && e0 + e < ee) ? gcv_w(g, item, e0 + e) : 0.0;
    }
    if (tid < E) {
      rreg = (e0 + tid < ee) ? gcv_ratio(g, e0 + tid) : INFINITY;
      mreg = (e0 + tid < ee) ? gcv_mult(g, e0 + tid) : 1.0;
    }
  };
  if (eb < ee) fetch(eb);
  for (long long e0 = eb; e0 < ee; e0 += E) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) Wt[tid + 256 * q] = wreg[q];
    if (tid < E) {
      Rt[tid] = rreg;
      Mt[tid] = mreg;
    }
    __syncthreads();
    if (e0 + E < ee) fetch(e0 + E);
    // sigma^2 for (element e, grid value kk); GP threads share one grid value
    constexpr int EPT = E / GP;
#pragma unroll
    for (int e4 = 0; e4 < EPT; e4 += 4) {
      const int eb4 = part * EPT + e4;
      double x[4], pre[4], sg[4];
      bool dead[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double r = Rt[eb4 + t];
        dead[t] = !(r < 1e30);  // s = 0 (inf) or absurdly large: handled below
        x[t] = dead[t] ? 1.0 : r + mu;
      }
      pre[0] = x[0];
#pragma unroll
      for (int t = 1; t < 4; ++t) pre[t] = pre[t - 1] * x[t];
      double inv = rcp_pos(pre[3]);
#pragma unroll
      for (int t = 3; t >= 1; --t) {
        sg[t] = inv * pre[t - 1];
        inv *= x[t];
      }
      sg[0] = inv;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (dead[t]) {
          const double r = Rt[eb4 + t];
          sg[t] = isinf(r) ? 0.0 : 1.0 / (r + mu);
        }
        den = fma(Mt[eb4 + t], sg[t], den);
        Sg[(eb4 + t) * BK + kk] = sg[t] * sg[t];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int e = 0; e < E; ++e) {
      double a[8], b[NJ];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) a[s2] = Wt[(ty * 8 + s2) * E + e];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = Sg[e * BK + tx + 32 * j];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[s2][j] = fma(a[s2], b[j], acc[s2][j]);
    }
    __syncthreads();
  }
  Dn[tid] = den;
  __syncthreads();
  if (tid < BK) {
    double dsum = 0.0;
    for (int p = 0; p < GP; ++p) dsum += Dn[p * BK + tid];
    Dn[tid] = dsum;
  }
  __syncthreads();
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2) {
    const int item = item0 + ty * 8 + s2;
    if (item >= g.items) continue;
    double* base = partial + ((long long)item * nch + er) * 2 * K;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = kb0 + tx + 32 * j;
      if (k < K) {
        base[k] = acc[s2][j];
        base[K + k] = Dn[tx + 32 * j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// GCV grid, GEMM form with a precomputed sigma^2 table (batches sharing one
// operator, 1D).  sigma depends only on (operator, smoother, grid), so
//   S2[e][k] = sigma_e(mu_k)^2  (N x Kp, L2-resident),  den[k] = sum_e mult_e sigma_e(mu_k)
// are formed once per call; the GEMM num = W S2 then streams 32-element tiles
// of the weights W (|ghat|^2 written by k_ranalyze, pairs pre-summed) and of S2
// into shared memory with cp.async.bulk + mbarrier, double buffered, so the
// copy engine fills stage c+1 while the DFMA micro-tiles consume stage c.
// ---------------------------------------------------------------------------
__global__ void k_gcv_s2(GcvData g, GcvGrid grid, long long Np, int Kp, double* S2) {
  const long long tot = Np * Kp;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / Kp;
    const int kk = (int)(t % Kp);
    double v = 0.0;
    if (e < g.N && kk < grid.count) {
      const double r = gcv_ratio(g, e);
      if (!isinf(r)) {
        const double s = 1.0 / (r + grid.mus[kk]);
        v = s * s;
      }
    }
    S2[t] = v;
  }
}

// grid (K, nsplit): CTA (k, y) sums the elements of split y; nsplit == 1 writes
// den[k], otherwise out[k * nsplit + y] (reduced in split order afterwards)
__global__ void __launch_bounds__(256) k_gcv_den(GcvData g, GcvGrid grid, double* out) {
  __shared__ double red[32];
  const int kk = blockIdx.x;
  const double mu = grid.mus[kk];
  const long long chunk = (g.N + gridDim.y - 1) / gridDim.y;
  const long long e0 = (long long)blockIdx.y * chunk, e1 = min(g.N, e0 + chunk);
  double acc[1] = {0.0};
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const double r = gcv_ratio(g, e);
    if (!isinf(r)) acc[0] = fma(gcv_mult(g, e), 1.0 / (r + mu), acc[0]);
  }
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) out[(long long)kk * gridDim.y + blockIdx.y] = acc[0];
}

// ---- interval screen of the grid for single large items ----
// The elements are binned by r = |d|^2/s^2 on 64 bins per octave (the bin of r
// is its exponent and top 6 mantissa bits, so bin b holds r in
// [r_lo(b), r_hi(b)) with r_hi/r_lo <= 1 + 2^-6; r = 0 has its own exact bin).
// From the per-bin sums of the weights and multiplicities every grid point gets
// an interval [G_lo, G_hi] that contains G (sigma is monotone in r); only grid
// points with G_lo <= min_j G_hi can hold the first minimum or a 1e-12 tie, and
// only those are evaluated exactly (fd_capi.cu gcv_select_dev).
constexpr int kHistShift = 46;  // 52 - 6 mantissa bits kept

__device__ __forceinline__ long long hist_key(double r) {
  return (long long)(__double_as_longlong(r) >> kHistShift);
}

// min over positive finite r and max over finite r: per-CTA partials
// mm[2 cta], mm[2 cta + 1] (min / max are order-independent)
__global__ void __launch_bounds__(256) k_gcv_rrange(GcvData g, double* mm) {
  __shared__ double red[64];
  double lo = INFINITY, hi = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.N;
       e += (long long)gridDim.x * blockDim.x) {
    const double r = gcv_ratio(g, e);
    if (isinf(r)) continue;
    if (r > 0.0) lo = fmin(lo, r);
    hi = fmax(hi, r);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = lo;
    red[32 + (threadIdx.x >> 5)] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = fmin(lo, red[w]);
      hi = fmax(hi, red[32 + w]);
    }
    lo = fmin(lo, red[0]);
    hi = fmax(hi, red[32]);
    mm[2 * blockIdx.x] = lo;
    mm[2 * blockIdx.x + 1] = hi;
  }
}


// per-CTA histogram of (sum W, sum mult) over bins [0, nb) (keys base + b) and
// the zero bin nb; partial[cta][2 (nb + 1)]
__global__ void __launch_bounds__(512) k_gcv_hist(GcvData g, long long base, int nb,
                                                  double* partial) {
  extern __shared__ double hist[];
  const int nw = 2 * (nb + 1);
  for (int i = threadIdx.x; i < nw; i += blockDim.x) hist[i] = 0.0;
  __syncthreads();
  // Neighbouring elements have nearly equal r at low frequencies: when a whole
  // warp adds into one bin its 64 shared-memory atomics serialise, so that case
  // is reduced by shuffles into one pair of atomics.  (Walking the distinct bins
  // of every warp instead measured 3.7x slower: at high frequencies the 32
  // lanes hit ~32 bins.)
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); e0 < g.N;
       e0 += stride) {
    const long long e = e0 + lane;
    double w = 0.0, mlt = 0.0;
    int b = -1;  // -1: nothing to add (past the end, or s_e = 0)
    if (e < g.N) {
      const double r = gcv_ratio(g, e);
      if (!isinf(r)) {
        b = r > 0.0 ? (int)(hist_key(r) - base) : nb;
        w = gcv_w(g, 0, e);
        mlt = gcv_mult(g, e);
      }
    }
    const int b0 = __shfl_sync(full, b, 0);
    if (__all_sync(full, b == b0)) {
      if (b0 < 0) continue;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w += __shfl_xor_sync(full, w, o);
        mlt += __shfl_xor_sync(full, mlt, o);
      }
      if (lane == 0) {
        atomicAdd(&hist[2 * b0], w);
        atomicAdd(&hist[2 * b0 + 1], mlt);
      }
    } else if (b >= 0) {
      atomicAdd(&hist[2 * b], w);
      atomicAdd(&hist[2 * b + 1], mlt);
    }
  }
  __syncthreads();
  double* out = partial + (long long)blockIdx.x * nw;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) out[i] = hist[i];
}

// bounds[k] = (G_lo, G_hi) from the reduced histogram; one CTA per grid point
// `widen` is the relative rounding allowance of the bounds: every histogram
// sum is a sum of positive terms in no fixed order (shared atomics, then the
// cross-CTA reduction), so its relative error is below (terms)*2^-53; G is a
// ratio num/den^2 of such sums, and the exact pass that later decides among the
// candidates rounds the same way.  The caller passes
// 4*(N + bins + CTAs + 8)*2^-53 + 1e-12.
__global__ void __launch_bounds__(256) k_gcv_bounds(const double* __restrict__ hist,
                                                    long long base, int nb, GcvGrid grid,
                                                    double widen, double* bounds) {
  __shared__ double red[32 * 4];
  const int k = blockIdx.x;
  const double mu = grid.mus[k];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // num_hi, num_lo, den_hi, den_lo
  for (int b = threadIdx.x; b <= nb; b += blockDim.x) {
    const double W = hist[2 * b], cnt = hist[2 * b + 1];
    if (cnt == 0.0 && W == 0.0) continue;
    double rlo = 0.0, rhi = 0.0;
    if (b < nb) {
      rlo = __longlong_as_double((base + b) << kHistShift);
      rhi = __longlong_as_double((base + b + 1) << kHistShift);
    }
    const double shi = 1.0 / (rlo + mu), slo = 1.0 / (rhi + mu);
    acc[0] = fma(W, shi * shi, acc[0]);
    acc[1] = fma(W, slo * slo, acc[1]);
    acc[2] = fma(cnt, shi, acc[2]);
    acc[3] = fma(cnt, slo, acc[3]);
  }
  block_sum<4>(acc, red);
  if (threadIdx.x == 0) {
    // widened for the rounding of these sums and of the exact pass
    bounds[2 * k] = acc[1] / (acc[2] * acc[2]) * (1.0 - widen);
    bounds[2 * k + 1] = acc[0] / (acc[3] * acc[3]) * (1.0 + widen);
  }
}

// ---- tensor-core screening of the grid (fd_tc.cuh) and exact candidates ----
// rmin = min over elements of the finite ratios r_e (one CTA)
// r table of a batch sharing one 2D operator (gcv_ratio for every element)
// compact GCV weights of a batch sharing one 2D operator: W[item][e] =
// mult_e |ghat_e|^2 (the half-spectrum pair rows counted twice), rows padded
// with zeros to wstride -- the batched grid then runs as the W . S2 product
// (k_gcv_gemm2) and every later pass streams 8 B per element instead of the
// 16 B complex coefficient plus the index arithmetic of the 2D ratio
__global__ void __launch_bounds__(256) k_gcv_wbuild(GcvData g, long long wstride, double* W) {
  const long long tot = (long long)g.items * wstride;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long item = t / wstride, e = t - item * wstride;
    W[t] = e < g.N ? gcv_w(g, (int)item, e) : 0.0;
  }
}

__global__ void k_gcv_rtab(GcvData g, double* r) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.N;
       e += (long long)gridDim.x * blockDim.x)
    r[e] = gcv_ratio(g, e);
}

__global__ void __launch_bounds__(256) k_gcv_rmin(GcvData g, double* rmin) {
  __shared__ double red[32];
  double v = INFINITY;
  for (long long e = threadIdx.x; e < g.N; e += blockDim.x) v = fmin(v, gcv_ratio(g, e));
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, red[w]);
    *rmin = m;
  }
}

// S32[k][e] = ((rmin + mu_k) / (r_e + mu_k))^2 = S2[e][k] / S2max_k  (<= 1),
// zero for padding rows k >= K and elements e >= N; written as the TF32 split
// (hi, lo) in screen tiles of BN rows (tc_tile_index)
__global__ void k_gcv_s32(GcvData g, GcvGrid grid, int BN, long long Ep,
                          const double* __restrict__ rmin, float* S32h, float* S32l) {
  const long long tot = (long long)BN * Ep;
  const double r0 = *rmin;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t / Ep);
    const long long e = t % Ep;
    double v = 0.0;
    if (k < grid.count && e < g.N) {
      const double r = gcv_ratio(g, e);
      if (!isinf(r)) {
        const double q = (r0 + grid.mus[k]) / (r + grid.mus[k]);
        v = q * q;
      }
    }
    float hi, lo;
    tf32_split(v, hi, lo);
    const long long d = tc_tile_index(k, e, BN, Ep >> 5);
    S32h[d] = hi;
    S32l[d] = lo;
  }
}

// gscale_k = S2max_k / den_k^2 (G~ = num~ gscale); a zero den is the
// degenerate case (regularize.hpp:78-79)
__global__ void k_gcv_gscale(GcvGrid grid, const double* __restrict__ den,
                             const double* __restrict__ rmin, double* gscale, int* status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= grid.count) return;
  const double d = den[k];
  if (d == 0.0) {
    atomicExch(status, 3);
    gscale[k] = NAN;
    return;
  }
  const double s = 1.0 / (*rmin + grid.mus[k]);
  gscale[k] = (s * s) / (d * d);
}

// Stream the elements [e0, e1) of one item through f(r_e, W_e): lane-strided,
// U elements per lane and step with all their loads issued before any use
// (the weights stream from HBM; one load in flight per warp is latency-bound).
template <int U, class F>
__device__ __forceinline__ void gcv_stream(const GcvData& g, int item, long long e0, long long e1,
                                           int lane, F&& f) {
  for (long long e = e0 + lane; e < e1; e += 32 * U) {
    double r[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long x = e + 32 * u;
      r[u] = x < e1 ? gcv_ratio(g, x) : INFINITY;
      w[u] = x < e1 ? gcv_w(g, item, x) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) f(r[u], w[u]);
  }
}

// num at CH grid values (mu[i], i < nv; the rest padding) for one item:
// warp-strided elements, the CH reciprocals of each element from one
// division (batch inversion), shuffle-tree sum; lane i < nv returns num_i.
template <int CH>
__device__ __forceinline__ double exact_num(const GcvData& g, int item, const double (&mu)[CH],
                                            int lane) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = 0.0;
  auto one = [&](double r, double w) {
    if (isinf(r)) return;
    double a[CH], pre[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = r + mu[i];
    pre[0] = a[0];
#pragma unroll
    for (int i = 1; i < CH; ++i) pre[i] = pre[i - 1] * a[i];
    if (pre[CH - 1] < 1e300 && pre[CH - 1] > 1e-300) {
      double inv = rcp_pos(pre[CH - 1]);
#pragma unroll
      for (int i = CH - 1; i >= 1; --i) {
        const double s = inv * pre[i - 1];
        inv *= a[i];
        acc[i] = fma(w, s * s, acc[i]);
      }
      acc[0] = fma(w, inv * inv, acc[0]);
    } else {
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const double s = 1.0 / a[i];
        acc[i] = fma(w, s * s, acc[i]);
      }
    }
  };
  gcv_stream<4>(g, item, 0, g.N, lane, one);
#pragma unroll
  for (int i = 0; i < CH; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  double v = acc[0];
#pragma unroll
  for (int i = 1; i < CH; ++i)
    if (lane == i) v = acc[i];
  return v;
}

// exact num / den of one item at CH explicit grid values (lanes over the
// elements of a chunk, the CH reciprocals of an element by batch inversion):
// partial[chunk][2 CH] = (num_0..num_{CH-1}, den_0..den_{CH-1}); padding mu = 1
template <int CH>
__global__ void __launch_bounds__(256) k_gcv_cand(GcvData g, const double* __restrict__ mus,
                                                  int nc, long long chunk, int nch,
                                                  double* partial) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nch) return;
  double mu[CH], num[CH], den[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    mu[i] = i < nc ? mus[i] : 1.0;
    num[i] = den[i] = 0.0;
  }
  const long long e0 = (long long)warp * chunk, e1 = min(g.N, e0 + chunk);
  gcv_stream<4>(g, 0, e0, e1, lane, [&](double r, double w) {
    if (isinf(r)) return;
    double a[CH], pre[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = r + mu[i];
    pre[0] = a[0];
#pragma unroll
    for (int i = 1; i < CH; ++i) pre[i] = pre[i - 1] * a[i];
    double s[CH];
    if (pre[CH - 1] < 1e300 && pre[CH - 1] > 1e-300) {
      double inv = rcp_pos(pre[CH - 1]);
#pragma unroll
      for (int i = CH - 1; i >= 1; --i) {
        s[i] = inv * pre[i - 1];
        inv *= a[i];
      }
      s[0] = inv;
    } else {
#pragma unroll
      for (int i = 0; i < CH; ++i) s[i] = 1.0 / a[i];
    }
    const double mult = 1.0;  // 2D / unpaired elements (interval_screen's items)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      num[i] = fma(w, s[i] * s[i], num[i]);
      den[i] = fma(mult, s[i], den[i]);
    }
  });
#pragma unroll
  for (int i = 0; i < CH; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], o);
      den[i] += __shfl_xor_sync(0xffffffffu, den[i], o);
    }
  if (lane == 0) {
    double* out = partial + (long long)warp * 2 * CH;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      out[i] = num[i];
      out[CH + i] = den[i];
    }
  }
}

// Exact G(mu_k) = num_k / den_k^2 at the screened candidates of each item
// (every grid point when the item is flagged) and gcv_pick over them -- the
// other grid points are above the minimum by more than the screen's error, so
// the first minimum, the 1e-12 ties and the bracket are those of the full
// grid.  One warp per item; candidates in groups of up to 8 (exact_num).
// Fixed lane order + shuffle tree: deterministic.
__global__ void __launch_bounds__(256, 4) k_gcv_exact(GcvData g, GcvGrid grid,
                                                   const uint32_t* __restrict__ mask,
                                                   const int* __restrict__ flag,
                                                   const double* __restrict__ den, double* mu_out,
                                                   int* best_k, double* center, int* need,
                                                   double* bestG, int* status) {
  __shared__ int lists[8][256];
  __shared__ double vals[8][256];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= g.items) return;
  const int K = grid.count;
  int* list = lists[wib];
  double* val = vals[wib];
  // the item's weight row into L2 while the candidate list is built (the
  // warp then streams it at L2 latency)
  if (lane == 0 && g.wred) gcv_prefetch_row(g, item);
  const bool all = flag[item] != 0;
  // candidate list (ascending k) in shared memory
  int nc = 0;
  for (int w0 = 0; w0 < 8; ++w0) {
    const uint32_t bits = all ? 0xffffffffu : __ldg(&mask[(long long)item * 8 + w0]);
    const int k = w0 * 32 + lane;
    const bool on = k < K && ((bits >> lane) & 1u);
    const uint32_t ball = __ballot_sync(0xffffffffu, on);
    if (on) list[nc + __popc(ball & ((1u << lane) - 1u))] = k;
    nc += __popc(ball);
  }
  __syncwarp();
  for (int c0 = 0; c0 < nc;) {
    const int nv = min(8, nc - c0);
    double v;
    if (nv <= 4) {
      double mu[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mu[i] = i < nv ? grid.mus[list[c0 + i]] : 1.0;
      v = exact_num<4>(g, item, mu, lane);
    } else {
      double mu[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mu[i] = i < nv ? grid.mus[list[c0 + i]] : 1.0;
      v = exact_num<8>(g, item, mu, lane);
    }
    if (lane < nv) {
      const double d = den[list[c0 + lane]];
      val[c0 + lane] = d == 0.0 ? NAN : v / (d * d);
    }
    c0 += nv;
  }
  __syncwarp();
  if (lane == 0) {  // gcv_pick (fd_gcv_core.h) restricted to the candidates
    int bi = 0;
    double best = val[0];
    for (int i = 1; i < nc; ++i)
      if (val[i] < best) {
        best = val[i];
        bi = i;
      }
    int ntied = 0;
    double mean_log = 0.0;
    for (int i = 0; i < nc; ++i) {
      const bool tie = best == 0.0 ? val[i] == 0.0 : val[i] <= best + 1e-12 * fabs(best);
      if (tie) {
        ++ntied;
        mean_log += grid.logmus[list[i]];
      }
    }
    if (isnan(best)) atomicExch(status, 3);
    const int k = list[bi];
    best_k[item] = k;
    bestG[item] = best;
    if (ntied > 1) {
      mu_out[item] = exp(mean_log / (double)ntied);
      need[item] = 0;
      center[item] = 0.0;
    } else {
      need[item] = 1;
      center[item] = sqrt(grid.mus[k > 0 ? k - 1 : 0] * grid.mus[k + 1 < K ? k + 1 : K - 1]);
      mu_out[item] = grid.mus[k];
    }
  }
}

template <int NJ>
__global__ void __launch_bounds__(256) k_gcv_gemm2(const double* __restrict__ W, long long Np,
                                                   int items, const double* __restrict__ S2,
                                                   int Kp, int K, int kb0, long long echunk,
                                                   int nch, const double* __restrict__ den,
                                                   double* partial) {
  constexpr int BS = 64, E = 32, BK = 32 * NJ;
  constexpr int STAGE = BS * E + E * BK;  // doubles per stage
  extern __shared__ __align__(128) double gsm2[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(gsm2 + 2 * STAGE);
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int item0 = blockIdx.x * BS;
  const int rows = min(BS, items - item0);
  const long long eb = (long long)blockIdx.y * echunk;
  const long long ee = min(Np, eb + echunk);
  const int nck = (int)((ee - eb + E - 1) / E);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = (uint32_t)(rows * E + E * BK) * 8u;
  auto issue = [&](int c) {  // warp 0 fills stage c & 1 with chunk c
    double* st = gsm2 + (c & 1) * STAGE;
    const long long e0 = eb + (long long)c * E;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tx == 0) mbar_expect_tx(&bars[c & 1], bytes);
    __syncwarp();
    for (int s = tx; s < rows; s += 32)
      bulk_g2s(st + s * E, W + (long long)(item0 + s) * Np + e0, E * 8, &bars[c & 1]);
    if (BK == Kp) {
      if (tx == 0) bulk_g2s(st + BS * E, S2 + e0 * Kp, E * BK * 8, &bars[c & 1]);
    } else {
      bulk_g2s(st + BS * E + tx * BK, S2 + (e0 + tx) * Kp + kb0, BK * 8, &bars[c & 1]);
    }
  };
  double acc[8][NJ];
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[s][j] = 0.0;
  if (ty == 0 && nck > 0) issue(0);
  for (int c = 0; c < nck; ++c) {
    if (ty == 0 && c + 1 < nck) issue(c + 1);
    mbar_wait(&bars[c & 1], (c >> 1) & 1);
    const double* Wt = gsm2 + (c & 1) * STAGE;
    const double* St = Wt + BS * E;
#pragma unroll 4
    for (int e = 0; e < E; ++e) {
      double a[8], b[NJ];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2) a[s2] = Wt[(ty * 8 + s2) * E + e];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = St[e * BK + tx + 32 * j];
#pragma unroll
      for (int s2 = 0; s2 < 8; ++s2)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[s2][j] = fma(a[s2], b[j], acc[s2][j]);
    }
    __syncthreads();  // stage (c & 1) is refilled by iteration c + 1's issue(c + 2)
  }
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2) {
    const int item = item0 + ty * 8 + s2;
    if (item >= items) continue;
    double* base = partial + ((long long)item * nch + blockIdx.y) * 2 * K;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int kk = kb0 + tx + 32 * j;
      if (kk < K) {
        base[kk] = acc[s2][j];
        base[K + kk] = blockIdx.y == 0 ? den[kk] : 0.0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// GCV selection (gcv_minimize, regularize.cpp:144-214), one thread per item:
// reduce the grid partials in chunk order, G_k = num/den^2, first minimum,
// 1e-12 tie test, and the golden-section refinement evaluated from Taylor
// moments about mu_c = sqrt(lo*hi):
//   den(mu) = sum_j (-d)^j B_j,  num(mu) = sum_j (j+1)(-d)^j A_j,  d = mu-mu_c,
//   B_j = sum_e t_e^{j+1}, A_j = sum_e w_e t_e^{j+2}, t_e = 1/(r_e + mu_c).
// Every point the golden section visits lies in [lo, hi], where the series
// ratio |d|/(r+mu_c) <= sqrt(hi/lo)-1, so J terms give ~1e-17 relative error.
// ---------------------------------------------------------------------------
__global__ void k_gcv_reduce_grid(const double* __restrict__ partial, int items, int nchunks,
                                  int K, double* G, int* status) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)items * K) return;
  const int item = (int)(t / K), k = (int)(t % K);
  double num = 0.0, den = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const double* base = partial + ((long long)item * nchunks + c) * 2 * K;
    num += base[k];
    den += base[K + k];
  }
  if (den == 0.0) {
    atomicExch(status, 3);  // DegenerateError (regularize.hpp:78-79)
    G[t] = NAN;
    return;
  }
  G[t] = num / (den * den);
}

// out[item][w] = sum_c partial[item][c][w], c = 0..nch-1, in a fixed order:
// a CTA owns (item, 32 consecutive w); lane = w, warp = chunk residue mod 8,
// then the 8 warp partials are added in warp order.  Coalesced over w.
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ partial,
                                                         int nch, int width, double* out) {
  __shared__ double sm[8][33];
  const int item = blockIdx.x;
  const int w0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, cg = threadIdx.x >> 5;
  const int w = w0 + lane;
  double acc = 0.0;
  if (w < width)
    for (int c = cg; c < nch; c += 8)
      acc += partial[((long long)item * nch + c) * width + w];
  sm[cg][lane] = acc;
  __syncthreads();
  if (cg == 0 && w < width) {
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) s += sm[g][lane];
    out[(long long)item * width + w] = s;
  }
}

__global__ void k_gcv_pick(const double* __restrict__ G, int items, GcvGrid grid, double* mu_out,
                           int* best_k, double* center, int* need_refine, double* bestG) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= items) return;
  const GcvPick pk = gcv_pick(grid.mus, grid.logmus, G + (long long)item * grid.count, grid.count);
  best_k[item] = pk.best_k;
  bestG[item] = G[(long long)item * grid.count + pk.best_k];
  if (pk.tied) {
    mu_out[item] = pk.mu_tie;
    need_refine[item] = 0;
    center[item] = 0.0;
  } else {
    need_refine[item] = 1;
    center[item] = sqrt(pk.lo * pk.hi);
    mu_out[item] = grid.mus[pk.best_k];
  }
}

// Taylor moments of the golden-section refinement around the item's bracket
// center mc = sqrt(mu_{k-1} mu_{k+1}) (k = best_k, clamped):
//   mc^2 num(mu) = sum_j (j+1) A_j x^j,  A_j = sum_e W_e t_e^{j+2},
//   mc den(mu)   = sum_j B_j x^j,        B_j = sum_e mult_e t_e^{j+1},
// t_e = mc/(r_e + mc) in (0, 1], x = (mc - mu)/mc: the powers of mc cancel in
// G = num/den^2, and no moment can overflow (unscaled, t^(J+2) = mc^-(J+2)
// passes 1e308 for mc below ~1e-8 at J = 36).  B depends on the item only through k, so it is one
// table over the K grid points (k_gcv_bmom); the per-item pass accumulates A
// with two operations per term.
// WITH_B: also accumulate B per item (few large items: a B table over all K
// grid points would cost K passes over the elements); partial holds [A | B].
template <int J, bool WITH_B>
__global__ void __launch_bounds__(256, WITH_B ? 2 : 3) k_gcv_moments(GcvData g, const double* __restrict__ center,
                                                     const int* __restrict__ need, long long chunk,
                                                     int nchunks, double* partial) {
  // one warp per (item, chunk); lanes stride over elements
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= g.items * nchunks) return;
  const int item = warp_global / nchunks, ch = warp_global % nchunks;
  if (!need[item]) return;
  if (lane == 0 && g.wred && nchunks == 1) gcv_prefetch_row(g, item);
  const double mc = center[item];
  constexpr int NB = WITH_B ? J : 1;
  double A[J], B[NB];
#pragma unroll
  for (int j = 0; j < J; ++j) A[j] = 0.0;
#pragma unroll
  for (int j = 0; j < NB; ++j) B[j] = 0.0;
  const long long e0 = (long long)ch * chunk;
  const long long e1 = min(g.N, e0 + chunk);
  if (WITH_B) {
    for (long long e = e0 + lane; e < e1; e += 32) {
      const double r = gcv_ratio(g, e);
      if (isinf(r)) continue;
      const double w = gcv_w(g, item, e);
      const double t = mc * rcp_pos(r + mc);
      double pa = (w * t) * t, pb = gcv_mult(g, e) * t;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        A[j] += pa;
        pa *= t;
        if (WITH_B) {
          B[j % NB] += pb;
          pb *= t;
        }
      }
    }
  } else {
    gcv_stream<4>(g, item, e0, e1, lane, [&](double r, double w) {
      if (isinf(r)) return;
      const double t = mc * rcp_pos(r + mc);
      // four interleaved power chains (step t^4): dependency depth J/4, not J
      const double t2 = t * t, t4 = t2 * t2;
      double p[4];
      p[0] = w * t2;
      p[1] = p[0] * t;
      p[2] = p[0] * t2;
      p[3] = p[1] * t2;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        A[j] += p[j & 3];
        p[j & 3] *= t4;
      }
    });
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) A[j] += __shfl_xor_sync(0xffffffffu, A[j], o);
    if (WITH_B)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) B[j % NB] += __shfl_xor_sync(0xffffffffu, B[j % NB], o);
  }
  if (lane == 0) {
    double* base = partial + ((long long)item * nchunks + ch) * (WITH_B ? 2 : 1) * J;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      base[j] = A[j];
      if (WITH_B) base[J + j] = B[j % NB];
    }
  }
}

// center of grid point k's golden bracket (k_gcv_pick uses the same expression)
__device__ __forceinline__ double bracket_center(const GcvGrid& grid, int k) {
  const int K = grid.count;
  return sqrt(grid.mus[k > 0 ? k - 1 : 0] * grid.mus[k + 1 < K ? k + 1 : K - 1]);
}

// Btab[k][j] = sum_e mult_e t_e^{j+1}, t_e = 1/(r_e + center_k); one CTA per k
template <int J>
__global__ void __launch_bounds__(256) k_gcv_bmom(GcvData g, GcvGrid grid, double* Btab) {
  __shared__ double red[32 * J];
  const int k = blockIdx.x;
  const double mc = bracket_center(grid, k);
  double B[J];
#pragma unroll
  for (int j = 0; j < J; ++j) B[j] = 0.0;
  for (long long e = threadIdx.x; e < g.N; e += blockDim.x) {
    const double r = gcv_ratio(g, e);
    if (isinf(r)) continue;
    const double t = mc * rcp_pos(r + mc);
    double p = gcv_mult(g, e) * t;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      B[j] += p;
      p *= t;
    }
  }
  block_sum<J>(B, red);
  if (threadIdx.x < J) {
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (threadIdx.x == j) Btab[(long long)k * J + j] = B[j];
  }
}

struct MomentG {
  const double* A;
  const double* B;
  int J;
  double mc;
  __device__ double operator()(double mu) const {
    const double d = -(mu - mc) / mc;
    double num = 0.0, den = 0.0;
    for (int j = J - 1; j >= 0; --j) {
      num = fma(num, d, (double)(j + 1) * A[j]);
      den = fma(den, d, B[j]);
    }
    return num / (den * den);
  }
};

__global__ void k_gcv_golden(const double* __restrict__ partial, int items, int nchunks, int J,
                             const double* __restrict__ Btab, const double* __restrict__ bestG,
                             GcvGrid grid, const int* __restrict__ best_k,
                             const double* __restrict__ center, const int* __restrict__ need,
                             double* mu_out) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= items || !need[item]) return;
  double A[64], B[64];
  const int k = best_k[item];
  const int w = Btab ? J : 2 * J;  // per-item B follows A in partial when there is no table
  for (int j = 0; j < J; ++j) {
    A[j] = 0.0;
    B[j] = Btab ? Btab[(long long)k * J + j] : 0.0;
  }
  for (int c = 0; c < nchunks; ++c) {
    const double* base = partial + ((long long)item * nchunks + c) * w;
    for (int j = 0; j < J; ++j) A[j] += base[j];
    if (!Btab)
      for (int j = 0; j < J; ++j) B[j] += base[J + j];
  }
  MomentG f{A, B, J, center[item]};
  const double best = bestG[item];
  mu_out[item] = gcv_golden(grid.mus, grid.count, k, best, f);
}

// direct G(mu_item) for every item (gcv_value, regularize.cpp:119-142)
__global__ void __launch_bounds__(256) k_gcv_direct(GcvData g, const double* __restrict__ mu_item,
                                                    long long chunk, int nchunks,
                                                    double* partial) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= g.items * nchunks) return;
  const int item = warp_global / nchunks, ch = warp_global % nchunks;
  const double mu = mu_item[item];
  double num = 0.0, den = 0.0;
  const long long e0 = (long long)ch * chunk;
  const long long e1 = min(g.N, e0 + chunk);
  for (long long e = e0 + lane; e < e1; e += 32) {
    const double r = gcv_ratio(g, e);
    if (isinf(r)) continue;
    const double sig = 1.0 / (r + mu);
    den = fma(gcv_mult(g, e), sig, den);
    num = fma(sig * sig, gcv_w(g, item, e), num);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if (lane == 0) {
    double* base = partial + ((long long)item * nchunks + ch) * 2;
    base[0] = num;
    base[1] = den;
  }
}

__global__ void k_gcv_direct_reduce(const double* __restrict__ partial, int items, int nchunks,
                                    double* G, int* status) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= items) return;
  double num = 0.0, den = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    num += partial[((long long)item * nchunks + c) * 2];
    den += partial[((long long)item * nchunks + c) * 2 + 1];
  }
  if (den == 0.0) {
    atomicExch(status, 3);
    G[item] = NAN;
    return;
  }
  G[item] = num / (den * den);
}

// per-item residue: sqrt of the summed per-line Im^2 (operators.cpp:222-229)
// rre (regularize.cpp:249-260) partial sums of `items` restorations against
// one truth: partial[item][chunk] = (sum t^2, sum (t - f)^2) over the chunk
__global__ void __launch_bounds__(256) k_rre_partials(const double* __restrict__ f,
                                                      const double* __restrict__ t, long long N,
                                                      long long chunk, double* partial) {
  __shared__ double red[64];
  const int b = blockIdx.x, ch = blockIdx.y;
  const long long e0 = (long long)ch * chunk, e1 = min(N, e0 + chunk);
  double acc[2] = {0.0, 0.0};
  const double* fb = f + (long long)b * N;
  for (long long i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
    const double tv = __ldg(&t[i]);
    const double e = tv - __ldg(&fb[i]);
    acc[0] = fma(tv, tv, acc[0]);
    acc[1] = fma(e, e, acc[1]);
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    double* o = partial + ((long long)b * gridDim.y + ch) * 2;
    o[0] = acc[0];
    o[1] = acc[1];
  }
}

// rre[item] = sqrt(en / tn) from the reduced sums; NaN flags a zero truth
__global__ void k_rre_final(const double* __restrict__ sums, int items, double* rre) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= items) return;
  const double tn = sums[2 * b], en = sums[2 * b + 1];
  rre[b] = tn == 0.0 ? NAN : sqrt(en / tn);
}

__global__ void k_resid_reduce(const double* __restrict__ r2, int items, int per_item,
                               double* out) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= items) return;
  double acc = 0.0;
  for (int l = 0; l < per_item; ++l) acc += r2[(long long)item * per_item + l];
  out[item] = sqrt(acc);
}

// elementwise c <- c * d (complex or real), used by the 2D matvec between passes
__global__ void k_scale_full(void* c, int cplx, long long N, int items, Spectral sp) {
  const long long tot = N * items;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t % N;
    const int i = (int)(e / sp.n2), j = (int)(e % sp.n2);
    double2 d;
    if (sp.mode == 2)
      d = cmul(sp.dA[i], sp.dB[j]);
    else
      d = sp.dA[e];
    if (cplx) {
      double2* p = reinterpret_cast<double2*>(c) + t;
      *p = cmul(*p, d);
    } else {
      double* p = reinterpret_cast<double*>(c) + t;
      *p = *p * d.x;
    }
  }
}

}  // namespace fdb
