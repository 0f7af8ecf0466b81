// Block-level fp64 FFT engine for sm_100a.
//
// One CTA owns one length-M complex buffer in shared memory (M = 2^k, padded
// one slot per 16 so strided passes are bank-conflict free) and runs
//   DIF (natural -> digit-reversed)  then  DIT (digit-reversed -> natural).
// Each pass fuses up to four radix-2 stages in registers (radix-16 butterflies,
// 16 complex values per thread item), so an M = 8192 transform touches shared
// memory 4 times instead of 13.  Twiddles come from two small shared-memory
// tables (TwSm) plus compile-time radix-16 constants.
//
// Arbitrary lengths L (the interior lengths n-2 = 2*7*73, 2*23*89, 2*8191 of
// the BASELINE sizes are never powers of two) use Bluestein:
//   X_k = c_k * sum_j (x_j c_j) conj(c_{k-j}),   c_j = e^{-i pi j^2/L},
// evaluated as DIF -> pointwise multiply by the precomputed DIF(b)/M (already
// in digit-reversed order, so no permutation is ever materialised) -> DIT.
// The chirp pre/post multiplies are fused into the callers' load/store loops.
#pragma once

#include <cuda_runtime.h>

#include "fd_internal.h"

namespace fdb {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// padded shared-memory slot of logical index i
__host__ __device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }

// d * e^{-2 pi i k/16} for a compile-time k in [0, 8)
__device__ __forceinline__ double2 mul_w16(double2 d, int k) {
  constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173;
  constexpr double H = 0.70710678118654752440;
  switch (k) {
    case 0: return d;
    case 1: return cmul(d, make_double2(C1, -S1));
    case 2: return make_double2(H * (d.x + d.y), H * (d.y - d.x));
    case 3: return cmul(d, make_double2(S1, -C1));
    case 4: return make_double2(d.y, -d.x);
    case 5: return cmul(d, make_double2(-S1, -C1));
    case 6: return make_double2(H * (d.y - d.x), -H * (d.x + d.y));
    default: return cmul(d, make_double2(-C1, -S1));
  }
}
// d * e^{+2 pi i k/16}
__device__ __forceinline__ double2 mul_w16c(double2 d, int k) {
  return cconj(mul_w16(cconj(d), k));
}

// Twiddles e^{-2 pi i j/M} from two small shared-memory tables,
// W^j = hi[j >> lob] * lo[j & (2^lob - 1)]: exact table entries, one complex
// multiply (<= 2 ulp), and no L2 round trip inside the barrier-separated passes.
struct TwSm {
  const double2* lo;
  const double2* hi;
  int lob;
  __device__ __forceinline__ double2 operator()(int j) const {
    return cmul(hi[j >> lob], lo[j & ((1 << lob) - 1)]);
  }
};

constexpr int kTwSlots = 256;  // lo + hi entries of the on-chip sizes (M <= 2^14: 192)
// slots of a size-2^logM transform: kTwSlots on chip, the exact count beyond
// (long lines through a global-memory buffer, M up to 2^24: 6144 entries)
__host__ __device__ __forceinline__ int tw_slots(int logM) {
  const int b = logM > 1 ? logM - 1 : 0;
  const int lob = (b + 1) / 2;
  const int need = (1 << lob) + (1 << (b - lob));
  return need > kTwSlots ? need : kTwSlots;
}

// fill the two tables from the global table of M/2 entries; returns the view
__device__ __forceinline__ TwSm load_twiddles(double2* slots, const FftTables& T) {
  const int b = T.logM > 1 ? T.logM - 1 : 0;
  const int lob = (b + 1) / 2;
  const int nlo = 1 << lob, nhi = 1 << (b - lob);
  double2* lo = slots;
  double2* hi = slots + nlo;
  for (int i = threadIdx.x; i < nlo; i += blockDim.x) lo[i] = T.tw[i];
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) hi[i] = T.tw[(long long)i << lob];
  return TwSm{lo, hi, lob};
}

// ws[st] = w^(2^st): the twiddles of the LR radix-2 stages of one item from
// one table lookup and LR-1 squarings (relative error <= ~2^LR ulp)
template <int LR>
__device__ __forceinline__ void tw_pow2(double2 (&ws)[LR], double2 w) {
  ws[0] = w;
#pragma unroll
  for (int st = 1; st < LR; ++st) {
    const double2 a = ws[st - 1];
    ws[st] = make_double2(fma(a.x, a.x, -a.y * a.y), 2.0 * a.x * a.y);
  }
}

// ACC: every stage twiddle w^(2^st) straight from the tables (<= 2 ulp each)
// instead of by squaring (error doubling per stage, ~2^LR ulp).  The
// boundary-corrected real-line kernels fold a border polynomial of up to
// ~n times the data's magnitude into the transform input, so the FFT's own
// rounding constant sets their parity with the reference (DESIGN 4).
template <int LR, bool ACC, class TW>
__device__ __forceinline__ void tw_stage(double2 (&ws)[LR], const TW& tw, int j) {
  if constexpr (ACC) {
#pragma unroll
    for (int st = 0; st < LR; ++st) ws[st] = tw(j << st);
  } else {
    tw_pow2<LR>(ws, tw(j));
  }
}

// One fused pass of LOGR radix-2 decimation-in-frequency stages on blocks of
// size S (S >= 2^LOGR).  Items are disjoint element sets, so the pass is
// in-place with no barrier inside.
// nvalid < M: entries [nvalid, M) are read as zero (first pass of a
// zero-padded convolution; saves the padding stores and a barrier).
template <int LOGR, bool PAD = false, bool ACC = false>
__device__ __forceinline__ void dif_pass(double2* __restrict__ x, int M, int S, const TwSm& tw,
                                         int Mtw, int nvalid) {
  constexpr int R = 1 << LOGR;
  const int SR = S >> LOGR;
  const int items = M >> LOGR;
  const int twstep = Mtw >> (__ffs(S) - 1);  // Mtw / S: tw is a table for size Mtw >= M
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int j0 = it & (SR - 1);
    const int base = (it - j0) * R + j0;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q)
      v[q] = (!PAD || base + q * SR < nvalid) ? x[pidx(base + q * SR)] : czero();
    double2 ws[LOGR];
    tw_stage<LOGR, ACC>(ws, tw, j0 * twstep);
#pragma unroll
    for (int st = 0; st < LOGR; ++st) {
      const int half = R >> (st + 1);
      const double2 w = ws[st];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q], b = v[q + half];
        v[q] = cadd(a, b);
        const double2 d = mul_w16(csub(a, b), (qq << st) * (16 / R));
        v[q + half] = cmul(d, w);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[pidx(base + q * SR)] = v[q];
  }
}

// Exact inverse (times 2 per stage) of dif_pass with conjugate twiddles: the
// mirrored DIT pass of the backward transform.
template <int LOGR, bool ACC = false>
__device__ __forceinline__ void dit_pass(double2* __restrict__ x, int M, int S, const TwSm& tw,
                                         int Mtw) {
  constexpr int R = 1 << LOGR;
  const int SR = S >> LOGR;
  const int items = M >> LOGR;
  const int twstep = Mtw >> (__ffs(S) - 1);  // Mtw / S: tw is a table for size Mtw >= M
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int j0 = it & (SR - 1);
    const int base = (it - j0) * R + j0;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = x[pidx(base + q * SR)];
    double2 ws[LOGR];
    tw_stage<LOGR, ACC>(ws, tw, j0 * twstep);
#pragma unroll
    for (int st = LOGR - 1; st >= 0; --st) {
      const int half = R >> (st + 1);
      const double2 w = ws[st];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q];
        const double2 b = mul_w16c(cmulc(v[q + half], w), (qq << st) * (16 / R));
        v[q] = cadd(a, b);
        v[q + half] = csub(a, b);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[pidx(base + q * SR)] = v[q];
  }
}

// Pass sequence of a size-2^logM transform: the remainder radix first, then
// radix-16 passes, so every pass but the innermost has a sub-block stride
// SR >= 16 (padded addresses linear in q) and the innermost (mid) pass is
// radix 16 whenever logM >= 4.  k_bhat, the generic and the specialised
// Bluestein cores all use this sequence (bhat is stored in its DIF order).
__host__ __device__ __forceinline__ int num_passes(int logM) { return (logM + 3) / 4; }
__host__ __device__ __forceinline__ int pass_radix(int logM, int p) {
  const int rem = logM % 4;
  return (rem != 0 && p == 0) ? rem : 4;
}

// radix (log2) of the last DIF pass of a size-2^logM transform (the mid pass)
__host__ __device__ __forceinline__ int mid_logr(int logM) {
  return logM <= 0 ? 0 : (logM >= 4 ? 4 : logM);
}
// storage slot of DIF-order entry j of a bhat block of M = 2^logM points
__host__ __device__ __forceinline__ int bhat_store_index(int j, int logM) {
  const int lr = mid_logr(logM);
  const int items = (1 << logM) >> lr;
  return (j & ((1 << lr) - 1)) * items + (j >> lr);
}

// DIF passes over a local block of M points with twiddles of size Mtw.
__device__ __forceinline__ void fft_dif_local(double2* x, int M, int logM, int Mtw,
                                              const TwSm& tw) {
  int S = M;
  const int np = num_passes(logM);
  for (int p = 0; p < np; ++p) {
    const int l = pass_radix(logM, p);
    switch (l) {
      case 4: dif_pass<4>(x, M, S, tw, Mtw, M); break;
      case 3: dif_pass<3>(x, M, S, tw, Mtw, M); break;
      case 2: dif_pass<2>(x, M, S, tw, Mtw, M); break;
      default: dif_pass<1>(x, M, S, tw, Mtw, M); break;
    }
    S >>= l;
    __syncthreads();
  }
}

// The innermost DIF pass, the pointwise multiply by DIF(b)/M and the
// outermost DIT pass act on the same disjoint element groups (blocks of S
// consecutive positions, S = 2^LOGR), so they run as one register pass: load
// the group and its bhat values, LOGR DIF stages, multiply, LOGR DIT stages,
// store.  Saves two shared-memory round trips per Bluestein convolution.
// bhat is stored thread-major for this pass (bhat_store_index), so load q of
// all threads in a warp is one contiguous 512-byte read.
template <int LOGR, bool PAD = false>
__device__ __forceinline__ void mid_pass(double2* __restrict__ x, int M,
                                         const double2* __restrict__ bhat, const TwSm& tw,
                                         int nvalid) {
  constexpr int R = 1 << LOGR;
  const int items = M >> LOGR;
  const int twstep = M / R;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int base = it * R;  // S = R: SR = 1, j0 = 0
    double2 v[R], bh[R];
#pragma unroll
    for (int q = 0; q < R; ++q) bh[q] = __ldcg(&bhat[q * items + it]);  // L2 only: keep L1 for the filter tables
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = (!PAD || base + q < nvalid) ? x[pidx(base + q)] : czero();
    (void)twstep;
    // DIF stages with j0 = 0: every twiddle is a radix-16 constant
#pragma unroll
    for (int st = 0; st < LOGR; ++st) {
      const int half = R >> (st + 1);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q], b = v[q + half];
        v[q] = cadd(a, b);
        v[q + half] = mul_w16(csub(a, b), (qq << st) * (16 / R));
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = cmul(v[q], bh[q]);
#pragma unroll
    for (int st = LOGR - 1; st >= 0; --st) {
      const int half = R >> (st + 1);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q];
        const double2 b = mul_w16c(v[q + half], (qq << st) * (16 / R));
        v[q] = cadd(a, b);
        v[q + half] = csub(a, b);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) x[pidx(base + q)] = v[q];
  }
  (void)tw;
}

// Convolution with DIF(b)/M on a local block of Mloc points whose twiddles are
// those of size Mtw (Mloc = Mtw for an ordinary convolution; Mloc = Mtw/2 for
// one half of a split convolution, see bluestein_core).  bhat points at the
// Mloc entries of this block.  Requires a barrier before; ends with one.
template <bool ACC = false>
__device__ __forceinline__ void bluestein_run(double2* x, int M, int logM, int Mtw,
                                              const double2* bhat, const TwSm& tw, int nvalid) {
  if (logM == 0) {
    if (threadIdx.x == 0) x[0] = nvalid > 0 ? cmul(x[0], bhat[0]) : czero();
    __syncthreads();
    return;
  }
  int ls[8];
  const int np = num_passes(logM);
  for (int p = 0; p < np; ++p) ls[p] = pass_radix(logM, p);
  int S = M;
  for (int p = 0; p < np - 1; ++p) {
    if (p == 0 && nvalid < M) {  // zero padding: only the first pass reads it
      switch (ls[p]) {
        case 4: dif_pass<4, true, ACC>(x, M, S, tw, Mtw, nvalid); break;
        case 3: dif_pass<3, true, ACC>(x, M, S, tw, Mtw, nvalid); break;
        case 2: dif_pass<2, true, ACC>(x, M, S, tw, Mtw, nvalid); break;
        default: dif_pass<1, true, ACC>(x, M, S, tw, Mtw, nvalid); break;
      }
    } else {
      switch (ls[p]) {
        case 4: dif_pass<4, false, ACC>(x, M, S, tw, Mtw, M); break;
        case 3: dif_pass<3, false, ACC>(x, M, S, tw, Mtw, M); break;
        case 2: dif_pass<2, false, ACC>(x, M, S, tw, Mtw, M); break;
        default: dif_pass<1, false, ACC>(x, M, S, tw, Mtw, M); break;
      }
    }
    S >>= ls[p];
    __syncthreads();
  }
  if (np == 1 && nvalid < M) {
    switch (ls[0]) {
      case 4: mid_pass<4, true>(x, M, bhat, tw, nvalid); break;
      case 3: mid_pass<3, true>(x, M, bhat, tw, nvalid); break;
      case 2: mid_pass<2, true>(x, M, bhat, tw, nvalid); break;
      default: mid_pass<1, true>(x, M, bhat, tw, nvalid); break;
    }
  } else {
    switch (ls[np - 1]) {  // S == 2^ls[np-1] here
      case 4: mid_pass<4>(x, M, bhat, tw, M); break;
      case 3: mid_pass<3>(x, M, bhat, tw, M); break;
      case 2: mid_pass<2>(x, M, bhat, tw, M); break;
      default: mid_pass<1>(x, M, bhat, tw, M); break;
    }
  }
  __syncthreads();
  for (int p = np - 2; p >= 0; --p) {
    S <<= ls[p];
    switch (ls[p]) {
      case 4: dit_pass<4, ACC>(x, M, S, tw, Mtw); break;
      case 3: dit_pass<3, ACC>(x, M, S, tw, Mtw); break;
      case 2: dit_pass<2, ACC>(x, M, S, tw, Mtw); break;
      default: dit_pass<1, ACC>(x, M, S, tw, Mtw); break;
    }
    __syncthreads();
  }
}

// Bluestein core: x holds a_j = z_j c_j (j < nvalid <= L; entries beyond are
// taken as zero, whatever the buffer holds); on return x_k holds the circular
// convolution (a * b)_k; the caller multiplies by c_k.
// Requires a barrier before the call (the caller's loads); ends with one.
template <bool ACC = false>
__device__ __forceinline__ void bluestein_core(double2* x, const FftTables& T, const TwSm& tw,
                                               int nvalid) {
  bluestein_run<ACC>(x, T.M, T.logM, T.M, T.bhat, tw, nvalid);
}

// Split convolution for M beyond shared memory (M = 2 * Mloc).  The input a
// is supported on [0, L) with L <= M/2, so the first DIF stage degenerates to
// upper = lower (.) W_M^t and the last DIT stage only has to produce the lower
// half: out[t] = y0[t] + conj(W_M^t) y1[t], where y_p is the half-size
// convolution of half p (DIF(b)/M entries [p Mloc, (p+1) Mloc)).
//   part 1: x = a (.) W^t  ->  y1   (caller saves y1)
//   part 0: x = a          ->  y0   (caller combines)
template <bool ACC = false>
__device__ __forceinline__ void bluestein_half(double2* x, const FftTables& T, const TwSm& tw,
                                               int part, int nvalid) {
  const int Mloc = T.M >> 1;
  if (part == 1) {
    for (int j = threadIdx.x; j < nvalid; j += blockDim.x) x[pidx(j)] = cmul(x[pidx(j)], tw(j));
    __syncthreads();
  }
  bluestein_run<ACC>(x, Mloc, T.logM - 1, T.M, T.bhat + part * Mloc, tw, nvalid);
}

// ----------------------------------------------------------------------------
// Size-specialised Bluestein core (LOGM known at compile time).  Same
// arithmetic, pass sequence and bhat layout as bluestein_run, but the launch
// uses exactly FftShape<LOGM>::NT threads, every pass is unrolled, and every
// shared-memory address is one per-thread base plus compile-time offsets
// (pidx(base + q SR) = pidx(base) + q (SR + SR/16) for SR a multiple of 16).
// NTH != 0 overrides the thread count (one CTA per SM at large M wants more warps)
template <int LOGM, int NTH = 0>
struct FftShape {
  static constexpr int M = 1 << LOGM;
  static constexpr int NT =
      NTH ? NTH : (M / 16 >= 256 ? 256 : (M / 16 <= 64 ? 64 : M / 16));
  static constexpr int NP = (LOGM + 3) / 4;
  static constexpr int LOB = ((LOGM > 1 ? LOGM - 1 : 0) + 1) / 2;  // load_twiddles' split
};

template <int LOB>
__device__ __forceinline__ double2 tw_t(const TwSm& tw, int j) {
  return cmul(tw.hi[j >> LOB], tw.lo[j & ((1 << LOB) - 1)]);
}

template <int LOGM, int LR, int S, bool PAD, int NTH = 0, bool ACC = false>
__device__ __forceinline__ void dif_pass_t(double2* __restrict__ x, const TwSm& tw, int nvalid) {
  using F = FftShape<LOGM, NTH>;
  constexpr int R = 1 << LR, SR = S >> LR, ITEMS = F::M >> LR;
  constexpr int TWSTEP = F::M / S;
  constexpr int QS = SR + SR / 16;
  static_assert(SR % 16 == 0, "outer passes have SR >= 16");
#pragma unroll
  for (int i0 = 0; i0 < ITEMS; i0 += F::NT) {
    const int it = i0 + threadIdx.x;
    if (ITEMS < F::NT && it >= ITEMS) break;
    const int j0 = it & (SR - 1);
    const int base = (it - j0) * R + j0;
    double2* xb = x + pidx(base);
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = (!PAD || base + q * SR < nvalid) ? xb[q * QS] : czero();
    double2 ws[LR];
    if constexpr (ACC) {
#pragma unroll
      for (int st = 0; st < LR; ++st) ws[st] = tw_t<F::LOB>(tw, (j0 * TWSTEP) << st);
    } else {
      tw_pow2<LR>(ws, tw_t<F::LOB>(tw, j0 * TWSTEP));
    }
#pragma unroll
    for (int st = 0; st < LR; ++st) {
      const int half = R >> (st + 1);
      const double2 w = ws[st];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q], b = v[q + half];
        v[q] = cadd(a, b);
        v[q + half] = cmul(mul_w16(csub(a, b), (qq << st) * (16 / R)), w);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) xb[q * QS] = v[q];
  }
}

template <int LOGM, int LR, int S, int NTH = 0, bool ACC = false>
__device__ __forceinline__ void dit_pass_t(double2* __restrict__ x, const TwSm& tw) {
  using F = FftShape<LOGM, NTH>;
  constexpr int R = 1 << LR, SR = S >> LR, ITEMS = F::M >> LR;
  constexpr int TWSTEP = F::M / S;
  constexpr int QS = SR + SR / 16;
  static_assert(SR % 16 == 0, "outer passes have SR >= 16");
#pragma unroll
  for (int i0 = 0; i0 < ITEMS; i0 += F::NT) {
    const int it = i0 + threadIdx.x;
    if (ITEMS < F::NT && it >= ITEMS) break;
    const int j0 = it & (SR - 1);
    const int base = (it - j0) * R + j0;
    double2* xb = x + pidx(base);
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = xb[q * QS];
    double2 ws[LR];
    if constexpr (ACC) {
#pragma unroll
      for (int st = 0; st < LR; ++st) ws[st] = tw_t<F::LOB>(tw, (j0 * TWSTEP) << st);
    } else {
      tw_pow2<LR>(ws, tw_t<F::LOB>(tw, j0 * TWSTEP));
    }
#pragma unroll
    for (int st = LR - 1; st >= 0; --st) {
      const int half = R >> (st + 1);
      const double2 w = ws[st];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q];
        const double2 b = mul_w16c(cmulc(v[q + half], w), (qq << st) * (16 / R));
        v[q] = cadd(a, b);
        v[q + half] = csub(a, b);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) xb[q * QS] = v[q];
  }
}

// innermost radix-16 pass: DIF stages, multiply by bhat, DIT stages
template <int LOGM, bool PAD, int NTH = 0>
__device__ __forceinline__ void mid_pass_t(double2* __restrict__ x,
                                           const double2* __restrict__ bhat, int nvalid) {
  using F = FftShape<LOGM, NTH>;
  constexpr int R = 16, ITEMS = F::M / 16;
#pragma unroll
  for (int i0 = 0; i0 < ITEMS; i0 += F::NT) {
    const int it = i0 + threadIdx.x;
    if (ITEMS < F::NT && it >= ITEMS) break;
    const int base = it * R;
    double2* xb = x + pidx(base);
    double2 v[R], bh[R];
#pragma unroll
    for (int q = 0; q < R; ++q) bh[q] = __ldcg(&bhat[q * ITEMS + it]);  // L2 only: keep L1 for the filter tables
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = (!PAD || base + q < nvalid) ? xb[q] : czero();
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      const int half = R >> (st + 1);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q], b = v[q + half];
        v[q] = cadd(a, b);
        v[q + half] = mul_w16(csub(a, b), qq << st);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = cmul(v[q], bh[q]);
#pragma unroll
    for (int st = 3; st >= 0; --st) {
      const int half = R >> (st + 1);
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (q & half) continue;
        const int qq = q & (half - 1);
        const double2 a = v[q];
        const double2 b = mul_w16c(v[q + half], qq << st);
        v[q] = cadd(a, b);
        v[q + half] = csub(a, b);
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) xb[q] = v[q];
  }
}

// Barrier between passes.  GRP == 0: the whole CTA.  GRP > 0: the threads
// [g GRP, (g+1) GRP) only (named barrier 1 + g) -- for pass sequences whose
// items split into independent element sets per thread group (the two halves
// of a folded convolution at NT = M/16: thread group g owns half g in every
// pass), so the groups drift out of phase and one group's shared-memory
// traffic overlaps the other's arithmetic.
template <int GRP>
__device__ __forceinline__ void pass_sync() {
  if constexpr (GRP == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / GRP)), "n"(GRP) : "memory");
  }
}

// pass P of the DIF sequence (block size S), the inner passes, then its DIT mirror
template <int LOGM, int P, int S, int NTH = 0, bool ACC = false, int GRP = 0>
__device__ __forceinline__ void bluestein_rec(double2* x, const double2* bhat, const TwSm& tw,
                                              int nvalid) {
  using F = FftShape<LOGM, NTH>;
  if constexpr (P == F::NP - 1) {
    if (P == 0 && nvalid < F::M)
      mid_pass_t<LOGM, true, NTH>(x, bhat, nvalid);
    else
      mid_pass_t<LOGM, false, NTH>(x, bhat, nvalid);
    pass_sync<GRP>();
  } else {
    constexpr int LR = (P == 0 && LOGM % 4 != 0) ? LOGM % 4 : 4;
    if (P == 0 && nvalid < F::M)
      dif_pass_t<LOGM, LR, S, true, NTH, ACC>(x, tw, nvalid);
    else
      dif_pass_t<LOGM, LR, S, false, NTH, ACC>(x, tw, nvalid);
    pass_sync<GRP>();
    bluestein_rec<LOGM, P + 1, (S >> LR), NTH, ACC, GRP>(x, bhat, tw, nvalid);
    dit_pass_t<LOGM, LR, S, NTH, ACC>(x, tw);
    pass_sync<GRP>();
  }
}

// bluestein_core for a compile-time size (LOGM >= 4), blockDim.x == FftShape<LOGM, NTH>::NT
template <int LOGM, int NTH = 0, bool ACC = false>
__device__ __forceinline__ void bluestein_t(double2* x, const FftTables& T, const TwSm& tw,
                                            int nvalid) {
  bluestein_rec<LOGM, 0, (1 << LOGM), NTH, ACC>(x, T.bhat, tw, nvalid);
}

// ----------------------------------------------------------------------------
// block reductions (deterministic: fixed shuffle tree, then warp order)
// ----------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch /* >= 32*NV */) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[warp * NV + k] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc += scratch[w * NV + k];
    v[k] = acc;
  }
  __syncthreads();
}

}  // namespace fdb
