// Direct mixed-radix DFT for the pair kernels when the interior length m is
// a product of small odd radices (3, 5, 7, 9, 11, 13): m = 4095 = 13*9*7*5 at
// n = 4096, d = 1.  Bluestein (fd_pair.cuh) spends two 8192-point FFTs per
// pair of lines; the direct in-place decimation-in-frequency transform of
// length m needs ~45 fp64 instructions per point and four shared-memory
// passes over 64 KB instead of seven over 139 KB.
//
// Stage s (radix r, block size S, stride L = S/r) applies, for every block and
// j < L, the r-point DFT to x[blk S + j + q L] (q < r) and multiplies output p
// by w_S^{jp} = w_m^{jp m/S}; after the last stage frequency k sits at
// mperm[k] (mixed-radix digit reversal, a host-built table).  The r-point
// DFTs use the symmetric split (x_j +- x_{r-j}) with constant-memory cos/sin.
// Everything else -- border fold, Hermitian split of the two lines, packed
// coefficients, GCV weights, TF32 tiles, filtered synthesis -- is the pair
// kernels' (fd_pair.cuh), without the chirp.
#pragma once

namespace fdb {

constexpr int kMixMaxStages = 6;
#ifndef FD_MIX_NT
#define FD_MIX_NT 256
#endif
constexpr int kMixNTc = FD_MIX_NT;  // threads per CTA of k_manalyze / k_msynth (kMixNT below)
// cos / sin (2 pi t / r) for t = 0 .. 6, radix r = 3 .. 13 (row r)
constexpr int kMixMaxR = 13;
__constant__ double c_mix_cos[kMixMaxR + 1][7];
__constant__ double c_mix_sin[kMixMaxR + 1][7];

// forward r-point DFT in registers: v[p] <- sum_q v[q] e^{-2 pi i pq / r}, r odd
template <int R>
__device__ __forceinline__ void mix_codelet(double2 (&v)[R]) {
  constexpr int H = R / 2;
  double2 s[H], d[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    s[j - 1] = cadd(v[j], v[R - j]);
    d[j - 1] = csub(v[j], v[R - j]);
  }
  double2 x0 = v[0];
#pragma unroll
  for (int j = 0; j < H; ++j) x0 = cadd(x0, s[j]);
  double2 out[R];
  out[0] = x0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 A = v[0], B = czero();
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int t = (j * k) % R;
      const double cv = c_mix_cos[R][t <= H ? t : R - t];
      const double sv = t <= H ? c_mix_sin[R][t] : -c_mix_sin[R][R - t];
      A.x = fma(s[j - 1].x, cv, A.x);
      A.y = fma(s[j - 1].y, cv, A.y);
      B.x = fma(d[j - 1].x, sv, B.x);
      B.y = fma(d[j - 1].y, sv, B.y);
    }
    out[k] = make_double2(A.x + B.y, A.y - B.x);      // A - iB
    out[R - k] = make_double2(A.x - B.y, A.y + B.x);  // A + iB
  }
#pragma unroll
  for (int p = 0; p < R; ++p) v[p] = out[p];
}

// twiddles w_m^t from two shared-memory tables: hi[t >> 6] * lo[t & 63]
struct MixTw {
  const double2* lo;
  const double2* hi;
  __device__ __forceinline__ double2 operator()(int t) const { return cmul(hi[t >> 6], lo[t & 63]); }
};

// v[p] *= w1^p for p = 1 .. R-1, the powers by a squaring tree (depth
// log2 R, <= 4 roundings): two shared-memory loads per item instead of
// 2 (R - 1) scattered twiddle-table reads
template <int R>
__device__ __forceinline__ void mix_twiddle(double2 (&v)[R], double2 w1) {
  double2 w[R];
  w[1] = w1;
#pragma unroll
  for (int p = 2; p < R; ++p) w[p] = (p & 1) ? cmul(w[p - 1], w1) : cmul(w[p / 2], w[p / 2]);
#pragma unroll
  for (int p = 1; p < R; ++p) v[p] = cmul(v[p], w[p]);
}

template <int R>
__device__ __forceinline__ void mix_stage(double2* __restrict__ x, int N, int S, const MixTw& tw,
                                          int nt) {
  const int L = S / R, items = N / R, tstep = N / S;
  for (int it = threadIdx.x; it < items; it += nt) {
    const int blk = it / L, j = it - blk * L;
    double2* xb = x + blk * S + j;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = xb[q * L];
    mix_codelet<R>(v);
    if (L > 1) mix_twiddle<R>(v, tw(j * tstep));
#pragma unroll
    for (int p = 0; p < R; ++p) xb[p * L] = v[p];
  }
}

// first stage (S = N) reading its inputs through ld(j) instead of x: the
// analysis computes them from global memory (border fold included), which
// saves the load phase's shared-memory pass and barrier
template <int R, class LD>
__device__ __forceinline__ void mix_stage_first(double2* __restrict__ x, int N, const MixTw& tw,
                                                int nt, LD&& ld) {
  const int L = N / R;
  for (int j = threadIdx.x; j < L; j += nt) {
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = ld(j + q * L);
    mix_codelet<R>(v);
    if (L > 1) mix_twiddle<R>(v, tw(j));
#pragma unroll
    for (int p = 0; p < R; ++p) x[j + p * L] = v[p];
  }
}

// Compile-time stage sequences (BASELINE config 1, d = 1: m = 4095 = 5 13 9 7):
// block sizes, strides and item counts are constants, so the item -> (block,
// j) split is a multiply-shift and every shared-memory offset an immediate --
// the generic stages spend two of three issued instructions on that arithmetic.
template <int N, int S, int R, int NT>
__device__ __forceinline__ void mix_stage_c(double2* __restrict__ x, const MixTw& tw) {
  constexpr int L = S / R, ITEMS = N / R, TSTEP = N / S;
#pragma unroll 1
  for (int it = threadIdx.x; it < ITEMS; it += NT) {
    const int blk = it / L, j = it - blk * L;
    double2* xb = x + blk * S + j;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = xb[q * L];
    mix_codelet<R>(v);
    if constexpr (L > 1) mix_twiddle<R>(v, tw(j * TSTEP));
#pragma unroll
    for (int p = 0; p < R; ++p) xb[p * L] = v[p];
  }
}
template <int N, int S, int NT, int R, int... REST>
__device__ __forceinline__ void mix_stages_c(double2* x, const MixTw& tw) {
  mix_stage_c<N, S, R, NT>(x, tw);
  __syncthreads();
  if constexpr (sizeof...(REST) > 0) mix_stages_c<N, S / R, NT, REST...>(x, tw);
}
template <int N, int R, int NT, class LD>
__device__ __forceinline__ void mix_stage_first_c(double2* __restrict__ x, const MixTw& tw,
                                                  LD&& ld) {
  constexpr int L = N / R;
#pragma unroll 2
  for (int j = threadIdx.x; j < L; j += NT) {
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = ld(j + q * L);
    mix_codelet<R>(v);
    mix_twiddle<R>(v, tw(j));
#pragma unroll
    for (int p = 0; p < R; ++p) x[j + p * L] = v[p];
  }
}
// the plan is the compile-time sequence 5 13 9 7 (build_mixed_plan's order)
__device__ __forceinline__ bool mix_plan_4095(const AxisDev& ax) {
  return ax.m == 4095 && ax.mstages == 4 && ax.mrad[0] == 5 && ax.mrad[1] == 13 &&
         ax.mrad[2] == 9 && ax.mrad[3] == 7;
}

// in-place DIF DFT of length ax.m (natural order in, mperm order out); with a
// loader the first stage reads x_j = ld(j) (FIRST_LD)
template <bool FIRST_LD = false, class LD = int, class AF = int>
__device__ __forceinline__ void mix_dft(double2* x, const AxisDev& ax, const MixTw& tw, int nt,
                                        LD&& ld = 0, AF&& after_first = 0) {
  if (mix_plan_4095(ax) && nt == kMixNTc) {
    if constexpr (FIRST_LD) {
      mix_stage_first_c<4095, 5, kMixNTc>(x, tw, ld);
      after_first();  // before the stage barrier
      __syncthreads();
      mix_stages_c<4095, 819, kMixNTc, 13, 9, 7>(x, tw);
    } else {
      mix_stages_c<4095, 4095, kMixNTc, 5, 13, 9, 7>(x, tw);
    }
    return;
  }
  int S = ax.m;
  int s0 = 0;
  if constexpr (FIRST_LD) {
    const int r = ax.mrad[0];
    switch (r) {
      case 3: mix_stage_first<3>(x, ax.m, tw, nt, ld); break;
      case 5: mix_stage_first<5>(x, ax.m, tw, nt, ld); break;
      case 7: mix_stage_first<7>(x, ax.m, tw, nt, ld); break;
      case 9: mix_stage_first<9>(x, ax.m, tw, nt, ld); break;
      case 11: mix_stage_first<11>(x, ax.m, tw, nt, ld); break;
      default: mix_stage_first<13>(x, ax.m, tw, nt, ld); break;
    }
    after_first();  // before the stage barrier
    S /= r;
    s0 = 1;
    __syncthreads();
  }
  for (int s = s0; s < ax.mstages; ++s) {
    const int r = ax.mrad[s];
    switch (r) {
      case 3: mix_stage<3>(x, ax.m, S, tw, nt); break;
      case 5: mix_stage<5>(x, ax.m, S, tw, nt); break;
      case 7: mix_stage<7>(x, ax.m, S, tw, nt); break;
      case 9: mix_stage<9>(x, ax.m, S, tw, nt); break;
      case 11: mix_stage<11>(x, ax.m, S, tw, nt); break;
      default: mix_stage<13>(x, ax.m, S, tw, nt); break;
    }
    S /= r;
    __syncthreads();
  }
}

// threads per CTA (two CTAs per SM).  320 threads (98 / 71 / 91 / 85 % full stage rounds at m = 4095
// instead of 61 / 89 / 76 / 80 %) at 96 registers measured no faster (k_msynth 2.27 -> 2.36 ms, r02)
#ifndef FD_MIX_NT
#define FD_MIX_NT 256
#endif
constexpr int kMixNT = FD_MIX_NT;

// L2 prefetch of the line pair q (contiguous lines only), issued one pair
// ahead so the load phase of the persistent loop hits L2 instead of HBM
__device__ __forceinline__ void mix_prefetch_pair(const void* base, const Lines& g, int q, int n) {
  if (threadIdx.x != 0 || g.elem_stride != 1 || 2 * q >= g.count || (n & 1)) return;
#pragma unroll
  for (int l = 2 * q; l < 2 * q + 2; ++l) {
    if (l >= g.count) break;
    const double* src = reinterpret_cast<const double*>(base) + line_offset(g, l);
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) bulk_prefetch_l2(src, (uint32_t)n * 8);
  }
}

// smem (double2 slots): DFT buffer (max(m + 1, n): the two output lines of n
// doubles are assembled in it) | twiddle lo (64), hi | weight rows of the pair
// (wslots = wstride of the analysis with GCV weights, else 0) | output
// permutation (u16) | the two zero-line flag words (zf_add / zf_take)
constexpr int kMixK = 8;   // Hermitian slots per thread of the staged-output path: h + 1 <= 8 NT
constexpr int kMixP = 16;  // sample slots per thread: m <= 16 NT
__host__ __device__ __forceinline__ int mix_x_slots(int m, int n) { return m + 1 > n ? m + 1 : n; }
__host__ __device__ __forceinline__ size_t mix_smem_bytes(int m, int n, long long wslots) {
  return ((size_t)mix_x_slots(m, n) + 64 + ((m + 63) >> 6) + (size_t)wslots + (m + 7) / 8 + 1) * 16;
}
struct MixLay {
  MixTw tw;
  double* wrows;
  const unsigned short* perm;
  int* zf;
};
// twiddle tables and permutation into shared memory (before the first barrier)
__device__ __forceinline__ MixLay mix_setup(double2* sm, const AxisDev& ax, long long wslots) {
  const int m = ax.m, nhi = (m + 63) >> 6;
  double2* lo = sm + mix_x_slots(m, ax.n);
  double2* hi = lo + 64;
  double2* wr = hi + nhi;
  unsigned short* ps = reinterpret_cast<unsigned short*>(wr + wslots);
  int* zf = reinterpret_cast<int*>(reinterpret_cast<double2*>(ps) + (m + 7) / 8);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) lo[i] = i < m ? ax.mtw[i] : czero();
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) hi[i] = ax.mtw[i << 6];
  for (int i = threadIdx.x; i < m; i += blockDim.x) ps[i] = (unsigned short)ax.mperm[i];
  if (threadIdx.x < 2) zf[threadIdx.x] = 0;  // zero-line flags
  return MixLay{MixTw{lo, hi}, reinterpret_cast<double*>(wr), ps, zf};
}
// the output lines can be assembled in the buffer and bulk-stored
__device__ __forceinline__ bool mix_out_staged(const AxisDev& ax, const double* o0,
                                               const double* o1, long long eso) {
  return pair_out_staged(o0, o1, ax.n, eso) && (ax.m - 1) / 2 < kMixK * kMixNT &&
         ax.m <= kMixP * kMixNT;
}

// analyze, two real lines per direct DFT (see k_panalyze)
__global__ void __launch_bounds__(kMixNT, 2) k_manalyze(AxisDev ax, LineIO io, int wslots) {
  extern __shared__ double2 sm[];
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  const MixLay lay = mix_setup(sm, ax, wslots);
  const MixTw tw = lay.tw;
  const unsigned short* perm = lay.perm;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const long long es = io.gi.elem_stride;
  const double isq = ax.inv_sqrt_m;
  const long long nkb32 = io.wstride >> 5;
  int* zf = lay.zf;
  double* wA = lay.wrows;
  double* wB = wA + io.wstride;
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    // streaming loads (the pair was prefetched into L2; nothing re-reads it)
    auto ld0 = [&](int e) { return __ldcs(g0 + e * es); };
    auto ld1 = [&](int e) { return has1 ? __ldcs(g1 + e * es) : 0.0; };
    double a0[kHoMax], a1[kHoMax];
    ho_amps_real(ax, ld0, a0);
    ho_amps_real(ax, ld1, a1);
    const Cubic p0 = ho_cubic(ax, a0), p1 = ho_cubic(ax, a1);
    long long nzb0 = 0, nzb1 = 0;  // OR of the bit patterns of line 0 / 1 (-0.0 counts as nonzero)
    // the previous pair's output lines must have left x (and the weight rows);
    // the SM's other CTA computes meanwhile
    if (threadIdx.x == 0) bulk_wait_read();
    __syncthreads();
    mix_dft<true>(x, ax, tw, kMixNT, [&](int j) {
      const int e = kl + j;
      const double t = fma((double)e, ax.ho_ta, ax.ho_tb);
      const double y0 = ld0(e), y1 = ld1(e);
      nzb0 |= __double_as_longlong(y0);  // integer pipe: the fp64 pipe is the bound
      nzb1 |= __double_as_longlong(y1);
      return make_double2(y0 - p0(t), y1 - p1(t));
    }, [&] { zf_add(zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0)); });
    // the next pair into L2 while the outputs stream out
    mix_prefetch_pair(io.in, io.gi, q + gridDim.x, n);

    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    double* w0 = io.wout ? io.wout + (long long)l0 * io.wstride : nullptr;
    double* w1 = (w0 && has1) ? w0 + io.wstride : nullptr;
    // an all-zero line gets exactly zero coefficients (its partner's DFT
    // round-off would otherwise leak into it through the Hermitian split)
    const int nz = zf_take(zf, it);
    const bool z0 = !(nz & 1) && ho_zero(a0), z1 = !(nz & 2) && ho_zero(a1);
    // Staged output (see k_panalyze): the packed coefficient lines are
    // assembled in x and the weight rows in their staging area, both leave by
    // bulk stores; the TF32 tiles are written chunk-wise from the staged rows
    const bool tout = mix_out_staged(ax, o0, o1, io.go.elem_stride) && (hk & 1);
    const bool wst = tout && w0 && wslots >= io.wstride && (io.wstride & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(w0) & 15) == 0;
    auto wset = [&](int line, double* wl, long long i, double v) {
      wl[i] = v;
      if (io.wout32) {
        float hi, lo;
        tf32_split(v, hi, lo);
        const long long t = tc_tile_index(line, i, kTcBM, nkb32);
        io.wout32[t] = hi;
        io.wout32lo[t] = lo;
      }
    };
    if (tout) {
      double2 X0r[kMixK], X1r[kMixK];
#pragma unroll
      for (int t = 0; t < kMixK; ++t) {
        const int kq = threadIdx.x + t * kMixNT;
        const int kk = kq <= h ? kq : h;  // clamped: branch-free slots interleave
        const double2 Zk = x[perm[kk]];
        const double2 Zm = x[perm[kk ? m - kk : 0]];
        const double2 Zc = kk ? Zm : Zk;
        const double2 D = csub(Zk, cconj(Zc));
        const double2 X0 = z0 ? czero() : cscale(cadd(Zk, cconj(Zc)), 0.5 * isq);
        const double2 X1 = z1 ? czero() : make_double2(0.5 * isq * D.y, -0.5 * isq * D.x);
        X0r[t] = X0;
        X1r[t] = X1;
        if (w0 && kq <= h) {
          const double f = kk ? 2.0 : 1.0;  // |X_k|^2 + |X_{m-k}|^2
          const double v0 = f * (X0.x * X0.x + X0.y * X0.y), v1 = f * (X1.x * X1.x + X1.y * X1.y);
          if (wst) {
            wA[kl + kk] = v0;
            wB[kl + kk] = v1;
          } else {
            wset(l0, w0, kl + kk, v0);
            if (w1) wset(l0 + 1, w1, kl + kk, v1);
          }
        }
      }
      if (wst) {
        if (threadIdx.x < hk) {
          const int l = threadIdx.x, i = ho_wred(ax, l, h);
          wA[i] = a0[l] * a0[l];
          wB[i] = a1[l] * a1[l];
        }
        for (int i = (int)io.wn + threadIdx.x; i < (int)io.wstride; i += kMixNT) wA[i] = wB[i] = 0.0;
      }
      __syncthreads();  // every Z_k has been read; the weight rows are complete
      double* lineA = reinterpret_cast<double*>(x);
      double* lineB = lineA + n;
#pragma unroll
      for (int t = 0; t < kMixK; ++t) {
        const int kk = threadIdx.x + t * kMixNT;
        if (kk > h) continue;
        if (kk == 0) {
          lineA[hk] = X0r[t].x;
          lineB[hk] = X1r[t].x;
        } else {  // hk odd: (Re, Im) 16-byte aligned
          *reinterpret_cast<double2*>(lineA + hk + 2 * kk - 1) = X0r[t];
          *reinterpret_cast<double2*>(lineB + hk + 2 * kk - 1) = X1r[t];
        }
      }
      if (threadIdx.x < hk) {
        lineA[threadIdx.x] = a0[threadIdx.x];
        lineB[threadIdx.x] = a1[threadIdx.x];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (wst && io.wout32) {  // task c: chunk c >> 1 (4 elements) of line l0 + (c & 1)
        float* th = io.wout32 + tc_tile_index(l0, 0, kTcBM, nkb32);
        float* tl = io.wout32lo + tc_tile_index(l0, 0, kTcBM, nkb32);
        const int ntask = (int)(io.wstride >> 1);
        for (int c = threadIdx.x; c < ntask; c += kMixNT) {
          const int row = c & 1, i = (c >> 1) * 4;
          if (row && !has1) continue;
          const double2* src = reinterpret_cast<const double2*>((row ? wB : wA) + i);
          const double2 u0 = src[0], u1 = src[1];
          float4 hi, lo;
          tf32_split(u0.x, hi.x, lo.x);
          tf32_split(u0.y, hi.y, lo.y);
          tf32_split(u1.x, hi.z, lo.z);
          tf32_split(u1.y, hi.w, lo.w);
          const int eo = (i >> 5) * (kTcBM * 32) + ((i & 31) >> 2) * (kTcBM * 4) + row * 4;
          *reinterpret_cast<float4*>(th + eo) = hi;
          *reinterpret_cast<float4*>(tl + eo) = lo;
        }
      }
    } else {
      for (int kk = threadIdx.x; kk <= h; kk += kMixNT) {
        const double2 Zk = x[perm[kk]];
        const double2 Zc = kk ? x[perm[m - kk]] : Zk;
        const double2 D = csub(Zk, cconj(Zc));
        const double2 X0 = z0 ? czero() : cscale(cadd(Zk, cconj(Zc)), 0.5 * isq);
        const double2 X1 = z1 ? czero() : make_double2(0.5 * isq * D.y, -0.5 * isq * D.x);
        if (kk == 0) {
          __stcs(o0 + hk, X0.x);
          if (o1) __stcs(o1 + hk, X1.x);
        } else {
          __stcs(o0 + hk + 2 * kk - 1, X0.x);
          __stcs(o0 + hk + 2 * kk, X0.y);
          if (o1) {
            __stcs(o1 + hk + 2 * kk - 1, X1.x);
            __stcs(o1 + hk + 2 * kk, X1.y);
          }
        }
        if (w0) {
          const double f = kk ? 2.0 : 1.0;
          wset(l0, w0, kl + kk, f * (X0.x * X0.x + X0.y * X0.y));
          if (w1) wset(l0 + 1, w1, kl + kk, f * (X1.x * X1.x + X1.y * X1.y));
        }
      }
    }
    if (threadIdx.x < hk) {
      const int l = threadIdx.x;
      if (!tout) {
        o0[l] = a0[l];
        if (o1) o1[l] = a1[l];
      }
      if (w0 && !wst) {
        wset(l0, w0, ho_wred(ax, l, h), a0[l] * a0[l]);
        if (w1) wset(l0 + 1, w1, ho_wred(ax, l, h), a1[l] * a1[l]);
      }
    }
    if (w0 && !wst)
      for (long long i = io.wn + threadIdx.x; i < io.wstride; i += kMixNT) {
        wset(l0, w0, i, 0.0);
        if (w1) wset(l0 + 1, w1, i, 0.0);
      }
    __syncthreads();
    if (tout && threadIdx.x == 0) {
      bulk_s2g(o0, x, (uint32_t)n * 8);
      if (o1) bulk_s2g(o1, reinterpret_cast<double*>(x) + n, (uint32_t)n * 8);
      if (wst) {
        bulk_s2g(w0, wA, (uint32_t)io.wstride * 8);
        if (has1) bulk_s2g(w0 + io.wstride, wB, (uint32_t)io.wstride * 8);
      }
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

// synthesis with the filter fused, two lines per direct DFT (see k_psynth)
__global__ void __launch_bounds__(kMixNT, 2) k_msynth(AxisDev ax, LineIO io, SynthArgs sa) {
  extern __shared__ double2 sm[];
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  const MixLay lay = mix_setup(sm, ax, 0);
  const MixTw tw = lay.tw;
  const unsigned short* perm = lay.perm;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
  int* zf = lay.zf;
  const double tt0 = fma((double)(kl + (int)threadIdx.x), ax.ho_ta, ax.ho_tb);
  auto pair_mu = [&](int q, double& m0, double& m1) {  // read one pair ahead
    m0 = m1 = 0.0;
    if (q < npairs) {
      m0 = line_mu(sa, io.gi, 2 * q);
      m1 = 2 * q + 1 < count ? line_mu(sa, io.gi, 2 * q + 1) : m0;
    }
  };
  double mu0n, mu1n;
  pair_mu(blockIdx.x, mu0n, mu1n);
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    const double mu0 = mu0n, mu1 = mu1n;
    pair_mu(q + gridDim.x, mu0n, mu1n);
    auto f0 = [&](int e, double2 c) { return coeff_filter_fast(ax, sa, io.gi, l0, e, c, mu0); };
    auto f1 = [&](int e, double2 c) {
      return has1 ? coeff_filter_fast(ax, sa, io.gi, l0 + 1, e, c, mu1) : czero();
    };
    // streaming loads: the pair was prefetched into L2 and is read once, so
    // L1 keeps the filter's spectral table
    auto ld0 = [&](int i) { return __ldcs(g0 + i); };
    auto ld1 = [&](int i) { return has1 ? __ldcs(g1 + i) : 0.0; };
    // (Re, Im) of coefficient kk >= 1 at [hk + 2 kk - 1]: one 16-byte load when aligned
    const bool v2 = (hk & 1) && ((reinterpret_cast<uintptr_t>(g0) | reinterpret_cast<uintptr_t>(g1)) & 15) == 0;
    auto ldp0 = [&](int i) {
      return v2 ? __ldcs(reinterpret_cast<const double2*>(g0 + i)) : make_double2(ld0(i), ld0(i + 1));
    };
    auto ldp1 = [&](int i) {
      if (!has1) return czero();
      return v2 ? __ldcs(reinterpret_cast<const double2*>(g1 + i)) : make_double2(ld1(i), ld1(i + 1));
    };
    // the previous pair's output lines must have left x
    if (threadIdx.x == 0) bulk_wait_read();
    __syncthreads();
    double ua0[kHoMax], ua1[kHoMax];
    long long nzb0 = 0, nzb1 = 0;  // all-zero filtered lines are written as exact zeros
    // Fast path (1D filter of a complex basis, aligned lines, h + 1 <= 8 NT):
    // straight-line batches of four slots, every load of a batch -- coefficient
    // pairs and spectral values -- issued before its first use.  The generic
    // loop below runs slot after slot behind the filter's mode branches, one
    // L2 round trip each (39 % of the kernel, 40 % long-scoreboard stalls).
    const bool fast = sa.mode == 1 && sa.sp.mode == 1 && ax.cplx && v2 && h < kMixK * kMixNT;
    if (fast) {
      const double2* dA = sa.sp.dA;
      const double* sA = sa.sp.sA;
      const double* gz = has1 ? g1 : g0;  // a valid address for the absent partner line
      auto fil = [&](double2 d, double sv, double mu) {  // conj(d) / (|d|^2 + mu s^2)
        const double r = rcp_pos((d.x * d.x + d.y * d.y) + mu * sv * sv);
        return make_double2(d.x * r, -d.y * r);
      };
      {
        double2 bd[kHoMax];
        double bs[kHoMax], c0[kHoMax], c1[kHoMax];
#pragma unroll
        for (int l = 0; l < kHoMax; ++l) {
          const int lc = l < hk ? l : 0, e = ho_coef_elem(ax, lc);
          bd[l] = __ldg(dA + e);
          bs[l] = sA ? __ldg(sA + e) : 1.0;
          c0[l] = __ldcs(g0 + lc);
          c1[l] = __ldcs(gz + lc);
        }
#pragma unroll
        for (int l = 0; l < kHoMax; ++l) {
          ua0[l] = l < hk ? c0[l] * fil(bd[l], bs[l], mu0).x : 0.0;
          ua1[l] = (l < hk && has1) ? c1[l] * fil(bd[l], bs[l], mu1).x : 0.0;
        }
      }
#pragma unroll
      for (int b = 0; b < kMixK / 4; ++b) {
        double2 c0[4], c1[4], d[4];
        double sv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kq = threadIdx.x + (4 * b + u) * kMixNT;
          const int kk = kq <= h ? kq : h;
          // (Re, Im) at [hk - 1 + 2 kk, hk + 2 kk] (16-byte aligned); X_0 is real, at [hk]
          c0[u] = __ldcs(reinterpret_cast<const double2*>(g0 + hk - 1 + 2 * kk));
          c1[u] = __ldcs(reinterpret_cast<const double2*>(gz + hk - 1 + 2 * kk));
          d[u] = __ldg(dA + kl + kk);
          sv[u] = sA ? __ldg(sA + kl + kk) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kq = threadIdx.x + (4 * b + u) * kMixNT;
          double2 X0 = c0[u], X1 = has1 ? c1[u] : czero();
          if (kq == 0) {
            X0 = make_double2(X0.y, 0.0);
            X1 = make_double2(X1.y, 0.0);
          }
          X0 = cmul(X0, fil(d[u], sv[u], mu0));
          X1 = cmul(X1, fil(d[u], sv[u], mu1));
          if (kq <= h) {
            nzb0 |= __double_as_longlong(X0.x) | __double_as_longlong(X0.y);
            nzb1 |= __double_as_longlong(X1.x) | __double_as_longlong(X1.y);
            // F^H v = conj(F conj v), v = X0 + i X1 (natural order input)
            x[kq] = make_double2(X0.x - X1.y, -(X0.y + X1.x));
            if (kq) x[m - kq] = make_double2(X0.x + X1.y, X0.y - X1.x);
          }
        }
      }
    } else {
#pragma unroll
      for (int l = 0; l < kHoMax; ++l) {
        ua0[l] = l < hk ? f0(ho_coef_elem(ax, l), make_double2(ld0(l), 0.0)).x : 0.0;
        ua1[l] = l < hk ? f1(ho_coef_elem(ax, l), make_double2(ld1(l), 0.0)).x : 0.0;
      }
#pragma unroll 4
      for (int kk = threadIdx.x; kk <= h; kk += kMixNT) {
        const int e = kl + kk;
        double2 X0, X1;
        if (kk == 0) {
          X0 = make_double2(ld0(hk), 0.0);
          X1 = make_double2(ld1(hk), 0.0);
        } else {
          X0 = ldp0(hk + 2 * kk - 1);
          X1 = ldp1(hk + 2 * kk - 1);
        }
        X0 = f0(e, X0);
        X1 = f1(e, X1);
        nzb0 |= __double_as_longlong(X0.x) | __double_as_longlong(X0.y);
        nzb1 |= __double_as_longlong(X1.x) | __double_as_longlong(X1.y);
        // F^H v = conj(F conj v), v = X0 + i X1 (natural order input)
        x[kk] = make_double2(X0.x - X1.y, -(X0.y + X1.x));
        if (kk) x[m - kk] = make_double2(X0.x + X1.y, X0.y - X1.x);
      }
    }
    zf_add(zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    __syncthreads();
    mix_dft(x, ax, tw, kMixNT);
    mix_prefetch_pair(io.in, io.gi, q + gridDim.x, ax.n);

    const Cubic p0 = ho_cubic(ax, ua0), p1 = ho_cubic(ax, ua1);
    const long long eso = io.go.elem_stride;
    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    const int nz = zf_take(zf, it);
    const double s0 = (nz & 1) ? isq : 0.0, s1 = (nz & 2) ? -isq : 0.0;
    const bool tout = mix_out_staged(ax, o0, o1, eso);
    if (tout) {  // lines assembled in x, two bulk stores (see k_psynth)
      double y0r[kMixP], y1r[kMixP];
#pragma unroll
      for (int t = 0; t < kMixP; ++t) {  // branch-free: the slots interleave
        const int p = threadIdx.x + t * kMixNT;
        const double2 z = x[perm[p < m ? p : m - 1]];
        y0r[t] = z.x * s0;
        y1r[t] = z.y * s1;
      }
      // border element bord[l] repeats the interior sample wrap[l] (thread l)
      double yb0 = 0.0, yb1 = 0.0;
      if (threadIdx.x < hk) {
        const double2 z = x[perm[ax.wrap[threadIdx.x]]];
        yb0 = z.x * s0;
        yb1 = z.y * s1;
      }
      __syncthreads();  // every sample has been read
      double* lineA = reinterpret_cast<double*>(x);
      double* lineB = lineA + n;
#pragma unroll
      for (int t = 0; t < kMixP; ++t) {
        const int p = threadIdx.x + t * kMixNT;
        const double tt = fma((double)(t * kMixNT), ax.ho_ta, tt0);
        const double r0 = y0r[t] + p0(tt), r1 = y1r[t] + p1(tt);
        if (p < m) {
          lineA[kl + p] = r0;
          lineB[kl + p] = r1;
        }
      }
      if (threadIdx.x < hk) {
        const int eb = ax.bord[threadIdx.x];
        const double tb = fma((double)eb, ax.ho_ta, ax.ho_tb);
        lineA[eb] = yb0 + p0(tb);
        lineB[eb] = yb1 + p1(tb);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    } else
#pragma unroll 4
    for (int p = threadIdx.x; p < m; p += kMixNT) {
      const double2 z = x[perm[p]];
      const double y0 = z.x * s0, y1 = z.y * s1;
      const int e = kl + p;
      const double t = fma((double)e, ax.ho_ta, ax.ho_tb);
      __stcs(o0 + e * eso, y0 + p0(t));
      if (o1) __stcs(o1 + e * eso, y1 + p1(t));
#pragma unroll
      for (int l = 0; l < kHoMax; ++l)
        if (l < hk && ax.wrap[l] == p) {
          const int eb = ax.bord[l];
          const double tb = fma((double)eb, ax.ho_ta, ax.ho_tb);
          o0[eb * eso] = y0 + p0(tb);
          if (o1) o1[eb * eso] = y1 + p1(tb);
        }
    }
    __syncthreads();
    if (tout && threadIdx.x == 0) {
      bulk_s2g(o0, x, (uint32_t)n * 8);
      if (o1) bulk_s2g(o1, reinterpret_cast<double*>(x) + n, (uint32_t)n * 8);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

}  // namespace fdb
