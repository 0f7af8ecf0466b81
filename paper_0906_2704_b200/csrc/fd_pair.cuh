// Two real lines per complex Bluestein DFT of the full interior length m:
// the real-data path of the higher-order borders (AxisDev::hob), whose
// interior length m = n - d is odd for even n (d = 1, 3), so the half-length
// R2C split of k_ranalyze / k_rsynth does not apply.
//
//   analyze    (oracle ho_analyze):  a = S^-1 (y[bord] - y[kl + wrap]) per line,
//              z = (y0_I - P_I a0) + i (y1_I - P_I a1),  Z = DFT_m(z),
//              X0_k = (Z_k + conj Z_{m-k}) / 2,  X1_k = (Z_k - conj Z_{m-k}) / 2i
//   synthesize (oracle ho_synthesize): v = X0 + i X1 over all m (X_{m-k} = conj X_k),
//              y0 + i y1 = F^H v,  y_I += P_I a,  y[bord] = y[kl + wrap] + P[bord] a
//
// Persistent CTAs (one per SM at m ~ 4096: 139 KB buffer + 64 KB chirp),
// each streaming line pairs; the next pair's 2n doubles are bulk-copied (TMA
// engine, mbarrier completion) into the upper half of the FFT buffer, free
// from the end of the convolution to the next load phase.
//
// Coefficients of real data are stored Hermitian-packed, n doubles per line
// (io.pack == 2):  [a_0 .. a_{k-1}, X_0, Re X_1, Im X_1, .., Re X_h, Im X_h],
// h = (m-1)/2; the GCV weights |ghat|^2 (Hermitian pairs pre-summed, reduced
// order of build_pairs) and their TF32 screen tiles are written alongside.
// The border columns enter as one cubic per line in t_e = ho_ta e + ho_tb
// (the Legendre closed form of the P table).
#pragma once

namespace fdb {

// SYN: the synthesis kernel (filter fused into its load phase) runs 512
// threads at M = 8192; the analysis kernel runs 256 threads with up to 255
// registers (two radix-16 items per thread per pass) -- measured faster for
// analyze (4.45 -> 4.31 ms at config 1), much slower for synthesize
template <int LOGM, bool SYN = false>
struct PairShape {
  static constexpr int M = 1 << LOGM;
  static constexpr int NT = M / 16 >= (SYN ? 512 : 256) ? (SYN ? 512 : 256)
                                                         : (M / 16 <= 64 ? 64 : M / 16);
  // LOGM = 1 (mod 4): the Bluestein pass sequence starts with a radix-2 DIF
  // stage whose upper input half is zero padding (m <= M/2), i.e. the stage is
  // (v, v W^j): the load phase writes both halves itself, and the matching
  // last DIT stage is only needed on the lower half, so it is folded into the
  // post phase -- two full shared-memory passes saved per line pair.
  static constexpr bool FOLD = (LOGM % 4 == 1) && LOGM >= 9;
  static constexpr int HM = M / 2;
  static constexpr int JS = (HM + NT - 1) / NT;  // register slots per thread (j < HM)
};

// tw(j) at j = j0 + t NT for the FOLD phases: with NT a multiple of the lo
// table's length the lo factor is the same for every t, so each thread loads
// it once and the per-element lookup is one (warp-broadcast) hi entry
template <int LOGM>
struct FoldTw {
  static constexpr int LOB = FftShape<LOGM>::LOB;
  const double2* hi;
  double2 lo;
  __device__ __forceinline__ FoldTw(const TwSm& tw, int j0)
      : hi(tw.hi), lo(tw.lo[j0 & ((1 << LOB) - 1)]) {}
  __device__ __forceinline__ double2 operator()(int j) const { return cmul(hi[j >> LOB], lo); }
};

// the Bluestein convolution of the pair kernels; with FOLD the buffer must
// hold both halves of the first DIF stage already, and on return the lower
// half [0, m) holds the result
// Optional phase timing of the pair kernels (-DFD_PHASE_CLOCKS): thread 0 of
// every CTA adds the SM clocks between phase marks, g_pair_clocks[kernel][phase]
// (kernel: 0 k_panalyze, 1 k_psynth, 2 k_panalyze_e, 3 k_psynth_e)
#ifdef FD_PHASE_CLOCKS
__device__ unsigned long long g_pair_clocks[4][12];
#define FD_PCLK_INIT() long long pclk_ = clock64()
#define FD_PCLK(k, i)                                                                 \
  do {                                                                                \
    const long long now_ = clock64();                                                 \
    if (threadIdx.x == 0) atomicAdd(&g_pair_clocks[k][i], (unsigned long long)(now_ - pclk_)); \
    pclk_ = now_;                                                                     \
  } while (0)
#else
#define FD_PCLK_INIT()
#define FD_PCLK(k, i)
#endif

// bluestein_rec<LOGM, P, S, NT> with phase marks after every pass (marks base + 0 ..)
template <int LOGM, int P, int S, int NT, int KERN, int BASE, int GRP = 0>
__device__ __forceinline__ void bluestein_rec_clk(double2* x, const double2* bhat, const TwSm& tw,
                                                  int nvalid, long long& pclk_) {
#ifdef FD_PHASE_CLOCKS
  using F = FftShape<LOGM, NT>;
  if constexpr (P == F::NP - 1) {
    mid_pass_t<LOGM, false, NT>(x, bhat, nvalid);
    pass_sync<GRP>();
    FD_PCLK(KERN, BASE);
  } else {
    dif_pass_t<LOGM, 4, S, false, NT, false>(x, tw, nvalid);
    pass_sync<GRP>();
    FD_PCLK(KERN, BASE);
    bluestein_rec_clk<LOGM, P + 1, (S >> 4), NT, KERN, BASE + 1, GRP>(x, bhat, tw, nvalid, pclk_);
    dit_pass_t<LOGM, 4, S, NT, false>(x, tw);
    pass_sync<GRP>();
    FD_PCLK(KERN, BASE + 2 * (F::NP - 1 - P));
  }
#endif
}

// experiment knob: SM clocks the upper-half thread group waits before its
// passes (FASTDEBLUR_PAIR_SKEW), to start the two groups out of phase
__device__ int g_pair_skew = 1200;

// the folded convolution's last step: lower half += conj(W^k) upper half, k < m
template <int LOGM, int NT>
__device__ __forceinline__ void pair_combine(double2* x, const TwSm& tw, int m) {
  using S = PairShape<LOGM>;
  const FoldTw<LOGM> ft(tw, threadIdx.x);
  constexpr int JS = (S::HM + NT - 1) / NT;
#pragma unroll
  for (int t = 0; t < JS; ++t) {  // clamped, branch-free: the slots' loads batch
    const int k = threadIdx.x + t * NT;
    const int kc = k < m ? k : m - 1;
    const double2 r = cadd(x[pidx(kc)], cmulc(x[pidx(kc + S::HM)], ft(kc)));
    if (k < m) x[pidx(k)] = r;
  }
  __syncthreads();
}

// SKEW: what the upper half's thread group does before its passes while the
// lower half's group starts -- work worth ~1200 SM clocks (deferred stores of
// the previous pair), or a spin of g_pair_skew clocks
struct SkewSpin {
  __device__ __forceinline__ void operator()() const {
    const long long t0 = clock64();
    const int skew = g_pair_skew;
    while (clock64() - t0 < skew) {}
  }
};

struct SkewNone {
  __device__ __forceinline__ void operator()() const {}
};
// TAIL: what the lower half's group does after its passes, while the (late)
// upper group finishes
template <int LOGM, int NT, int KERN = 0, class SKEW = SkewSpin, class TAIL = SkewNone>
__device__ __forceinline__ void pair_conv(double2* x, const FftTables& T, const TwSm& tw, int m,
                                          long long& pclk_, SKEW skew = SKEW(),
                                          TAIL tail = TAIL()) {
  using S = PairShape<LOGM>;
  if constexpr (S::FOLD) {
    static_assert(NT % (1 << FoldTw<LOGM>::LOB) == 0, "FoldTw needs NT % lo length == 0");
    // NT == M/16: threads [0, NT/2) own the lower half's items in every pass,
    // [NT/2, NT) the upper half's -- the halves synchronise separately
    constexpr int GRP = (NT == S::M / 16 && NT >= 64) ? NT / 2 : 0;
    if constexpr (GRP != 0) {
      if (threadIdx.x >= GRP) skew();
    }
#ifdef FD_PHASE_CLOCKS
    if constexpr (LOGM == 13) {
      bluestein_rec_clk<LOGM, 1, S::HM, NT, KERN, 2, GRP>(x, T.bhat, tw, S::M, pclk_);
      if constexpr (GRP != 0) {
        if (threadIdx.x < GRP) tail();
        __syncthreads();
      }
      pair_combine<LOGM, NT>(x, tw, m);
      FD_PCLK(KERN, 7);
      return;
    }
#endif
    bluestein_rec<LOGM, 1, S::HM, NT, false, GRP>(x, T.bhat, tw, S::M);
    if constexpr (GRP != 0) {
      if (threadIdx.x < GRP) tail();
      __syncthreads();
    }
    pair_combine<LOGM, NT>(x, tw, m);
  } else {
    bluestein_t<LOGM, NT>(x, T, tw, m);
  }
}

// Shared-memory slots (double2) of the pair kernels:
//   FFT buffer | twiddles | chirp c_0 .. c_h | mbarrier + zero-line flags |
//   border spectral values (8) | synthesis filter table: d (h + 1), s ((h + 2) / 2)
// Only half the chirp is stored: c_{m-j} = e^{-i pi (m-j)^2/m} = (-1)^m c_j = -c_j
// for the odd m of this path.  The freed space holds the 1D filter's spectral
// table (k_psynth), which was re-read from L2 for every line pair.
__host__ __device__ __forceinline__ int pair_cs_slots(int m) { return (m - 1) / 2 + 1; }
__host__ __device__ __forceinline__ int pair_slots(int M, int m) {
  return pidx(M) + 1 + kTwSlots + pair_cs_slots(m) + 1;
}
__host__ __device__ __forceinline__ int pair_smem_slots(int M, int m) {
  return pair_slots(M, m) + 8 + pair_cs_slots(m) + (pair_cs_slots(m) + 1) / 2;
}
struct HalfChirp {
  const double2* cs;
  int m, h;
  __device__ __forceinline__ double2 operator()(int j) const {
    const double2 c = cs[j <= h ? j : m - j];
    return j <= h ? c : make_double2(-c.x, -c.y);
  }
};

// sum_l a_l P_l(t) as a cubic in t (P_1 = t, P_2 = (3t^2-1)/2, P_3 = (5t^3-3t)/2)
struct Cubic {
  double c0, c1, c2, c3;
  __device__ __forceinline__ double operator()(double t) const {
    return fma(fma(fma(c3, t, c2), t, c1), t, c0);
  }
};
__device__ __forceinline__ Cubic ho_cubic(const AxisDev& ax, const double (&a)[kHoMax]) {
  const double b0 = ax.hk > 0 ? a[0] * ax.ho_s[0] : 0.0;
  const double b1 = ax.hk > 1 ? a[1] * ax.ho_s[1] : 0.0;
  const double b2 = ax.hk > 2 ? a[2] * ax.ho_s[2] : 0.0;
  return Cubic{-0.5 * b1, b0 - 1.5 * b2, 1.5 * b1, 2.5 * b2};
}

// a = sinv (y[bord] - y[kl + wrap]) of one real line
template <class LD>
__device__ __forceinline__ void ho_amps_real(const AxisDev& ax, LD ld, double (&a)[kHoMax]) {
  double r[kHoMax];
#pragma unroll
  for (int l = 0; l < kHoMax; ++l) r[l] = l < ax.hk ? ld(ax.bord[l]) - ld(ax.kl + ax.wrap[l]) : 0.0;
#pragma unroll
  for (int l = 0; l < kHoMax; ++l) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kHoMax; ++q) v += ax.sinv[l * kHoMax + q] * r[q];
    a[l] = v;
  }
}

// Zero-line flags of the line-pair kernels: two ints in shared memory, one per
// parity of the CTA's pair counter.  Warps OR their "line l has a nonzero
// input" bits in during the load phase (before an existing barrier); the post
// phase reads them and thread 0 clears the other parity's word for the next
// pair (the end-of-pair barrier orders that against its writers).
__device__ __forceinline__ void zf_add(int* zf, int it, int nzl) {
  nzl = (int)__reduce_or_sync(0xffffffffu, (unsigned)nzl);
  if ((threadIdx.x & 31) == 0 && nzl) atomicOr(&zf[it & 1], nzl);
}
__device__ __forceinline__ int zf_take(int* zf, int it) {
  const int v = zf[it & 1];
  if (threadIdx.x == 0) zf[(it + 1) & 1] = 0;
  return v;
}

// all border amplitudes of a line exactly zero
__device__ __forceinline__ bool ho_zero(const double (&a)[kHoMax]) {
  bool z = true;
#pragma unroll
  for (int l = 0; l < kHoMax; ++l) z = z && a[l] == 0.0;
  return z;
}

// reduced GCV index of border amplitude l (build_pairs: left singles, interior
// groups 0..h, right singles)
__device__ __forceinline__ int ho_wred(const AxisDev& ax, int l, int h) {
  return l < ax.kl ? l : ax.kl + h + 1 + (l - ax.kl);
}

// Output lines leave through the bulk-copy engine (shared -> global): an SM's
// own store path sustains only ~14 B/clock (measured: the direct stores of the
// post phases took 24 % of k_panalyze, 13 % of k_psynth), while a bulk store
// drains in the background of the next pair's load phase.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all committed bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// the staged output lines (2 n doubles at the start of the FFT buffer) need
// 16-byte aligned, unit-stride global lines of even length
__device__ __forceinline__ bool pair_out_staged(const double* o0, const double* o1, int n,
                                                long long eso) {
  return eso == 1 && !(n & 1) && (reinterpret_cast<uintptr_t>(o0) & 15) == 0 &&
         (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
}

struct PairStage {
  double* buf;
  uint64_t* bar;
  bool on;
  uint32_t phase;
};

// staging needs contiguous lines (item stride n, unit element stride) and the
// two lines to fit between the interior and the end of the buffer
__device__ __forceinline__ PairStage pair_stage_init(double2* x, int M, int m, int n,
                                                     const Lines& g, uint64_t* bar) {
  PairStage s;
  s.buf = reinterpret_cast<double*>(x + pidx(m) + 1);
  s.bar = bar;
  s.phase = 0;
  s.on = g.elem_stride == 1 && g.per_item == 1 && g.item_stride == n &&
         (long long)(pidx(M) - pidx(m) - 1) >= (long long)n;
  if (threadIdx.x == 0 && s.on) {
    mbar_init(s.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  return s;
}
__device__ __forceinline__ bool pair_staged(const PairStage& s, const void* base, const Lines& g,
                                            int q) {
  if (!s.on || 2 * q + 1 >= g.count) return false;  // full pairs only
  const double* src = reinterpret_cast<const double*>(base) + line_offset(g, 2 * q);
  return (reinterpret_cast<uintptr_t>(src) & 15) == 0;
}
__device__ __forceinline__ void pair_issue(PairStage& s, const void* base, const Lines& g, int q,
                                           int n) {
  if (!pair_staged(s, base, g, q)) return;
  const double* src = reinterpret_cast<const double*>(base) + line_offset(g, 2 * q);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(s.bar, (uint32_t)n * 16);
  bulk_g2s(s.buf, src, (uint32_t)n * 16, s.bar);
}

// WIDE: 512 threads x 128 registers at M = 8192 (one radix-16 item per thread
// per pass, the two halves' thread groups synchronising separately) instead of
// 256 x 255
template <int LOGM, bool WIDE = false>
__global__ void __launch_bounds__(PairShape<LOGM, WIDE>::NT, 1) k_panalyze(AxisDev ax, LineIO io) {
  constexpr int NT = PairShape<LOGM, WIDE>::NT, M = 1 << LOGM;
  extern __shared__ double2 sm[];
  const FftTables& T = ax.fft;
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  double2* slots = sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(slots, T);
  double2* cs = slots + kTwSlots;
  for (int j = threadIdx.x; j <= h; j += NT) cs[j] = T.chirp[j];
  const HalfChirp chirp{cs, m, h};
  PairStage stg = pair_stage_init(x, M, m, n, io.gi,
                                  reinterpret_cast<uint64_t*>(sm + pair_slots(M, m) - 1));
  int* zf = reinterpret_cast<int*>(sm + pair_slots(M, m) - 1) + 2;
  if (threadIdx.x < 2) zf[threadIdx.x] = 0;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, blockIdx.x, n);
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const long long es = io.gi.elem_stride;
  const double isq = ax.inv_sqrt_m;
  const long long nkb32 = io.wstride >> 5;
  // t_e = ho_ta e + ho_tb at this thread's first element; slot t adds t NT ho_ta
  const double tt0 = fma((double)(kl + (int)threadIdx.x), ax.ho_ta, ax.ho_tb);
#ifdef FD_PHASE_CLOCKS
  long long pclk_ = clock64();
#else
  long long pclk_ = 0;
#endif
  // TF32 tiles of a pair's weight rows, from the rows staged in shared memory
  // (wA, wB below): task c = chunk c >> 1 (4 elements) of line l0 + (c & 1)
  using PSK = PairShape<LOGM, WIDE>;
  constexpr int GRPK = (PSK::FOLD && NT == M / 16 && NT >= 64) ? NT / 2 : 0;  // pair_conv's groups
  auto tf32_rows = [&](int l0p, int first, int step, int c0, int c1) {
    const double* wa = reinterpret_cast<const double*>(sm + pair_slots(M, m) + 8);
    const double* wb = wa + io.wstride;
    float* th = io.wout32 + tc_tile_index(l0p, 0, kTcBM, nkb32);
    float* tl = io.wout32lo + tc_tile_index(l0p, 0, kTcBM, nkb32);
    const bool two = l0p + 1 < count;
    for (int c = c0 + first; c < c1; c += step) {
      const int row = c & 1, i = (c >> 1) * 4;
      if (row && !two) continue;
      const double2* src = reinterpret_cast<const double2*>((row ? wb : wa) + i);
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
  };
  int tf_l0 = -1;  // pair whose tiles are still to be written
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const bool st = pair_staged(stg, io.in, io.gi, q);
    if (st) {
      mbar_wait(stg.bar, stg.phase);
      stg.phase ^= 1;
    }
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    const double* s0 = stg.buf;
    const double* s1 = stg.buf + n;
    double a0[kHoMax], a1[kHoMax];
    Cubic p0, p1;
    using PS = PairShape<LOGM, WIDE>;
    double2 vr[PS::FOLD ? PS::JS : 1];
    long long nzb0 = 0, nzb1 = 0;  // OR of the bit patterns of line 0 / 1 (-0.0 counts as nonzero)
    auto load_phase = [&](auto ld0, auto ld1) {
      ho_amps_real(ax, ld0, a0);
      ho_amps_real(ax, ld1, a1);
      p0 = ho_cubic(ax, a0);
      p1 = ho_cubic(ax, a1);
      auto val = [&](int j, double t) {
        const int e = kl + j;
        const double y0 = ld0(e), y1 = ld1(e);
        nzb0 |= __double_as_longlong(y0);  // integer pipe: the fp64 pipe is the bound
        nzb1 |= __double_as_longlong(y1);
        return cmul(make_double2(y0 - p0(t), y1 - p1(t)), chirp(j));
      };
      if constexpr (PS::FOLD) {
#pragma unroll
        for (int t = 0; t < PS::JS; ++t) {
          // branch-free (index clamped, result selected): the slots' loads
          // and arithmetic interleave instead of running slot after slot
          const int j = threadIdx.x + t * NT;
          const double2 vj = val(j < m ? j : m - 1, fma((double)(t * NT), ax.ho_ta, tt0));
          vr[t] = j < m ? vj : czero();
        }
      } else {
#pragma unroll 4
        for (int j = threadIdx.x; j < m; j += NT)
          x[pidx(j)] = val(j, fma((double)(kl + j), ax.ho_ta, ax.ho_tb));
      }
    };
    if (st)
      load_phase([&](int e) { return s0[e]; }, [&](int e) { return s1[e]; });
    else
      load_phase([&](int e) { return __ldg(g0 + e * es); },
                 [&](int e) { return has1 ? __ldg(g1 + e * es) : 0.0; });
    // an all-zero line gets exactly zero coefficients (its partner's DFT
    // round-off would otherwise leak into it through the Hermitian split)
    zf_add(zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    if (PS::FOLD && threadIdx.x == 0) bulk_wait_read();  // the previous pair's output lines
    __syncthreads();
    FD_PCLK(0, 0);
    if constexpr (PS::FOLD) {  // first DIF stage (v, v W^j), staged input consumed
      const FoldTw<LOGM> ft(tw, threadIdx.x);
#pragma unroll
      for (int t = 0; t < PS::JS; ++t) {
        const int j = threadIdx.x + t * NT;
        if (j < PS::HM) {
          x[pidx(j)] = vr[t];
          x[pidx(j + PS::HM)] = cmul(vr[t], ft(j));
        }
      }
      __syncthreads();
      FD_PCLK(0, 1);
    }
    pair_conv<LOGM, NT, 0>(x, T, tw, m, pclk_, [&] {
      if (tf_l0 >= 0) {
        const int ntask = (int)(io.wstride >> 1);
        tf32_rows(tf_l0, (int)threadIdx.x - GRPK, GRPK, (ntask / 2) & ~1, ntask);
      } else {
        SkewSpin()();
      }
    }, [&] {
      if (tf_l0 >= 0) {
        const int ntask = (int)(io.wstride >> 1);
        tf32_rows(tf_l0, (int)threadIdx.x, GRPK, 0, (ntask / 2) & ~1);
      }
    });
    tf_l0 = -1;
    // the post phase reads [0, m) only: stage the next pair behind it
    if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, q + gridDim.x, n);

    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    double* w0 = io.wout ? io.wout + (long long)l0 * io.wstride : nullptr;
    // weight i of both lines: fp64 rows, and their TF32 split in the screen's
    // tile layout (tc_tile_index = row part + element part; the pair's rows
    // l0, l0 + 1 are adjacent 16-byte chunks, 4 floats apart)
    float* t32h = io.wout32 ? io.wout32 + tc_tile_index(l0, 0, kTcBM, nkb32) : nullptr;
    float* t32l = io.wout32 ? io.wout32lo + tc_tile_index(l0, 0, kTcBM, nkb32) : nullptr;
    auto wset2 = [&](int i, double v0, double v1) {
      w0[i] = v0;
      if (has1) w0[io.wstride + i] = v1;
      if (t32h) {
        const int eo = (i >> 5) * (kTcBM * 32) + ((i & 31) >> 2) * (kTcBM * 4) + (i & 3);
        float hi, lo;
        tf32_split(v0, hi, lo);
        t32h[eo] = hi;
        t32l[eo] = lo;
        if (has1) {
          tf32_split(v1, hi, lo);
          t32h[eo + 4] = hi;
          t32l[eo + 4] = lo;
        }
      }
    };
    const int nz = zf_take(zf, it);
    const bool z0 = !(nz & 1) && ho_zero(a0), z1 = !(nz & 2) && ho_zero(a1);
    // FOLD sizes: the packed coefficient lines are assembled in shared memory
    // (the buffer's lower part, free once every thread has read its Z_k) and
    // leave as two bulk stores; only the GCV weights take the store path
    // kk <= h slots: M >= 2 m - 1 and m odd give h = (m - 1) / 2 <= HM / 2 - 1
    constexpr int KSA = PS::FOLD ? (PS::HM / 2 + NT - 1) / NT : 1;
    const bool tout = PS::FOLD && pair_out_staged(o0, o1, n, io.go.elem_stride) && (hk & 1);
    // ... and so do the fp64 weight rows (staged in the area the synthesis
    // kernel keeps its spectral table in); their TF32 tiles are written
    // chunk-wise from the staged rows: one lane per (16-byte chunk, line), so a
    // store instruction touches 16 lines instead of the 32 that per-element
    // 4-byte stores did (~2 clocks per line touched: 11 % of the kernel)
    double* wA = reinterpret_cast<double*>(sm + pair_slots(M, m) + 8);
    double* wB = wA + io.wstride;
    const bool wst = tout && w0 && (io.wstride & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(w0) & 15) == 0 &&
                     2 * io.wstride <= 2 * (pair_cs_slots(m) + (pair_cs_slots(m) + 1) / 2);
    if (tout) {
      double2 X0r[KSA], X1r[KSA];
#pragma unroll
      for (int t = 0; t < KSA; ++t) {
        const int kq = threadIdx.x + t * NT;
        const int kk = kq <= h ? kq : h;  // clamped: branch-free slots interleave
        const double2 ck = cs[kk];  // c_{m-kk} = -c_kk
        const double2 Zk = cmul(x[pidx(kk)], ck);
        const double2 Zm = cmul(x[pidx(m - kk)], make_double2(-ck.x, -ck.y));
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
            wset2(kl + kk, v0, v1);
          }
        }
      }
      if (wst) {
        if (threadIdx.x < hk) {
          const int l = threadIdx.x, i = ho_wred(ax, l, h);
          wA[i] = a0[l] * a0[l];
          wB[i] = a1[l] * a1[l];
        }
        for (int i = (int)io.wn + threadIdx.x; i < (int)io.wstride; i += NT) wA[i] = wB[i] = 0.0;
      }
      __syncthreads();  // every Z_k has been read; the weight rows are complete
      double* lineA = reinterpret_cast<double*>(x);
      double* lineB = lineA + n;
#pragma unroll
      for (int t = 0; t < KSA; ++t) {
        const int kk = threadIdx.x + t * NT;
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
      if (wst && t32h) {
        // with thread groups, the upper group writes the second half of the
        // tiles in the next pair's skew slot (~1200 clocks of store work
        // instead of a spin)
        // with thread groups the tiles are written during the NEXT pair's
        // convolution: the second half by the upper group in its skew slot
        // (work instead of a spin), the first half by the lower group while it
        // waits for the upper one to finish
        if constexpr (GRPK != 0) {
          tf_l0 = l0;
        } else {
          tf32_rows(l0, threadIdx.x, NT, 0, (int)(io.wstride >> 1));
        }
      }
    } else
    for (int kk = threadIdx.x; kk <= h; kk += NT) {
      const double2 ck = cs[kk];  // c_{m-kk} = -c_kk
      const double2 Zk = cmul(x[pidx(kk)], ck);
      const double2 Zc = kk ? cmul(x[pidx(m - kk)], make_double2(-ck.x, -ck.y)) : Zk;
      const double2 D = csub(Zk, cconj(Zc));
      const double2 X0 = z0 ? czero() : cscale(cadd(Zk, cconj(Zc)), 0.5 * isq);
      const double2 X1 = z1 ? czero() : make_double2(0.5 * isq * D.y, -0.5 * isq * D.x);
      if (kk == 0) {
        o0[hk] = X0.x;
        if (o1) o1[hk] = X1.x;
      } else {
        o0[hk + 2 * kk - 1] = X0.x;
        o0[hk + 2 * kk] = X0.y;
        if (o1) {
          o1[hk + 2 * kk - 1] = X1.x;
          o1[hk + 2 * kk] = X1.y;
        }
      }
      if (w0) {
        const double f = kk ? 2.0 : 1.0;  // |X_k|^2 + |X_{m-k}|^2
        wset2(kl + kk, f * (X0.x * X0.x + X0.y * X0.y), f * (X1.x * X1.x + X1.y * X1.y));
      }
    }
    if (threadIdx.x < hk) {
      const int l = threadIdx.x;
      if (!tout) {
        o0[l] = a0[l];
        if (o1) o1[l] = a1[l];
      }
      if (w0 && !wst) wset2(ho_wred(ax, l, h), a0[l] * a0[l], a1[l] * a1[l]);
    }
    if (w0 && !wst)
      for (int i = (int)io.wn + threadIdx.x; i < (int)io.wstride; i += NT) wset2(i, 0.0, 0.0);
    __syncthreads();  // x is reused by the next pair
    if (tout && threadIdx.x == 0) {
      bulk_s2g(o0, x, (uint32_t)n * 8);
      if (o1) bulk_s2g(o1, reinterpret_cast<double*>(x) + n, (uint32_t)n * 8);
      if (wst) {
        bulk_s2g(w0, wA, (uint32_t)io.wstride * 8);
        if (has1) bulk_s2g(w0 + io.wstride, wB, (uint32_t)io.wstride * 8);
      }
      bulk_commit();
    }
    FD_PCLK(0, 8);
  }
  if (tf_l0 >= 0)  // the last pair's deferred tiles
    tf32_rows(tf_l0, threadIdx.x, NT, 0, (int)(io.wstride >> 1));
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

template <int LOGM>
__global__ void __launch_bounds__(PairShape<LOGM, true>::NT, 1) k_psynth(AxisDev ax, LineIO io,
                                                                   SynthArgs sa) {
  constexpr int NT = PairShape<LOGM, true>::NT, M = 1 << LOGM;
  extern __shared__ double2 sm[];
  const FftTables& T = ax.fft;
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  double2* slots = sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(slots, T);
  double2* cs = slots + kTwSlots;
  for (int j = threadIdx.x; j <= h; j += NT) cs[j] = T.chirp[j];
  const HalfChirp chirp{cs, m, h};
  PairStage stg = pair_stage_init(x, M, m, n, io.gi,
                                  reinterpret_cast<uint64_t*>(sm + pair_slots(M, m) - 1));
  int* zf = reinterpret_cast<int*>(sm + pair_slots(M, m) - 1) + 2;
  if (threadIdx.x < 2) zf[threadIdx.x] = 0;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, blockIdx.x, n);
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
  using PS = PairShape<LOGM, true>;
  // kk slots: M >= 2 m - 1 and m odd give h = (m - 1) / 2 <= HM / 2 - 1
  constexpr int KS = PS::FOLD ? (PS::HM / 2 + NT - 1) / NT : 1;
  // 1D filter (one spectral table for every line): the table lives in shared
  // memory -- the per-pair reads from L2 were latency bound (27 % of the kernel
  // at config 1); the border coefficients' entries sit in the extras slots
  const bool spsm = sa.mode == 1 && sa.sp.mode == 1 && ax.cplx;
  double2* bsp = sm + pair_slots(M, m);        // [l] = d of border coefficient l, [4 + l].x = s
  double2* spd = bsp + 8;                      // d of interior coefficient kk
  double* sps = reinterpret_cast<double*>(spd + pair_cs_slots(m));
  if (spsm) {
    for (int kk = threadIdx.x; kk <= h; kk += NT) {
      spd[kk] = __ldg(&sa.sp.dA[kl + kk]);
      sps[kk] = sa.sp.sA ? __ldg(&sa.sp.sA[kl + kk]) : 1.0;
    }
    if (threadIdx.x < hk) {
      const int e = ho_coef_elem(ax, threadIdx.x);
      bsp[threadIdx.x] = __ldg(&sa.sp.dA[e]);
      bsp[4 + threadIdx.x].x = sa.sp.sA ? __ldg(&sa.sp.sA[e]) : 1.0;
    }
    __syncthreads();
  }
  const double tt0 = fma((double)(kl + (int)threadIdx.x), ax.ho_ta, ax.ho_tb);
  // regularisation parameters of the next pair, read one pair ahead
  auto pair_mu = [&](int q, double& m0, double& m1) {
    m0 = m1 = 0.0;
    if (q < npairs) {
      m0 = line_mu(sa, io.gi, 2 * q);
      m1 = 2 * q + 1 < count ? line_mu(sa, io.gi, 2 * q + 1) : m0;
    }
  };
  double mu0n, mu1n;
  pair_mu(blockIdx.x, mu0n, mu1n);
#ifdef FD_PHASE_CLOCKS
  long long pclk_ = clock64();
#else
  long long pclk_ = 0;
#endif
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const bool st = pair_staged(stg, io.in, io.gi, q);
    if (st) {
      mbar_wait(stg.bar, stg.phase);
      stg.phase ^= 1;
    }
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    const double mu0 = mu0n, mu1 = mu1n;
    pair_mu(q + gridDim.x, mu0n, mu1n);
    auto f0 = [&](int e, double2 c) { return coeff_filter_fast(ax, sa, io.gi, l0, e, c, mu0); };
    auto f1 = [&](int e, double2 c) {
      return has1 ? coeff_filter_fast(ax, sa, io.gi, l0 + 1, e, c, mu1) : czero();
    };
    double ua0[kHoMax], ua1[kHoMax];
    double2 vk[KS], vc[KS];
    // OR of the filtered coefficients' bit patterns: a line whose filtered
    // coefficients are all zero is written as exact zeros (its partner's
    // inverse-DFT round-off would otherwise leak into it)
    long long nzb0 = 0, nzb1 = 0;
    auto load_phase = [&](auto ld0, auto ld1, auto ldp0, auto ldp1) {
#pragma unroll
      for (int l = 0; l < kHoMax; ++l) {
        if (spsm) {  // Re(c conj(d) / den) of a real border coefficient c
          const double2 d = bsp[l];
          const double sv = bsp[4 + l].x;
          const double dd = d.x * d.x + d.y * d.y, ss = sv * sv;
          ua0[l] = l < hk ? ld0(l) * (d.x * rcp_pos(dd + mu0 * ss)) : 0.0;
          ua1[l] = (l < hk && has1) ? ld1(l) * (d.x * rcp_pos(dd + mu1 * ss)) : 0.0;
        } else {
          ua0[l] = l < hk ? f0(ho_coef_elem(ax, l), make_double2(ld0(l), 0.0)).x : 0.0;
          ua1[l] = l < hk ? f1(ho_coef_elem(ax, l), make_double2(ld1(l), 0.0)).x : 0.0;
        }
      }
      // Bluestein inputs of index kk and m - kk (F^H v = conj(F conj v):
      // conj(v_k) c_k, v = X0 + i X1)
      auto one = [&](int kk, int t, double2& a, double2& b) {
        const int e = kl + kk;
        double2 X0, X1;
        if (kk == 0) {
          X0 = make_double2(ld0(hk), 0.0);
          X1 = make_double2(ld1(hk), 0.0);
        } else {
          X0 = ldp0(hk + 2 * kk - 1);
          X1 = ldp1(hk + 2 * kk - 1);
        }
        if (spsm) {  // coeff_filter_fast on the shared-memory copy of (d, s)
          const double2 d = spd[kk];
          const double sv = sps[kk];
          const double dd = d.x * d.x + d.y * d.y, ss = sv * sv;
          const double r0 = rcp_pos(dd + mu0 * ss), r1 = rcp_pos(dd + mu1 * ss);
          X0 = cmul(X0, make_double2(d.x * r0, -d.y * r0));
          X1 = has1 ? cmul(X1, make_double2(d.x * r1, -d.y * r1)) : czero();
        } else {
          X0 = f0(e, X0);
          X1 = f1(e, X1);
        }
        nzb0 |= __double_as_longlong(X0.x) | __double_as_longlong(X0.y);
        nzb1 |= __double_as_longlong(X1.x) | __double_as_longlong(X1.y);
        const double2 ck = cs[kk];  // c_{m-kk} = -c_kk
        a = cmul(make_double2(X0.x - X1.y, -(X0.y + X1.x)), ck);
        b = kk ? cmul(make_double2(-(X0.x + X1.y), X1.x - X0.y), ck) : czero();
      };
      if constexpr (PS::FOLD) {
#pragma unroll
        for (int t = 0; t < KS; ++t) {
          const int kk = threadIdx.x + t * NT;
          vk[t] = vc[t] = czero();
          if (kk <= h) one(kk, t, vk[t], vc[t]);  // (branch-free slots spill at 128 registers)
        }
      } else {
#pragma unroll 2
        for (int kk = threadIdx.x; kk <= h; kk += NT) {
          double2 a, b;
          one(kk, 0, a, b);
          x[pidx(kk)] = a;
          if (kk) x[pidx(m - kk)] = b;
        }
      }
    };
    if (st && (hk & 1) && !(n & 1))  // (Re, Im) pairs 16-byte aligned in the staged lines
      load_phase([&](int i) { return stg.buf[i]; }, [&](int i) { return stg.buf[n + i]; },
                 [&](int i) { return *reinterpret_cast<const double2*>(stg.buf + i); },
                 [&](int i) { return *reinterpret_cast<const double2*>(stg.buf + n + i); });
    else if (st)
      load_phase([&](int i) { return stg.buf[i]; }, [&](int i) { return stg.buf[n + i]; },
                 [&](int i) { return make_double2(stg.buf[i], stg.buf[i + 1]); },
                 [&](int i) { return make_double2(stg.buf[n + i], stg.buf[n + i + 1]); });
    else
      load_phase([&](int i) { return __ldg(g0 + i); },
                 [&](int i) { return has1 ? __ldg(g1 + i) : 0.0; },
                 [&](int i) { return make_double2(__ldg(g0 + i), __ldg(g0 + i + 1)); },
                 [&](int i) {
                   return has1 ? make_double2(__ldg(g1 + i), __ldg(g1 + i + 1)) : czero();
                 });
    zf_add(zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    if (PS::FOLD && threadIdx.x == 0) bulk_wait_read();  // the previous pair's output lines
    __syncthreads();
    FD_PCLK(1, 0);
    if constexpr (PS::FOLD) {  // first DIF stage (v, v W^j); zero padding written explicitly
      const FoldTw<LOGM> fk(tw, threadIdx.x), fc(tw, m - threadIdx.x);
#pragma unroll
      for (int t = 0; t < KS; ++t) {
        const int kk = threadIdx.x + t * NT;
        if (kk <= h) {
          x[pidx(kk)] = vk[t];
          x[pidx(kk + PS::HM)] = cmul(vk[t], fk(kk));
          if (kk) {
            x[pidx(m - kk)] = vc[t];
            x[pidx(m - kk + PS::HM)] = cmul(vc[t], fc(m - kk));
          }
        }
      }
      for (int j = m + threadIdx.x; j < PS::HM; j += NT) {
        x[pidx(j)] = czero();
        x[pidx(j + PS::HM)] = czero();
      }
      __syncthreads();
      FD_PCLK(1, 1);
    }
    pair_conv<LOGM, NT, 1>(x, T, tw, m, pclk_);
    if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, q + gridDim.x, n);

    const Cubic p0 = ho_cubic(ax, ua0), p1 = ho_cubic(ax, ua1);
    const long long eso = io.go.elem_stride;
    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    const int nz = zf_take(zf, it);
    const double s0 = (nz & 1) ? isq : 0.0, s1 = (nz & 2) ? -isq : 0.0;
    const bool vec = eso == 1 && (reinterpret_cast<uintptr_t>(o0) & 15) == 0 &&
                     (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    // FOLD sizes: the restored lines are assembled in shared memory (the
    // buffer's lower part, free once every thread has read its samples) and
    // leave as two bulk stores
    constexpr int PSN = PS::FOLD ? (PS::HM + NT - 1) / NT : 1;
    const bool tout = PS::FOLD && pair_out_staged(o0, o1, n, eso);
    if (tout) {
      double y0r[PSN], y1r[PSN];
#pragma unroll
      for (int t = 0; t < PSN; ++t) {  // branch-free: the slots interleave
        const int p = threadIdx.x + t * NT;
        const int pc = p < m ? p : m - 1;
        const double2 z = cmul(x[pidx(pc)], chirp(pc));  // conj of (F^H v)_p sqrt(m)
        y0r[t] = z.x * s0;
        y1r[t] = z.y * s1;
      }
      // border element bord[l] repeats the interior sample wrap[l] (thread l)
      double yb0 = 0.0, yb1 = 0.0;
      if (threadIdx.x < hk) {
        const int pb = ax.wrap[threadIdx.x];
        const double2 z = cmul(x[pidx(pb)], chirp(pb));
        yb0 = z.x * s0;
        yb1 = z.y * s1;
      }
      __syncthreads();  // every sample has been read
      double* lineA = reinterpret_cast<double*>(x);
      double* lineB = lineA + n;
#pragma unroll
      for (int t = 0; t < PSN; ++t) {
        const int p = threadIdx.x + t * NT;
        const double tt = fma((double)(t * NT), ax.ho_ta, tt0);
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
    } else if (vec) {
      // element pairs (2u, 2u + 1) as 16-byte stores; a border element takes
      // the interior sample it wraps to (ax.wrap) with the cubic at its own t
      for (int u = threadIdx.x; 2 * u < n; u += NT) {
        double r0[2] = {0.0, 0.0}, r1[2] = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int e = 2 * u + c;
          if (e >= n) continue;
          int p = e - kl;
          if (p < 0)
            p = ax.wrap[e];
          else if (p >= m)
            p = ax.wrap[kl + (p - m)];
          const double2 z = cmul(x[pidx(p)], chirp(p));  // conj of (F^H v)_p sqrt(m)
          const double t = fma((double)e, ax.ho_ta, ax.ho_tb);
          r0[c] = z.x * s0 + p0(t);
          r1[c] = z.y * s1 + p1(t);
        }
        if (2 * u + 1 < n) {
          *reinterpret_cast<double2*>(o0 + 2 * u) = make_double2(r0[0], r0[1]);
          if (o1) *reinterpret_cast<double2*>(o1 + 2 * u) = make_double2(r1[0], r1[1]);
        } else {
          o0[2 * u] = r0[0];
          if (o1) o1[2 * u] = r1[0];
        }
      }
    } else
#pragma unroll 4
    for (int p = threadIdx.x; p < m; p += NT) {
      const double2 z = cmul(x[pidx(p)], chirp(p));  // conj of (F^H v)_p sqrt(m)
      const double y0 = z.x * s0, y1 = z.y * s1;
      const int e = kl + p;
      const double t = fma((double)e, ax.ho_ta, ax.ho_tb);
      o0[e * eso] = y0 + p0(t);
      if (o1) o1[e * eso] = y1 + p1(t);
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
    FD_PCLK(1, 8);
  }
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

}  // namespace fdb
