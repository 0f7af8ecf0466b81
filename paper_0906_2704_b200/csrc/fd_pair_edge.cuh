// Line-pair kernels of fd_pair.cuh with the OUTERMOST radix-16 passes kept in
// registers (M = 8192, 256 threads: BASELINE config 1 at d = 3, m = 4093).
//
// With the folded radix-2 stage (PairShape::FOLD) the Bluestein convolution is
// two independent 4096-point convolutions, of v and of v W^j.  At 256 threads
// the values a thread produces in the load phase, j = tid + 256 t (t < 16),
// are exactly the 16 inputs of its item of the first radix-16 DIF pass (block
// 4096, sub-block stride 256) -- of both halves.  So the first pass runs on
// the load phase's registers and only its results are stored; the last DIT
// pass likewise ends in registers, where the halves are combined
// (lo + conj(W^j) hi), multiplied by the chirp and -- synthesis -- written to
// global memory.  Against k_panalyze / k_psynth this removes, per line pair,
// the fold store sweep, the first pass's loads, the last pass's stores, the
// combine sweep and (synthesis) the post phase's reads: ~10k shared-memory
// wavefronts instead of ~16.7k, and 7 CTA barriers instead of 9.
//
// Arithmetic (twiddles, butterflies, pass order, bhat layout) is that of
// bluestein_rec<13, 1, 4096, 256>; the inner passes are its P >= 2 levels.
#pragma once

namespace fdb {

// the four radix-2 stages of one radix-16 item, in registers (dif_pass_t / dit_pass_t)
__device__ __forceinline__ void dif16(double2 (&v)[16], const double2 (&ws)[4]) {
#pragma unroll
  for (int st = 0; st < 4; ++st) {
    const int half = 16 >> (st + 1);
    const double2 w = ws[st];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q & half) continue;
      const int qq = q & (half - 1);
      const double2 a = v[q], b = v[q + half];
      v[q] = cadd(a, b);
      v[q + half] = cmul(mul_w16(csub(a, b), qq << st), w);
    }
  }
}
__device__ __forceinline__ void dit16(double2 (&v)[16], const double2 (&ws)[4]) {
#pragma unroll
  for (int st = 3; st >= 0; --st) {
    const int half = 16 >> (st + 1);
    const double2 w = ws[st];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q & half) continue;
      const int qq = q & (half - 1);
      const double2 a = v[q];
      const double2 b = mul_w16c(cmulc(v[q + half], w), qq << st);
      v[q] = cadd(a, b);
      v[q + half] = csub(a, b);
    }
  }
}

template <int LOGM>
struct EdgeShape {
  static_assert(LOGM == 13, "edge-fused pair kernels: M = 8192 at 256 threads");
  static constexpr int NT = 256, M = 1 << LOGM, HM = M / 2;
  static constexpr int SR = HM / 16;        // sub-block stride of the outermost radix-16 pass
  static constexpr int QS = SR + SR / 16;   // its padded slot stride
  static_assert(SR == NT, "thread t owns item t of each half");
};

// first pass of both halves from the load phase's registers (v is consumed)
template <int LOGM>
__device__ __forceinline__ void edge_first_pass(double2* x, double2 (&v)[16],
                                                const double2 (&ws)[4], const FoldTw<LOGM>& ft) {
  using E = EdgeShape<LOGM>;
  double2* xlo = x + pidx(threadIdx.x);
  double2* xhi = x + pidx(E::HM + threadIdx.x);
  {
    double2 u[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) u[t] = cmul(v[t], ft(threadIdx.x + t * E::NT));
    dif16(u, ws);
#pragma unroll
    for (int q = 0; q < 16; ++q) xhi[q * E::QS] = u[q];
  }
  dif16(v, ws);
#pragma unroll
  for (int q = 0; q < 16; ++q) xlo[q * E::QS] = v[q];
}

// last pass of both halves into registers: z[t] = (a * b)_j, j = tid + 256 t
template <int LOGM>
__device__ __forceinline__ void edge_last_pass(const double2* x, double2 (&z)[16],
                                               const double2 (&ws)[4], const FoldTw<LOGM>& ft) {
  using E = EdgeShape<LOGM>;
  const double2* xlo = x + pidx(threadIdx.x);
  const double2* xhi = x + pidx(E::HM + threadIdx.x);
  double2 u[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) u[q] = xhi[q * E::QS];
#pragma unroll
  for (int q = 0; q < 16; ++q) z[q] = xlo[q * E::QS];
  dit16(u, ws);
  dit16(z, ws);
#pragma unroll
  for (int t = 0; t < 16; ++t) z[t] = cadd(z[t], cmulc(u[t], ft(threadIdx.x + t * E::NT)));
}

template <int LOGM>
__global__ void __launch_bounds__(EdgeShape<LOGM>::NT, 1) k_panalyze_e(AxisDev ax, LineIO io) {
  using E = EdgeShape<LOGM>;
  constexpr int NT = E::NT, M = E::M;
  using F = FftShape<LOGM, NT>;
  extern __shared__ double2 sm[];
  const FftTables& T = ax.fft;
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  double2* slots = sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(slots, T);
  double2* cs = slots + kTwSlots;
  for (int j = threadIdx.x; j < m; j += NT) cs[j] = T.chirp[j];
  PairStage stg = pair_stage_init(x, M, m, n, io.gi,
                                  reinterpret_cast<uint64_t*>(sm + pair_slots(M, m) - 1));
  int* zf = reinterpret_cast<int*>(sm + pair_slots(M, m) - 1) + 2;
  if (threadIdx.x < 2) zf[threadIdx.x] = 0;
  __syncthreads();
  const FoldTw<LOGM> ft(tw, threadIdx.x);
  double2 ws[4];  // stage twiddles of this thread's outermost item: W_4096^tid and its squares
  tw_pow2<4>(ws, tw_t<F::LOB>(tw, 2 * threadIdx.x));
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, blockIdx.x, n);
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const long long es = io.gi.elem_stride;
  const double isq = ax.inv_sqrt_m;
  const long long nkb32 = io.wstride >> 5;
#ifdef FD_PHASE_CLOCKS
  long long pclk_ = clock64();
#else
  long long pclk_ = 0;
#endif
  (void)pclk_;
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
    double2 v[16];
    long long nzb0 = 0, nzb1 = 0;  // OR of the bit patterns of line 0 / 1 (-0.0 counts as nonzero)
    auto load_phase = [&](auto ld0, auto ld1) {
      ho_amps_real(ax, ld0, a0);
      ho_amps_real(ax, ld1, a1);
      const Cubic p0 = ho_cubic(ax, a0), p1 = ho_cubic(ax, a1);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int j = threadIdx.x + t * NT;
        if (j < m) {
          const int e = kl + j;
          const double tt = fma((double)e, ax.ho_ta, ax.ho_tb);
          const double y0 = ld0(e), y1 = ld1(e);
          nzb0 |= __double_as_longlong(y0);
          nzb1 |= __double_as_longlong(y1);
          v[t] = cmul(make_double2(y0 - p0(tt), y1 - p1(tt)), cs[j]);
        } else {
          v[t] = czero();
        }
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
    __syncthreads();  // staged input consumed; the previous pair's split reads are done
    FD_PCLK(2, 0);
    edge_first_pass<LOGM>(x, v, ws, ft);
    if (threadIdx.x == 0) zf[(it + 1) & 1] = 0;  // read before this pair's first barrier, written after its last
    __syncthreads();
    FD_PCLK(2, 2);
#ifdef FD_PHASE_CLOCKS
    bluestein_rec_clk<LOGM, 2, E::SR, NT, 2, 3>(x, T.bhat, tw, M, pclk_);
#else
    bluestein_rec<LOGM, 2, E::SR, NT>(x, T.bhat, tw, M);  // inner passes; ends with a barrier
#endif
    edge_last_pass<LOGM>(x, v, ws, ft);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int j = threadIdx.x + t * NT;
      v[t] = cmul(v[t], cs[j < m ? j : 0]);  // Z_j sqrt(m)
    }
    __syncthreads();  // the whole buffer has been read
    FD_PCLK(2, 6);
    if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, q + gridDim.x, n);
    // Z_j of the upper index half goes through shared memory to the thread of m - j
#pragma unroll
    for (int t = 7; t < 16; ++t) {
      const int j = threadIdx.x + t * NT;
      if (j > h && j < m) x[pidx(j)] = v[t];
    }
    __syncthreads();
    FD_PCLK(2, 7);

    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    double* w0 = io.wout ? io.wout + (long long)l0 * io.wstride : nullptr;
    auto wset = [&](int line, double* wl, long long i, double val) {
      wl[i] = val;
      if (io.wout32) {
        float hi, lo;
        tf32_split(val, hi, lo);
        const long long ti = tc_tile_index(line, i, kTcBM, nkb32);
        io.wout32[ti] = hi;
        io.wout32lo[ti] = lo;
      }
    };
    double* w1 = (w0 && has1) ? w0 + io.wstride : nullptr;
    const int nz = zf[it & 1];
    const bool z0 = !(nz & 1) && ho_zero(a0), z1 = !(nz & 2) && ho_zero(a1);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int kk = threadIdx.x + t * NT;
      if (kk > h) continue;
      const double2 Zk = v[t];
      const double2 Zc = kk ? x[pidx(m - kk)] : Zk;
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
        wset(l0, w0, kl + kk, f * (X0.x * X0.x + X0.y * X0.y));
        if (w1) wset(l0 + 1, w1, kl + kk, f * (X1.x * X1.x + X1.y * X1.y));
      }
    }
    if (threadIdx.x < hk) {
      const int l = threadIdx.x;
      o0[l] = a0[l];
      if (o1) o1[l] = a1[l];
      if (w0) {
        wset(l0, w0, ho_wred(ax, l, h), a0[l] * a0[l]);
        if (w1) wset(l0 + 1, w1, ho_wred(ax, l, h), a1[l] * a1[l]);
      }
    }
    if (w0)
      for (long long i = io.wn + threadIdx.x; i < io.wstride; i += NT) {
        wset(l0, w0, i, 0.0);
        if (w1) wset(l0 + 1, w1, i, 0.0);
      }
    // no barrier here: the next pair's first barrier orders these reads of x
    // against its first-pass stores
    FD_PCLK(2, 8);
  }
}

template <int LOGM>
__global__ void __launch_bounds__(EdgeShape<LOGM>::NT, 1) k_psynth_e(AxisDev ax, LineIO io,
                                                                     SynthArgs sa) {
  using E = EdgeShape<LOGM>;
  constexpr int NT = E::NT, M = E::M;
  using F = FftShape<LOGM, NT>;
  extern __shared__ double2 sm[];
  const FftTables& T = ax.fft;
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  double2* x = sm;
  double2* slots = sm + pidx(M) + 1;
  const TwSm tw = load_twiddles(slots, T);
  double2* cs = slots + kTwSlots;
  for (int j = threadIdx.x; j < m; j += NT) cs[j] = T.chirp[j];
  PairStage stg = pair_stage_init(x, M, m, n, io.gi,
                                  reinterpret_cast<uint64_t*>(sm + pair_slots(M, m) - 1));
  int* zf = reinterpret_cast<int*>(sm + pair_slots(M, m) - 1) + 2;
  if (threadIdx.x < 2) zf[threadIdx.x] = 0;
  __syncthreads();
  const FoldTw<LOGM> ft(tw, threadIdx.x);
  double2 ws[4];
  tw_pow2<4>(ws, tw_t<F::LOB>(tw, 2 * threadIdx.x));
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, blockIdx.x, n);
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
#ifdef FD_PHASE_CLOCKS
  long long pclk_ = clock64();
#else
  long long pclk_ = 0;
#endif
  (void)pclk_;
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
    const double mu0 = line_mu(sa, io.gi, l0);
    const double mu1 = has1 ? line_mu(sa, io.gi, l0 + 1) : mu0;
    auto f0 = [&](int e, double2 c) { return coeff_filter_fast(ax, sa, io.gi, l0, e, c, mu0); };
    auto f1 = [&](int e, double2 c) {
      return has1 ? coeff_filter_fast(ax, sa, io.gi, l0 + 1, e, c, mu1) : czero();
    };
    double ua0[kHoMax], ua1[kHoMax];
    double2 v[16];
    // OR of the filtered coefficients' bit patterns: a line whose filtered
    // coefficients are all zero is written as exact zeros (its partner's
    // inverse-DFT round-off would otherwise leak into it)
    long long nzb0 = 0, nzb1 = 0;
    auto load_phase = [&](auto ld0, auto ld1) {
#pragma unroll
      for (int l = 0; l < kHoMax; ++l) {
        ua0[l] = l < hk ? f0(ho_coef_elem(ax, l), make_double2(ld0(l), 0.0)).x : 0.0;
        ua1[l] = l < hk ? f1(ho_coef_elem(ax, l), make_double2(ld1(l), 0.0)).x : 0.0;
      }
      // Bluestein inputs of index kk (kept) and m - kk (to the thread of that
      // index, through the buffer): F^H v = conj(F conj v), v = X0 + i X1
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int kk = threadIdx.x + t * NT;
        v[t] = czero();
        if (kk > h) continue;
        const int e = kl + kk;
        double2 X0, X1;
        if (kk == 0) {
          X0 = make_double2(ld0(hk), 0.0);
          X1 = make_double2(ld1(hk), 0.0);
        } else {
          X0 = make_double2(ld0(hk + 2 * kk - 1), ld0(hk + 2 * kk));
          X1 = make_double2(ld1(hk + 2 * kk - 1), ld1(hk + 2 * kk));
        }
        X0 = f0(e, X0);
        X1 = f1(e, X1);
        nzb0 |= __double_as_longlong(X0.x) | __double_as_longlong(X0.y);
        nzb1 |= __double_as_longlong(X1.x) | __double_as_longlong(X1.y);
        v[t] = cmul(make_double2(X0.x - X1.y, -(X0.y + X1.x)), cs[kk]);
        if (kk) x[pidx(m - kk)] = cmul(make_double2(X0.x + X1.y, X0.y - X1.x), cs[m - kk]);
      }
    };
    if (st)
      load_phase([&](int i) { return stg.buf[i]; }, [&](int i) { return stg.buf[n + i]; });
    else
      load_phase([&](int i) { return __ldg(g0 + i); },
                 [&](int i) { return has1 ? __ldg(g1 + i) : 0.0; });
    zf_add(zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    __syncthreads();
    FD_PCLK(3, 0);
#pragma unroll
    for (int t = 7; t < 16; ++t) {
      const int j = threadIdx.x + t * NT;
      if (j > h) v[t] = j < m ? x[pidx(j)] : czero();
    }
    __syncthreads();  // staged input and the exchanged half consumed
    FD_PCLK(3, 1);
    edge_first_pass<LOGM>(x, v, ws, ft);
    if (threadIdx.x == 0) zf[(it + 1) & 1] = 0;
    __syncthreads();
    FD_PCLK(3, 2);
#ifdef FD_PHASE_CLOCKS
    bluestein_rec_clk<LOGM, 2, E::SR, NT, 3, 3>(x, T.bhat, tw, M, pclk_);
#else
    bluestein_rec<LOGM, 2, E::SR, NT>(x, T.bhat, tw, M);  // inner passes; ends with a barrier
#endif
    edge_last_pass<LOGM>(x, v, ws, ft);
    const int nz = zf[it & 1];
    __syncthreads();  // the whole buffer has been read
    FD_PCLK(3, 6);
    if (threadIdx.x == 0) pair_issue(stg, io.in, io.gi, q + gridDim.x, n);

    const Cubic p0 = ho_cubic(ax, ua0), p1 = ho_cubic(ax, ua1);
    const long long eso = io.go.elem_stride;
    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    const double s0 = (nz & 1) ? isq : 0.0, s1 = (nz & 2) ? -isq : 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int p = threadIdx.x + t * NT;
      if (p >= m) continue;
      const double2 z = cmul(v[t], cs[p]);  // conj of (F^H v)_p sqrt(m)
      const double y0 = z.x * s0, y1 = z.y * s1;
      const int e = kl + p;
      const double tt = fma((double)e, ax.ho_ta, ax.ho_tb);
      o0[e * eso] = y0 + p0(tt);
      if (o1) o1[e * eso] = y1 + p1(tt);
#pragma unroll
      for (int l = 0; l < kHoMax; ++l)
        if (l < hk && ax.wrap[l] == p) {
          const int eb = ax.bord[l];
          const double tb = fma((double)eb, ax.ho_ta, ax.ho_tb);
          o0[eb * eso] = y0 + p0(tb);
          if (o1) o1[eb * eso] = y1 + p1(tb);
        }
    }
    FD_PCLK(3, 8);
  }
}

}  // namespace fdb
