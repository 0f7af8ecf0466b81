// The direct mixed-radix line-pair kernels (fd_mixed.cuh) with all global
// traffic on the bulk-copy engine: one CTA of 512 threads per SM, the next
// pair's two lines staged into shared memory while the current pair is
// transformed, the output lines (and the GCV weight rows) assembled in shared
// memory and bulk-stored while the next pair starts.  In k_manalyze / k_msynth
// (2 CTAs x 256 threads, inputs by __ldg, outputs by per-element stores) the
// DFT stages were a third of the time: the load phases waited on L2 (38-44 %
// long-scoreboard stalls) and the post phases on the SM's store path.
//
// Requirements (checked by launch_pair, which otherwise takes the kernels of
// fd_mixed.cuh): contiguous unit-stride lines of even length, 16-byte aligned;
// m <= 4096 (4 Hermitian slots, 8 sample slots per thread); first-stage
// stride m / r0 <= 512 (its results are held in registers until the previous
// pair's output lines have left the buffer); synthesis: the 1D filter
// (spectral mode 1) of a complex basis, or no filter.
//
// Shared memory (double2 slots): DFT buffer x (max(m + 1, n): the two output
// lines of n doubles are assembled here) | twiddle lo (64), hi | staged input (n) |
// aux: weight rows (analysis) or the filter's spectral table (synthesis) |
// output permutation (u16) | mbarrier + zero-line flags.
#pragma once

namespace fdb {

constexpr int kMixSNT = 512;
constexpr int kMixSK = 4;  // Hermitian slots per thread: kk = tid + t NT <= h
constexpr int kMixSP = 8;  // sample slots per thread: p = tid + t NT < m

__host__ __device__ __forceinline__ int mixs_aux_slots(int m, long long wstride) {
  const int h = (m - 1) / 2;
  const int sp = (h + 1) + (h + 2) / 2 + 8;
  return wstride > sp ? (int)wstride : sp;
}
// the DFT buffer also holds the two assembled output lines (2 n doubles)
__host__ __device__ __forceinline__ int mixs_x_slots(int m, int n) { return m + 1 > n ? m + 1 : n; }
__host__ __device__ __forceinline__ size_t mixs_smem_bytes(int m, int n, long long wstride) {
  const int nhi = (m + 63) >> 6;
  return ((size_t)mixs_x_slots(m, n) + 64 + nhi + n + mixs_aux_slots(m, wstride) + (m + 7) / 8 + 1) *
         16;
}
__host__ __device__ __forceinline__ bool mixs_shape_ok(int m, int n, int r0) {
  return (m - 1) / 2 < kMixSK * kMixSNT && m <= kMixSP * kMixSNT && m / r0 <= kMixSNT &&
         !(n & 1) && (m & 1);
}

struct MixSm {
  double2* x;
  MixTw tw;
  double* S;      // staged input: line l0 at [0, n), line l0 + 1 at [n, 2n)
  double2* aux;
  const unsigned short* perm;
  uint64_t* bar;
  int* zf;
};

__device__ __forceinline__ MixSm mixs_setup(double2* sm, const AxisDev& ax, long long wstride) {
  const int m = ax.m, nhi = (m + 63) >> 6;
  MixSm s;
  s.x = sm;
  double2* lo = sm + mixs_x_slots(m, ax.n);
  double2* hi = lo + 64;
  s.tw = MixTw{lo, hi};
  s.S = reinterpret_cast<double*>(hi + nhi);
  s.aux = hi + nhi + ax.n;
  unsigned short* ps = reinterpret_cast<unsigned short*>(s.aux + mixs_aux_slots(m, wstride));
  s.perm = ps;
  s.bar = reinterpret_cast<uint64_t*>(reinterpret_cast<double2*>(ps) + (m + 7) / 8);
  s.zf = reinterpret_cast<int*>(s.bar) + 2;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) lo[i] = i < m ? ax.mtw[i] : czero();
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) hi[i] = ax.mtw[i << 6];
  for (int i = threadIdx.x; i < m; i += blockDim.x) ps[i] = (unsigned short)ax.mperm[i];
  if (threadIdx.x < 2) s.zf[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    mbar_init(s.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  return s;
}

// stage the lines of pair q (one bulk copy: the lines are adjacent)
__device__ __forceinline__ void mixs_issue(const MixSm& s, const void* base, const Lines& g, int q,
                                           int n) {
  if (2 * q >= g.count) return;
  const double* src = reinterpret_cast<const double*>(base) + line_offset(g, 2 * q);
  const uint32_t bytes = (uint32_t)(2 * q + 1 < g.count ? 2 * n : n) * 8;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(s.bar, bytes);
  bulk_g2s(s.S, src, bytes, s.bar);
}

// first stage of the DIF transform into registers: v[p], p < R, of item j
template <int R, class LD>
__device__ __forceinline__ void mixs_first(double2 (&v)[kMixMaxR], int j, int L, const MixTw& tw,
                                           LD&& ld) {
  double2 u[R];
#pragma unroll
  for (int q = 0; q < R; ++q) u[q] = ld(j + q * L, q);
  mix_codelet<R>(u);
  if (L > 1) mix_twiddle<R>(u, tw(j));
#pragma unroll
  for (int p = 0; p < R; ++p) v[p] = u[p];
}
template <class LD>
__device__ __forceinline__ void mixs_first_any(int r, double2 (&v)[kMixMaxR], int j, int L,
                                               const MixTw& tw, LD&& ld) {
  switch (r) {
    case 3: mixs_first<3>(v, j, L, tw, ld); break;
    case 5: mixs_first<5>(v, j, L, tw, ld); break;
    case 7: mixs_first<7>(v, j, L, tw, ld); break;
    case 9: mixs_first<9>(v, j, L, tw, ld); break;
    case 11: mixs_first<11>(v, j, L, tw, ld); break;
    default: mixs_first<13>(v, j, L, tw, ld); break;
  }
}
// stages s0 .. of the transform (block size S at stage s0), barrier after each
__device__ __forceinline__ void mixs_stages(double2* x, const AxisDev& ax, const MixTw& tw, int s0,
                                            int S) {
  for (int s = s0; s < ax.mstages; ++s) {
    const int r = ax.mrad[s];
    switch (r) {
      case 3: mix_stage<3>(x, ax.m, S, tw, kMixSNT); break;
      case 5: mix_stage<5>(x, ax.m, S, tw, kMixSNT); break;
      case 7: mix_stage<7>(x, ax.m, S, tw, kMixSNT); break;
      case 9: mix_stage<9>(x, ax.m, S, tw, kMixSNT); break;
      case 11: mix_stage<11>(x, ax.m, S, tw, kMixSNT); break;
      default: mix_stage<13>(x, ax.m, S, tw, kMixSNT); break;
    }
    S /= r;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kMixSNT, 1) k_manalyze_s(AxisDev ax, LineIO io) {
  constexpr int NT = kMixSNT;
  extern __shared__ double2 sm[];
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  const MixSm S = mixs_setup(sm, ax, io.wstride);
  double2* x = S.x;
  const unsigned short* perm = S.perm;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) mixs_issue(S, io.in, io.gi, blockIdx.x, n);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
  const long long nkb32 = io.wstride >> 5;
  const int r0 = ax.mrad[0], L = m / r0;
  // abscissa t_e = ho_ta e + ho_tb of first-stage input q of this thread's item
  const double tj0 = fma((double)(kl + (int)threadIdx.x), ax.ho_ta, ax.ho_tb);
  const double dL = (double)L * ax.ho_ta;
  double* wA = reinterpret_cast<double*>(S.aux);
  double* wB = wA + io.wstride;
  const double* s0 = S.S;
  const double* s1 = S.S + n;
  uint32_t phase = 0;
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    mbar_wait(S.bar, phase);
    phase ^= 1;
    auto ld0 = [&](int e) { return s0[e]; };
    auto ld1 = [&](int e) { return has1 ? s1[e] : 0.0; };
    double a0[kHoMax], a1[kHoMax];
    ho_amps_real(ax, ld0, a0);
    ho_amps_real(ax, ld1, a1);
    const Cubic p0 = ho_cubic(ax, a0), p1 = ho_cubic(ax, a1);
    long long nzb0 = 0, nzb1 = 0;  // OR of the bit patterns of line 0 / 1 (-0.0 counts as nonzero)
    double2 v[kMixMaxR];
    const int j = threadIdx.x;
    if (j < L)
      mixs_first_any(r0, v, j, L, S.tw, [&](int jj, int qq) {
        const int e = kl + jj;
        const double t = fma((double)qq, dL, tj0);
        const double y0 = ld0(e), y1 = ld1(e);
        nzb0 |= __double_as_longlong(y0);
        nzb1 |= __double_as_longlong(y1);
        return make_double2(y0 - p0(t), y1 - p1(t));
      });
    zf_add(S.zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    if (threadIdx.x == 0) bulk_wait_read();  // the previous pair's lines have left x and the rows
    __syncthreads();                         // staged input consumed
    if (threadIdx.x == 0) mixs_issue(S, io.in, io.gi, q + gridDim.x, n);
    if (j < L) {
#pragma unroll
      for (int p = 0; p < kMixMaxR; ++p)
        if (p < r0) x[j + p * L] = v[p];
    }
    __syncthreads();
    mixs_stages(x, ax, S.tw, 1, m / r0);

    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    double* w0 = io.wout ? io.wout + (long long)l0 * io.wstride : nullptr;
    // an all-zero line gets exactly zero coefficients (its partner's DFT
    // round-off would otherwise leak into it through the Hermitian split)
    const int nz = zf_take(S.zf, it);
    const bool z0 = !(nz & 1) && ho_zero(a0), z1 = !(nz & 2) && ho_zero(a1);
    double2 X0r[kMixSK], X1r[kMixSK];
#pragma unroll
    for (int t = 0; t < kMixSK; ++t) {
      const int kq = threadIdx.x + t * NT;
      const int kk = kq <= h ? kq : h;  // clamped: branch-free slots interleave
      const double2 Zk = x[perm[kk]];
      const double2 Zm = x[perm[m - kk < m ? m - kk : 0]];
      const double2 Zc = kk ? Zm : Zk;
      const double2 D = csub(Zk, cconj(Zc));
      const double2 X0 = z0 ? czero() : cscale(cadd(Zk, cconj(Zc)), 0.5 * isq);
      const double2 X1 = z1 ? czero() : make_double2(0.5 * isq * D.y, -0.5 * isq * D.x);
      X0r[t] = X0;
      X1r[t] = X1;
      if (w0 && kq <= h) {
        const double f = kk ? 2.0 : 1.0;  // |X_k|^2 + |X_{m-k}|^2
        wA[kl + kk] = f * (X0.x * X0.x + X0.y * X0.y);
        wB[kl + kk] = f * (X1.x * X1.x + X1.y * X1.y);
      }
    }
    if (w0) {
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
    for (int t = 0; t < kMixSK; ++t) {
      const int kk = threadIdx.x + t * NT;
      if (kk > h) continue;
      if (kk == 0) {
        lineA[hk] = X0r[t].x;
        lineB[hk] = X1r[t].x;
      } else if (hk & 1) {  // (Re, Im) 16-byte aligned
        *reinterpret_cast<double2*>(lineA + hk + 2 * kk - 1) = X0r[t];
        *reinterpret_cast<double2*>(lineB + hk + 2 * kk - 1) = X1r[t];
      } else {
        lineA[hk + 2 * kk - 1] = X0r[t].x;
        lineA[hk + 2 * kk] = X0r[t].y;
        lineB[hk + 2 * kk - 1] = X1r[t].x;
        lineB[hk + 2 * kk] = X1r[t].y;
      }
    }
    if (threadIdx.x < hk) {
      lineA[threadIdx.x] = a0[threadIdx.x];
      lineB[threadIdx.x] = a1[threadIdx.x];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (w0 && io.wout32) {
      // TF32 tiles from the staged rows: task c = chunk c >> 1 (4 elements)
      // of line l0 + (c & 1), one 16-byte store per array (see k_panalyze)
      float* th = io.wout32 + tc_tile_index(l0, 0, kTcBM, nkb32);
      float* tl = io.wout32lo + tc_tile_index(l0, 0, kTcBM, nkb32);
      const int ntask = (int)(io.wstride >> 1);
      for (int c = threadIdx.x; c < ntask; c += NT) {
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
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(o0, lineA, (uint32_t)n * 8);
      if (o1) bulk_s2g(o1, lineB, (uint32_t)n * 8);
      if (w0) {
        bulk_s2g(w0, wA, (uint32_t)io.wstride * 8);
        if (has1) bulk_s2g(w0 + io.wstride, wB, (uint32_t)io.wstride * 8);
      }
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

// synthesis with the filter fused (see k_msynth / k_psynth)
__global__ void __launch_bounds__(kMixSNT, 1) k_msynth_s(AxisDev ax, LineIO io, SynthArgs sa) {
  constexpr int NT = kMixSNT;
  extern __shared__ double2 sm[];
  const int m = ax.m, n = ax.n, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  const MixSm S = mixs_setup(sm, ax, 0);
  double2* x = S.x;
  const unsigned short* perm = S.perm;
  // the 1D filter's spectral table (launch_pair guarantees mode 1 / complex
  // when the synthesis filters): border entries, then d and s of the interior
  const bool filt = sa.mode == 1;
  double2* bsp = S.aux;  // [l] = d of border coefficient l, [4 + l].x = s
  double2* spd = bsp + 8;
  double* sps = reinterpret_cast<double*>(spd + h + 1);
  if (filt) {
    for (int kk = threadIdx.x; kk <= h; kk += NT) {
      spd[kk] = __ldg(&sa.sp.dA[kl + kk]);
      sps[kk] = sa.sp.sA ? __ldg(&sa.sp.sA[kl + kk]) : 1.0;
    }
    if (threadIdx.x < hk) {
      const int e = ho_coef_elem(ax, threadIdx.x);
      bsp[threadIdx.x] = __ldg(&sa.sp.dA[e]);
      bsp[4 + threadIdx.x].x = sa.sp.sA ? __ldg(&sa.sp.sA[e]) : 1.0;
    }
  }
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  if (threadIdx.x == 0) mixs_issue(S, io.in, io.gi, blockIdx.x, n);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
  const double tt0 = fma((double)(kl + (int)threadIdx.x), ax.ho_ta, ax.ho_tb);
  const double* s0 = S.S;
  const double* s1 = S.S + n;
  auto pair_mu = [&](int q, double& m0, double& m1) {  // read one pair ahead
    m0 = m1 = 0.0;
    if (q < npairs) {
      m0 = line_mu(sa, io.gi, 2 * q);
      m1 = 2 * q + 1 < count ? line_mu(sa, io.gi, 2 * q + 1) : m0;
    }
  };
  double mu0n, mu1n;
  pair_mu(blockIdx.x, mu0n, mu1n);
  uint32_t phase = 0;
  for (int q = blockIdx.x, it = 0; q < npairs; q += gridDim.x, ++it) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const double mu0 = mu0n, mu1 = mu1n;
    pair_mu(q + gridDim.x, mu0n, mu1n);
    mbar_wait(S.bar, phase);
    phase ^= 1;
    // conj(d) / (|d|^2 + mu s^2) (coeff_filter_fast), or 1 without a filter
    auto fil = [&](double2 d, double sv, double mu) {
      const double r = rcp_pos((d.x * d.x + d.y * d.y) + mu * (sv * sv));
      return make_double2(d.x * r, -d.y * r);
    };
    double ua0[kHoMax], ua1[kHoMax];
#pragma unroll
    for (int l = 0; l < kHoMax; ++l) {
      double g0 = 1.0, g1 = 1.0;
      if (filt) {
        g0 = fil(bsp[l], bsp[4 + l].x, mu0).x;
        g1 = fil(bsp[l], bsp[4 + l].x, mu1).x;
      }
      ua0[l] = l < hk ? s0[l] * g0 : 0.0;
      ua1[l] = (l < hk && has1) ? s1[l] * g1 : 0.0;
    }
    long long nzb0 = 0, nzb1 = 0;  // all-zero filtered lines are written as exact zeros
    double2 va[kMixSK], vb[kMixSK];
#pragma unroll
    for (int t = 0; t < kMixSK; ++t) {
      const int kq = threadIdx.x + t * NT;
      const int kk = kq <= h ? kq : h;
      // (Re X_kk, Im X_kk) at [hk - 1 + 2 kk, hk + 2 kk]; X_0 is real, at [hk]
      double2 X0, X1;
      const int i0 = hk - 1 + 2 * kk;
      if (hk & 1) {  // 16-byte aligned in the staged lines
        X0 = *reinterpret_cast<const double2*>(s0 + i0);
        X1 = *reinterpret_cast<const double2*>(s1 + i0);
      } else {
        X0 = make_double2(s0[i0 > 0 ? i0 : 0], s0[i0 + 1]);
        X1 = make_double2(s1[i0 > 0 ? i0 : 0], s1[i0 + 1]);
      }
      if (kk == 0) {
        X0 = make_double2(X0.y, 0.0);
        X1 = make_double2(X1.y, 0.0);
      }
      if (!has1) X1 = czero();
      if (filt) {
        const double2 d = spd[kk];
        const double sv = sps[kk];
        X0 = cmul(X0, fil(d, sv, mu0));
        X1 = cmul(X1, fil(d, sv, mu1));
      }
      nzb0 |= __double_as_longlong(X0.x) | __double_as_longlong(X0.y);
      nzb1 |= __double_as_longlong(X1.x) | __double_as_longlong(X1.y);
      // F^H v = conj(F conj v), v = X0 + i X1 (natural order input)
      va[t] = make_double2(X0.x - X1.y, -(X0.y + X1.x));
      vb[t] = make_double2(X0.x + X1.y, X0.y - X1.x);
    }
    zf_add(S.zf, it, (nzb0 != 0 ? 1 : 0) | (nzb1 != 0 ? 2 : 0));
    if (threadIdx.x == 0) bulk_wait_read();  // the previous pair's lines have left x
    __syncthreads();                         // staged input consumed
    if (threadIdx.x == 0) mixs_issue(S, io.in, io.gi, q + gridDim.x, n);
#pragma unroll
    for (int t = 0; t < kMixSK; ++t) {
      const int kk = threadIdx.x + t * NT;
      if (kk <= h) {
        x[kk] = va[t];
        if (kk) x[m - kk] = vb[t];
      }
    }
    __syncthreads();
    mixs_stages(x, ax, S.tw, 0, m);

    const Cubic p0 = ho_cubic(ax, ua0), p1 = ho_cubic(ax, ua1);
    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    const int nz = zf_take(S.zf, it);
    const double sc0 = (nz & 1) ? isq : 0.0, sc1 = (nz & 2) ? -isq : 0.0;
    double y0r[kMixSP], y1r[kMixSP];
#pragma unroll
    for (int t = 0; t < kMixSP; ++t) {  // branch-free: the slots interleave
      const int p = threadIdx.x + t * NT;
      const double2 z = x[perm[p < m ? p : m - 1]];
      y0r[t] = z.x * sc0;
      y1r[t] = z.y * sc1;
    }
    // border element bord[l] repeats the interior sample wrap[l] (thread l)
    double yb0 = 0.0, yb1 = 0.0;
    if (threadIdx.x < hk) {
      const double2 z = x[perm[ax.wrap[threadIdx.x]]];
      yb0 = z.x * sc0;
      yb1 = z.y * sc1;
    }
    __syncthreads();  // every sample has been read
    double* lineA = reinterpret_cast<double*>(x);
    double* lineB = lineA + n;
#pragma unroll
    for (int t = 0; t < kMixSP; ++t) {
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
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(o0, lineA, (uint32_t)n * 8);
      if (o1) bulk_s2g(o1, lineB, (uint32_t)n * 8);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_read();  // shared memory stays valid until the last lines are read
}

}  // namespace fdb
