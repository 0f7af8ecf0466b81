// Rader's algorithm for the pair kernels when the interior length m is an odd
// prime p whose p - 1 factors into radices 2..13 (e.g. m = 61, 2311, 4621).
// Not used for m = 4093 (n = 4096, d = 3): 4092 = 4*3*11*31 needs a radix-31
// stage whose O(r^2) butterfly on 132 threads made the pair 3x slower than
// Bluestein on B200 (measured, round 1); the radix set stops at 13.
// With g a primitive root mod p,
//   Z_0 = sum_j z_j,   Z_{g^-q} = z_0 + sum_n z_{g^n} w_p^{g^(n-q)}  (q < p-1),
// a cyclic convolution of length N = p - 1 of a_n = z_{g^n} with
// b_n = w_p^{g^-n}, evaluated as IDFT_N(DFT_N(a) . DFT_N(b)).  DFT_N(b)/N is a
// host-built table (rbhat, stored in the digit-reversed order the in-place
// DIF transform produces), so a line pair costs one forward DIF and one
// inverse DIT mixed-radix transform of length p - 1 (4 stages each at 4092)
// in 64 KB of shared memory, instead of two 8192-point FFTs over 139 KB
// (Bluestein, fd_pair.cuh).  The input permutation n -> g^n runs through
// registers (each thread gathers its entries, barrier, scatters them back).
// Border fold, Hermitian split, packed coefficients, GCV weights and the
// filtered synthesis are the pair kernels' (fd_pair.cuh).
#pragma once

namespace fdb {

// one butterfly of a radix-R stage (block stride L, twiddle step t1; t1 = 0:
// no twiddles).  Forward (DIF): y_p = (sum_q x_q w_R^{pq}) w^{t1 p}.  Inverse
// (DIT mirror): y_p = sum_q x_q conj(w^{t1 q}) w_R^{-pq}, computed as
// conj(F_R conj(...)).  Outputs are written as soon as they are formed, so a
// radix-31 butterfly holds only the (R-1) symmetric sums / differences.
template <int R, bool INV>
__device__ __forceinline__ void rad_bfly(double2* xb, int L, int t1, const MixTw& tw) {
  auto in = [&](int q) {
    double2 a = xb[q * L];
    if (INV) {
      a = cconj(a);
      if (t1 && q) a = cmul(a, tw(t1 * q));  // conj(x conj(w)) = conj(x) w
    }
    return a;
  };
  auto put = [&](int p, double2 y) {
    if (!INV && t1 && p) y = cmul(y, tw(t1 * p));
    if (INV) y = cconj(y);
    xb[p * L] = y;
  };
  if constexpr (R == 2) {
    const double2 a = in(0), b = in(1);
    put(0, cadd(a, b));
    put(1, csub(a, b));
  } else if constexpr (R == 4) {
    const double2 x0 = in(0), x1 = in(1), x2 = in(2), x3 = in(3);
    const double2 t0 = cadd(x0, x2), u1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = csub(x1, x3);
    put(0, cadd(t0, t2));
    put(2, csub(t0, t2));
    put(1, make_double2(u1.x + t3.y, u1.y - t3.x));  // u1 - i t3
    put(3, make_double2(u1.x - t3.y, u1.y + t3.x));  // u1 + i t3
  } else {
    constexpr int H = R / 2;
    double2 s[H], d[H];
    const double2 v0 = in(0);
    double2 x0 = v0;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const double2 a = in(j), b = in(R - j);
      s[j - 1] = cadd(a, b);
      d[j - 1] = csub(a, b);
      x0 = cadd(x0, s[j - 1]);
    }
    put(0, x0);
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double2 A = v0, B = czero();
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
      put(k, make_double2(A.x + B.y, A.y - B.x));
      put(R - k, make_double2(A.x - B.y, A.y + B.x));
    }
  }
}

template <int R, bool INV>
__device__ __forceinline__ void rad_stage(double2* __restrict__ x, int N, int S, const MixTw& tw,
                                          int nt) {
  const int L = S / R, items = N / R, tstep = N / S;
  for (int it = threadIdx.x; it < items; it += nt) {
    const int blk = it / L, j = it - blk * L;
    rad_bfly<R, INV>(x + blk * S + j, L, L > 1 ? j * tstep : 0, tw);
  }
}

template <bool INV>
__device__ __forceinline__ void rad_stage_any(int r, double2* x, int N, int S, const MixTw& tw,
                                              int nt) {
  switch (r) {
    case 2: rad_stage<2, INV>(x, N, S, tw, nt); break;
    case 3: rad_stage<3, INV>(x, N, S, tw, nt); break;
    case 4: rad_stage<4, INV>(x, N, S, tw, nt); break;
    case 5: rad_stage<5, INV>(x, N, S, tw, nt); break;
    case 7: rad_stage<7, INV>(x, N, S, tw, nt); break;
    case 9: rad_stage<9, INV>(x, N, S, tw, nt); break;
    case 11: rad_stage<11, INV>(x, N, S, tw, nt); break;
    default: rad_stage<13, INV>(x, N, S, tw, nt); break;
  }
}

// cyclic convolution of x (length N = m - 1, natural order) with b:
// DIF forward, pointwise DFT(b)/N, DIT inverse -> natural order
// (length N, DFT(b)/N table `bhat` in the DIF output order; plan in ax.mrad)
__device__ __forceinline__ void rader_conv_n(double2* x, int N, const AxisDev& ax,
                                             const double2* __restrict__ bhat, const MixTw& tw,
                                             int nt) {
  int S = N;
  for (int s = 0; s < ax.mstages; ++s) {
    rad_stage_any<false>(ax.mrad[s], x, N, S, tw, nt);
    S /= ax.mrad[s];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += nt) x[i] = cmul(x[i], __ldg(&bhat[i]));
  __syncthreads();
  for (int s = ax.mstages - 1; s >= 0; --s) {
    S *= ax.mrad[s];
    rad_stage_any<true>(ax.mrad[s], x, N, S, tw, nt);
    __syncthreads();
  }
}

__device__ __forceinline__ void rader_conv(double2* x, const AxisDev& ax, const MixTw& tw, int nt) {
  const int N = ax.m - 1;
  int S = N;
  for (int s = 0; s < ax.mstages; ++s) {
    rad_stage_any<false>(ax.mrad[s], x, N, S, tw, nt);
    S /= ax.mrad[s];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < N; i += nt) x[i] = cmul(x[i], __ldg(&ax.rbhat[i]));
  __syncthreads();
  for (int s = ax.mstages - 1; s >= 0; --s) {
    S *= ax.mrad[s];
    rad_stage_any<true>(ax.mrad[s], x, N, S, tw, nt);
    __syncthreads();
  }
}

constexpr int kRadNT = 256;
// register slots of the input permutation: N <= kRadPer * kRadNT
constexpr int kRadPer = (4096 + kRadNT - 1) / kRadNT;

// smem: DFT buffer (m complex), twiddle hi / lo of w_N, g^n table (N ints),
// output positions (m ints), reduction scratch, z_0
__host__ __device__ __forceinline__ size_t rad_smem_bytes(int m) {
  const int N = m - 1;
  return (size_t)m * 16 + (size_t)(64 + ((N + 63) >> 6)) * 16 + (size_t)((N + m + 3) & ~3) * 4 +
         64 * 8 + 32;
}

struct RadSm {
  double2* x;
  MixTw tw;
  const int* gidx;
  const int* opos;
  double* red;
  double2* z0;
};
__device__ __forceinline__ RadSm rad_setup(double2* sm, const AxisDev& ax) {
  const int m = ax.m, N = m - 1, nhi = (N + 63) >> 6;
  RadSm r;
  r.x = sm;
  double2* lo = sm + m;
  double2* hi = lo + 64;
  int* gi = reinterpret_cast<int*>(hi + nhi);
  int* op = gi + N;
  r.red = reinterpret_cast<double*>(gi + ((N + m + 3) & ~3));  // 16-byte aligned
  r.z0 = reinterpret_cast<double2*>(r.red + 64);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) lo[i] = i < N ? ax.mtw[i] : czero();
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) hi[i] = ax.mtw[i << 6];
  for (int i = threadIdx.x; i < N; i += blockDim.x) gi[i] = ax.rgidx[i];
  for (int i = threadIdx.x; i < m; i += blockDim.x) op[i] = ax.ropos[i];
  r.tw = MixTw{lo, hi};
  r.gidx = gi;
  r.opos = op;
  return r;
}

// x (natural order z_0 .. z_{m-1}) -> Z in place: X_0 = sum (`zsum`),
// Z_k = z_0 + conv[opos[k]]; returns nothing, the caller reads rad_Z
__device__ __forceinline__ void rader_dft(const RadSm& r, const AxisDev& ax, double2 zsum_part) {
  const int m = ax.m, N = m - 1;
  double2* x = r.x;
  // X_0 = sum_j z_j (block reduction; deterministic order)
  double v[2] = {zsum_part.x, zsum_part.y};
  block_sum<2>(v, r.red);
  // a_n = z_{g^n}: gather through registers, then scatter back
  double2 reg[kRadPer];
#pragma unroll
  for (int t = 0; t < kRadPer; ++t) {
    const int n = threadIdx.x + t * kRadNT;
    reg[t] = n < N ? x[r.gidx[n]] : czero();
  }
  if (threadIdx.x == 0) {
    r.z0[0] = x[0];
    r.z0[1] = make_double2(v[0], v[1]);
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < kRadPer; ++t) {
    const int n = threadIdx.x + t * kRadNT;
    if (n < N) x[n] = reg[t];
  }
  __syncthreads();
  rader_conv(x, ax, r.tw, kRadNT);
}
// Z_k after rader_dft
__device__ __forceinline__ double2 rad_Z(const RadSm& r, int k) {
  return k == 0 ? r.z0[1] : cadd(r.z0[0], r.x[r.opos[k]]);
}

// analyze, two real lines per Rader DFT (see k_panalyze)
__global__ void __launch_bounds__(kRadNT, 2) k_qanalyze(AxisDev ax, LineIO io) {
  extern __shared__ double2 sm[];
  const int m = ax.m, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  const RadSm r = rad_setup(sm, ax);
  double2* x = r.x;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const long long es = io.gi.elem_stride;
  const double isq = ax.inv_sqrt_m;
  const long long nkb32 = io.wstride >> 5;
  for (int q = blockIdx.x; q < npairs; q += gridDim.x) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    auto ld0 = [&](int e) { return __ldg(g0 + e * es); };
    auto ld1 = [&](int e) { return has1 ? __ldg(g1 + e * es) : 0.0; };
    double a0[kHoMax], a1[kHoMax];
    ho_amps_real(ax, ld0, a0);
    ho_amps_real(ax, ld1, a1);
    const Cubic p0 = ho_cubic(ax, a0), p1 = ho_cubic(ax, a1);
    double2 part = czero();
#pragma unroll 8
    for (int j = threadIdx.x; j < m; j += kRadNT) {
      const int e = kl + j;
      const double t = fma((double)e, ax.ho_ta, ax.ho_tb);
      const double2 z = make_double2(ld0(e) - p0(t), ld1(e) - p1(t));
      x[j] = z;
      part = cadd(part, z);
    }
    __syncthreads();
    rader_dft(r, ax, part);

    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
    double* w0 = io.wout ? io.wout + (long long)l0 * io.wstride : nullptr;
    double* w1 = (w0 && has1) ? w0 + io.wstride : nullptr;
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
    for (int kk = threadIdx.x; kk <= h; kk += kRadNT) {
      const double2 Zk = rad_Z(r, kk);
      const double2 Zc = kk ? rad_Z(r, m - kk) : Zk;
      const double2 X0 = cscale(cadd(Zk, cconj(Zc)), 0.5 * isq);
      const double2 D = csub(Zk, cconj(Zc));
      const double2 X1 = make_double2(0.5 * isq * D.y, -0.5 * isq * D.x);
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
        const double f = kk ? 2.0 : 1.0;
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
      for (long long i = io.wn + threadIdx.x; i < io.wstride; i += kRadNT) {
        wset(l0, w0, i, 0.0);
        if (w1) wset(l0 + 1, w1, i, 0.0);
      }
    __syncthreads();
  }
}

// synthesis with the filter fused, two lines per Rader DFT (see k_psynth)
__global__ void __launch_bounds__(kRadNT, 2) k_qsynth(AxisDev ax, LineIO io, SynthArgs sa) {
  extern __shared__ double2 sm[];
  const int m = ax.m, kl = ax.kl, hk = ax.hk, h = (m - 1) / 2;
  const RadSm r = rad_setup(sm, ax);
  double2* x = r.x;
  __syncthreads();
  const int count = io.gi.count, npairs = (count + 1) / 2;
  const double* in = reinterpret_cast<const double*>(io.in);
  double* out = reinterpret_cast<double*>(io.out);
  const double isq = ax.inv_sqrt_m;
  for (int q = blockIdx.x; q < npairs; q += gridDim.x) {
    const int l0 = 2 * q;
    const bool has1 = l0 + 1 < count;
    const double* g0 = in + line_offset(io.gi, l0);
    const double* g1 = has1 ? in + line_offset(io.gi, l0 + 1) : g0;
    const double mu0 = line_mu(sa, io.gi, l0);
    const double mu1 = has1 ? line_mu(sa, io.gi, l0 + 1) : mu0;
    auto f0 = [&](int e, double2 c) { return coeff_filter_fast(ax, sa, io.gi, l0, e, c, mu0); };
    auto f1 = [&](int e, double2 c) {
      return has1 ? coeff_filter_fast(ax, sa, io.gi, l0 + 1, e, c, mu1) : czero();
    };
    auto ld0 = [&](int i) { return __ldg(g0 + i); };
    auto ld1 = [&](int i) { return has1 ? __ldg(g1 + i) : 0.0; };
    double ua0[kHoMax], ua1[kHoMax];
#pragma unroll
    for (int l = 0; l < kHoMax; ++l) {
      ua0[l] = l < hk ? f0(ho_coef_elem(ax, l), make_double2(ld0(l), 0.0)).x : 0.0;
      ua1[l] = l < hk ? f1(ho_coef_elem(ax, l), make_double2(ld1(l), 0.0)).x : 0.0;
    }
    double2 part = czero();
#pragma unroll 4
    for (int kk = threadIdx.x; kk <= h; kk += kRadNT) {
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
      // F^H v = conj(F conj v), v = X0 + i X1
      const double2 wk = make_double2(X0.x - X1.y, -(X0.y + X1.x));
      x[kk] = wk;
      part = cadd(part, wk);
      if (kk) {
        const double2 wc = make_double2(X0.x + X1.y, X0.y - X1.x);
        x[m - kk] = wc;
        part = cadd(part, wc);
      }
    }
    __syncthreads();
    rader_dft(r, ax, part);

    const Cubic p0 = ho_cubic(ax, ua0), p1 = ho_cubic(ax, ua1);
    const long long eso = io.go.elem_stride;
    double* o0 = out + line_offset(io.go, l0);
    double* o1 = has1 ? out + line_offset(io.go, l0 + 1) : nullptr;
#pragma unroll 4
    for (int p = threadIdx.x; p < m; p += kRadNT) {
      const double2 z = rad_Z(r, p);
      const double y0 = z.x * isq, y1 = -z.y * isq;
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
  }
}

}  // namespace fdb
