// Real lines of a cosine basis (hoc-cosine, reflective) whose half length
// h = m/2 is an odd prime with h - 1 a product of 2, 3, 4, 5, 7, 9, 11, 13:
// BASELINE config 4 (n = 16384: m = 16382 = 2 * 8191, 8190 = 13 * 9 * 7 * 5 * 2).
//
// The DCT-II / DCT-III of the line is a complex DFT of length h on the
// interleaved Makhoul sequence plus an O(h) split (k_ranalyze / k_rsynth).
// Bluestein needs M = 16384 >= 2h - 1 for that DFT, which does not fit in
// shared memory: round 1 ran it as two half-size convolutions with a per-CTA
// global scratch line (12.9 ms per 16384^2 pass, 1.4x the algorithmic DRAM
// traffic).  Here the DFT is Rader's: with g a primitive root mod h,
//   Z_0 = sum_j z_j,   Z_{g^-q} = z_0 + (a * b)_q,  a_n = z_{g^n},  b_n = w_h^{g^-n},
// a cyclic convolution of length N = h - 1 evaluated in 131 KB of shared
// memory as inverse-DIT(DIF(a) . DFT(b)/N) over the mixed-radix stages of
// fd_rader.cuh -- no scratch, no chirp, ~60 % of Bluestein's arithmetic.  The
// load phase scatters sample j straight to its convolution slot (ilog[j]), the
// post phase gathers frequency k from opos[k]: no permutation pass.
// One persistent CTA of 512 threads per SM; the next line is prefetched into L2
// while the current one is in flight.
#pragma once

namespace fdb {

constexpr int kCdNT = 512;

struct CdSm {
  double2* x;     // N convolution slots
  MixTw tw;       // twiddles of w_N
  Tw2 rtw, dtw;   // real-FFT and DCT quarter-wave twiddles (as k_ranalyze)
  const unsigned short* ilog;  // sample j >= 1 -> convolution slot
  const unsigned short* opos;  // frequency k >= 1 -> convolution slot
  double* red;
  double2* z0;    // [0] = z_0, [1] = Z_0
};

// shared memory: x[N] | lo[64] hi[(N+63)/64] | rtw | dtw | ilog[h] opos[h] (u16) | red[64] | z0[2]
__host__ __device__ __forceinline__ size_t cd_smem_bytes(int h, int m) {
  const int N = h - 1;
  size_t b = (size_t)N * 16 + (size_t)(64 + ((N + 63) >> 6)) * 16;
  b += (size_t)(tw2_slots(h) + tw2_slots(m)) * 16;
  b += (size_t)((2 * h + 7) & ~7) * 2;
  b += 64 * 8 + 2 * 16;
  return b;
}

__device__ __forceinline__ CdSm cd_setup(double2* sm, const AxisDev& ax) {
  const int h = ax.hfft.L, N = h - 1, nhi = (N + 63) >> 6;
  CdSm r;
  r.x = sm;
  double2* lo = sm + N;
  double2* hi = lo + 64;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) lo[i] = i < N ? ax.mtw[i] : czero();
  for (int i = threadIdx.x; i < nhi; i += blockDim.x) hi[i] = ax.mtw[i << 6];
  r.tw = MixTw{lo, hi};
  double2* s1 = hi + nhi;
  r.rtw = load_tw2(s1, ax.rtw, h);
  double2* s2 = s1 + tw2_slots(h);
  r.dtw = load_tw2(s2, ax.dct_tw, ax.m);
  unsigned short* il = reinterpret_cast<unsigned short*>(s2 + tw2_slots(ax.m));
  unsigned short* op = il + h;
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    il[i] = (unsigned short)ax.cd_ilog[i];
    op[i] = (unsigned short)ax.cd_opos[i];
  }
  r.ilog = il;
  r.opos = op;
  r.red = reinterpret_cast<double*>(il + ((2 * h + 7) & ~7));
  r.z0 = reinterpret_cast<double2*>(r.red + 64);
  return r;
}

__device__ __forceinline__ double2 cd_Z(const CdSm& r, int k) {
  return k == 0 ? r.z0[1] : cadd(r.z0[0], r.x[r.opos[k]]);
}

__device__ __forceinline__ void cd_prefetch(const void* base, const Lines& g, int l, int n) {
  if (threadIdx.x != 0 || g.elem_stride != 1 || l >= g.count) return;
  const double* src = reinterpret_cast<const double*>(base) + line_offset(g, l);
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (n & 1) == 0)
    bulk_prefetch_l2(src, (uint32_t)n * 8);
}

// analyze: T_X^{-1} of real lines (cosine interior), as k_ranalyze
__global__ void __launch_bounds__(kCdNT, 1) k_canalyze(AxisDev ax, LineIO io) {
  extern __shared__ double2 sm[];
  const int h = ax.hfft.L, N = h - 1, n = ax.n, m = ax.m;
  const CdSm r = cd_setup(sm, ax);
  double2* x = r.x;
  __syncthreads();
  const double* in = reinterpret_cast<const double*>(io.in);
  const long long es = io.gi.elem_stride;
  const int half = (m + 1) / 2;
  const double s0 = ax.dct_s0, s1 = ax.dct_s1;
  const long long nkb32 = io.wstride >> 5;
  for (int l = blockIdx.x; l < io.gi.count; l += gridDim.x) {
    const double* gin = in + line_offset(io.gi, l);
    auto ld = [&](int e) { return __ldg(gin + (long long)e * es); };
    const Fold fd = fold_terms(ax, ld);
    double2 part = czero();
#pragma unroll 4
    for (int j = threadIdx.x; j < h; j += kCdNT) {
      const double a = ld(interior_elem(ax, makhoul_src(2 * j, m, half)));
      const double b = ld(interior_elem(ax, makhoul_src(2 * j + 1, m, half)));
      const double2 z = make_double2(a, b);
      part = cadd(part, z);
      if (j == 0)
        r.z0[0] = z;
      else
        x[r.ilog[j]] = z;
    }
    double v[2] = {part.x, part.y};
    block_sum<2>(v, r.red);  // barriers inside: x and z0[0] are complete after it
    if (threadIdx.x == 0) r.z0[1] = make_double2(v[0], v[1]);
    rader_conv_n(x, N, ax, ax.cd_bhat, r.tw, kCdNT);
    cd_prefetch(io.in, io.gi, l + gridDim.x, n);

    const long long oo = line_offset(io.go, l), eso = io.go.elem_stride;
    double* out = reinterpret_cast<double*>(io.out);
    double* wl = io.wout ? io.wout + (long long)l * io.wstride : nullptr;
    auto wset = [&](long long i, double val) {
      wl[i] = val;
      if (io.wout32) {
        float hi, lo;
        tf32_split(val, hi, lo);
        const long long t = tc_tile_index(l, i, kTcBM, nkb32);
        io.wout32[t] = hi;
        io.wout32lo[t] = lo;
      }
    };
    if (wl)
      for (long long i = io.wn + threadIdx.x; i < io.wstride; i += kCdNT) wset(i, 0.0);
    const bool brd = ax.bordered != 0;
    auto emit = [&](int i, double val) {  // interior coefficient i (boundary.cpp:271-287)
      if (brd) val += fd.c0 * __ldg(&ax.vr[i]) + fd.c1 * __ldg(&ax.wr[i]);
      const int e = interior_elem(ax, i);
      if (io.out_cplx)
        stc(io.out, 1, oo + e * eso, make_double2(val, 0.0));
      else if (eso == 1)
        __stcs(out + oo + e, val);  // streamed: keep L2 for the prefetched input
      else
        out[oo + e * eso] = val;  // column pass: neighbouring CTAs complete the sector in L2
      if (wl) wset(e, val * val);
    };
#pragma unroll 2
    for (int k = threadIdx.x; k < h; k += kCdNT) {
      const int kc = k == 0 ? 0 : h - k;
      const double2 Zk = cd_Z(r, k);
      const double2 Zc = cconj(cd_Z(r, kc));
      const double2 E = cscale(cadd(Zk, Zc), 0.5);
      const double2 D = csub(Zk, Zc);
      const double2 WO = cmul(r.rtw(k), make_double2(0.5 * D.y, -0.5 * D.x));
      const double2 X0 = cadd(E, WO), X1 = csub(E, WO);  // X_k, X_{k+h}
      const double2 t0 = r.dtw(k), t1 = r.dtw(k + h);
      emit(k, (k == 0 ? s0 : s1) * (t0.x * X0.x - t0.y * X0.y));
      emit(k + h, s1 * (t1.x * X1.x - t1.y * X1.y));
    }
    if (brd && threadIdx.x == 0) {
      stc(io.out, io.out_cplx, oo, make_double2(fd.o0, 0.0));
      stc(io.out, io.out_cplx, oo + (long long)(n - 1) * eso, make_double2(fd.on, 0.0));
      if (wl) {
        wset(0, fd.o0 * fd.o0);
        wset(n - 1, fd.on * fd.on);
      }
    }
    __syncthreads();  // x, z0 are reused by the next line
  }
}

// synthesis T_X c with the filter / matvec scale fused, as k_rsynth (cosine)
__global__ void __launch_bounds__(kCdNT, 1) k_csynth(AxisDev ax, LineIO io, SynthArgs sa) {
  extern __shared__ double2 sm[];
  const int h = ax.hfft.L, N = h - 1, n = ax.n, m = ax.m;
  const CdSm r = cd_setup(sm, ax);
  double2* x = r.x;
  __syncthreads();
  const double s0 = ax.dct_s0, s1 = ax.dct_s1;
  const int half = (m + 1) / 2;
  for (int l = blockIdx.x; l < io.gi.count; l += gridDim.x) {
    const long long oi = line_offset(io.gi, l);
    const double mu = line_mu(sa, io.gi, l);
    auto cf = [&](int e) {
      return coeff_filter_fast(ax, sa, io.gi, l, e,
                               ldc(io.in, io.in_cplx, oi + e * io.gi.elem_stride), mu);
    };
    double u0 = 0.0, un = 0.0;
    if (ax.bordered) {
      u0 = cf(0).x;
      un = cf(n - 1).x;
    }
    // conj(buf_i) = s_i c_i conj(tw_i) (DCT-III, trig.cpp:147-158)
    auto val_at = [&](int i) {
      const double2 c = cf(interior_elem(ax, i));
      const double2 t = r.dtw(i);
      const double ts = (i == 0 ? s0 : s1) * c.x;
      return make_double2(ts * t.x, -(ts * t.y));
    };
    double2 part = czero();
    auto place = [&](int k, double2 w) {
      part = cadd(part, w);
      if (k == 0)
        r.z0[0] = w;
      else
        x[r.ilog[k]] = w;
    };
    // C2R pre-pass over the closed index groups {k, h-k} (k_rsynth)
    for (int k = threadIdx.x; k <= h / 2; k += kCdNT) {
      const int kp = k == 0 ? 0 : h - k;
      const double2 vk = val_at(k), vkh = val_at(k + h);
      const double2 vp = kp != k ? val_at(kp) : vk, vph = kp != k ? val_at(kp + h) : vkh;
      const double2 Xk = cscale(cadd(vk, cconj(k == 0 ? vk : vph)), 0.5);
      const double2 Xkh = cscale(cadd(vkh, cconj(k == 0 ? vkh : vp)), 0.5);
      const double2 Xp = cscale(cadd(vp, cconj(k == 0 ? vp : vkh)), 0.5);
      const double2 Xph = cscale(cadd(vph, cconj(k == 0 ? vph : vk)), 0.5);
      auto zin = [&](int kk, double2 Xa, double2 Xb) {
        const double2 Od = cmulc(csub(Xa, Xb), r.rtw(kk));
        const double2 Ev = cadd(Xa, Xb);
        return make_double2(Ev.x - Od.y, Ev.y + Od.x);
      };
      place(k, cconj(zin(k, Xk, Xkh)));
      if (kp != k) place(kp, cconj(zin(kp, Xp, Xph)));
    }
    double v[2] = {part.x, part.y};
    block_sum<2>(v, r.red);
    if (threadIdx.x == 0) r.z0[1] = make_double2(v[0], v[1]);
    rader_conv_n(x, N, ax, ax.cd_bhat, r.tw, kCdNT);
    cd_prefetch(io.in, io.gi, l + gridDim.x, n);

    const long long oo = line_offset(io.go, l), eso = io.go.elem_stride;
    double* out = reinterpret_cast<double*>(io.out);
    const BorderPoly bp = border_poly(ax, u0, un);
    auto put = [&](int p, double val) {
      const int e = interior_elem(ax, p);
      if (ax.bordered) val += bp(p);
      if (eso == 1)
        __stcs(out + oo + e, val);
      else
        out[oo + e * eso] = val;
    };
#pragma unroll 2
    for (int j = threadIdx.x; j < h; j += kCdNT) {
      const double2 z = cconj(cd_Z(r, j));
      const int p0 = 2 * j, p1 = 2 * j + 1;
      put(p0 < half ? 2 * p0 : 2 * (m - 1 - p0) + 1, z.x);
      put(p1 < half ? 2 * p1 : 2 * (m - 1 - p1) + 1, z.y);
    }
    if (ax.bordered && threadIdx.x == 0) {
      auto interior_at = [&](int p) {
        const int sp = (p % 2 == 0) ? p / 2 : m - 1 - (p - 1) / 2;
        const double2 z = cconj(cd_Z(r, sp >> 1));
        return (sp & 1) ? z.y : z.x;
      };
      const double top = ax.correction ? interior_at(ax.top_i) : 0.0;
      const double bot = ax.correction ? interior_at(ax.bot_i) : 0.0;
      out[oo] = ax.q0 * u0 + top;
      out[oo + (long long)(n - 1) * eso] = bot + ax.q0 * un;
    }
    __syncthreads();
  }
}

}  // namespace fdb
