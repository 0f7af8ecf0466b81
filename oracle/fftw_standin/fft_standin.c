/*
 * TEST INFRASTRUCTURE ONLY (oracle/). Never linked into the product library.
 *
 * O(n log n) stand-in for the three FFTW3 calls the reference makes
 * (reference: proj/core/src/trig.cpp:53-70 plan cache, 105-112 execute).
 * FFTW 3.x (unpinned: found via find_library, core/CMakeLists.txt:1-2) is
 * absent from this image; this file restates its published contract:
 *
 *   out_k = sum_{j<n} in_j * exp(sign * 2*pi*i * j*k / n)    (unnormalised)
 *
 * Algorithm: recursive mixed-radix decimation in time, smallest prime factor
 * first; prime lengths <= 128 by a direct O(p^2) DFT on the exact twiddle
 * table (73, 89, 23, 7 at the BASELINE sizes), larger primes (8191) by the
 * Bluestein chirp-z convolution on a power-of-two FFT. Twiddles are computed
 * per entry with cos/sin of 2*pi*j/n (no recurrences), so the stand-in is
 * accurate to a few ulp, which the reference's own dense-matrix tests demand
 * (test_trig.cpp:103-125, <= 1e-13).
 *
 * Thread safety: plans are immutable after creation; every execute allocates
 * its own scratch, so concurrent executes on one plan are safe (the reference
 * relies on this, trig.cpp:95-112).
 */
#include "fftw3.h"

#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cx;

#define DIRECT_PRIME_MAX 128
#define MAX_BLUE 16

typedef struct {
  int L;                          /* prime length handled by Bluestein */
  int M;                          /* power-of-two convolution length   */
  cx* chirp;                      /* L entries exp(sign*i*pi*j^2/L)    */
  cx* bhat;                       /* FFT_M(b) / M                      */
  struct fd_standin_plan_s* fwd;  /* size-M plans (power of two)      */
  struct fd_standin_plan_s* bwd;
} blue_t;

struct fd_standin_plan_s {
  int n;
  int sign;
  cx* tw; /* tw[j] = exp(sign * 2 pi i j / n), j < n */
  int nblue;
  blue_t blue[MAX_BLUE];
};

static int smallest_factor(int n) {
  if (n % 2 == 0) return 2;
  for (int p = 3; (long)p * p <= n; p += 2)
    if (n % p == 0) return p;
  return n;
}

static struct fd_standin_plan_s* plan_create(int n, int sign);

static void add_blue(struct fd_standin_plan_s* P, int L) {
  for (int i = 0; i < P->nblue; ++i)
    if (P->blue[i].L == L) return;
  blue_t* b = &P->blue[P->nblue++];
  b->L = L;
  int M = 1;
  while (M < 2 * L - 1) M <<= 1;
  b->M = M;
  b->chirp = (cx*)malloc(sizeof(cx) * (size_t)L);
  for (int j = 0; j < L; ++j) {
    /* j^2 mod 2L keeps the angle argument small and exact */
    const int64_t q = ((int64_t)j * j) % (2 * (int64_t)L);
    const double ang = (double)P->sign * M_PI * (double)q / (double)L;
    b->chirp[j] = cos(ang) + I * sin(ang);
  }
  b->fwd = plan_create(M, FFTW_FORWARD);
  b->bwd = plan_create(M, FFTW_BACKWARD);
  cx* bb = (cx*)calloc((size_t)M, sizeof(cx));
  bb[0] = conj(b->chirp[0]);
  for (int j = 1; j < L; ++j) {
    bb[j] = conj(b->chirp[j]);
    bb[M - j] = conj(b->chirp[j]);
  }
  b->bhat = (cx*)malloc(sizeof(cx) * (size_t)M);
  fftw_execute_dft(b->fwd, (fftw_complex*)bb, (fftw_complex*)b->bhat);
  for (int j = 0; j < M; ++j) b->bhat[j] /= (double)M;
  free(bb);
}

static struct fd_standin_plan_s* plan_create(int n, int sign) {
  struct fd_standin_plan_s* P =
      (struct fd_standin_plan_s*)calloc(1, sizeof(struct fd_standin_plan_s));
  P->n = n;
  P->sign = sign;
  P->tw = (cx*)malloc(sizeof(cx) * (size_t)n);
  for (int j = 0; j < n; ++j) {
    const double ang = (double)sign * 2.0 * M_PI * (double)j / (double)n;
    P->tw[j] = cos(ang) + I * sin(ang);
  }
  int r = n;
  while (r > 1) {
    const int p = smallest_factor(r);
    if (p > DIRECT_PRIME_MAX) add_blue(P, p);
    while (r % p == 0) r /= p;
  }
  return P;
}

/* DFT of prime length p; W_p^j = P->tw[j * tws] */
static void prime_dft(const struct fd_standin_plan_s* P, int p, const cx* in, long is,
                      cx* out, long tws) {
  if (p <= DIRECT_PRIME_MAX) {
    for (int k = 0; k < p; ++k) {
      cx acc = 0;
      int idx = 0;
      for (int j = 0; j < p; ++j) {
        acc += in[j * is] * P->tw[idx * tws];
        idx += k;
        if (idx >= p) idx -= p;
      }
      out[k] = acc;
    }
    return;
  }
  const blue_t* b = NULL;
  for (int i = 0; i < P->nblue; ++i)
    if (P->blue[i].L == p) b = &P->blue[i];
  const int M = b->M;
  cx* a = (cx*)calloc((size_t)M, sizeof(cx));
  cx* A = (cx*)malloc(sizeof(cx) * (size_t)M);
  for (int j = 0; j < p; ++j) a[j] = in[j * is] * b->chirp[j];
  fftw_execute_dft(b->fwd, (fftw_complex*)a, (fftw_complex*)A);
  for (int j = 0; j < M; ++j) A[j] *= b->bhat[j];
  fftw_execute_dft(b->bwd, (fftw_complex*)A, (fftw_complex*)a);
  for (int k = 0; k < p; ++k) out[k] = a[k] * b->chirp[k];
  free(a);
  free(A);
}

/* out[0..n) = DFT_n(in[0], in[is], ...); W_n^j = P->tw[j * tws] */
static void dft_rec(const struct fd_standin_plan_s* P, int n, const cx* in, long is,
                    cx* out, long tws) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  if (n == 2) {
    const cx x0 = in[0], x1 = in[is];
    out[0] = x0 + x1;
    out[1] = x0 - x1;
    return;
  }
  const int p = smallest_factor(n);
  if (p == n) {
    prime_dft(P, n, in, is, out, tws);
    return;
  }
  const int m = n / p;
  for (int r = 0; r < p; ++r) dft_rec(P, m, in + r * is, is * p, out + r * m, tws * p);
  if (p == 2) {
    for (int k = 0; k < m; ++k) {
      const cx t0 = out[k];
      const cx t1 = out[k + m] * P->tw[(long)k * tws];
      out[k] = t0 + t1;
      out[k + m] = t0 - t1;
    }
    return;
  }
  cx tbuf[DIRECT_PRIME_MAX], xbuf[DIRECT_PRIME_MAX];
  cx* t = p <= DIRECT_PRIME_MAX ? tbuf : (cx*)malloc(sizeof(cx) * (size_t)p);
  cx* x = p <= DIRECT_PRIME_MAX ? xbuf : (cx*)malloc(sizeof(cx) * (size_t)p);
  for (int k = 0; k < m; ++k) {
    for (int r = 0; r < p; ++r) t[r] = out[k + r * m] * P->tw[((long)r * k) * tws];
    prime_dft(P, p, t, 1, x, tws * m);
    for (int q = 0; q < p; ++q) out[k + q * m] = x[q];
  }
  if (p > DIRECT_PRIME_MAX) {
    free(t);
    free(x);
  }
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  (void)in;
  (void)out;
  (void)flags;
  if (n < 1 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return NULL;
  return plan_create(n, sign);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const cx* src = (const cx*)in;
  cx* copy = NULL;
  if ((void*)in == (void*)out) {
    copy = (cx*)malloc(sizeof(cx) * (size_t)p->n);
    memcpy(copy, in, sizeof(cx) * (size_t)p->n);
    src = copy;
  }
  dft_rec(p, p->n, src, 1, (cx*)out, 1);
  free(copy);
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  for (int i = 0; i < p->nblue; ++i) {
    free(p->blue[i].chirp);
    free(p->blue[i].bhat);
    fftw_destroy_plan(p->blue[i].fwd);
    fftw_destroy_plan(p->blue[i].bwd);
  }
  free(p->tw);
  free(p);
}
