// Input generation on the GPU: the "true-extended" blur and
// the noise model the reference uses to build its observations,
//   convolve_valid / convolve_valid_2d   (pipeline.cpp:14-51)
//   add_noise                            (operators.cpp:332-358; SplitMix64
//                                         operators.cpp:78-90, Box-Muller)
// so a benchmark scene never has to cross the host link.  Every sample is a
// pure function of (seed, index), as in the reference: the kernels evaluate the
// counter-based stream in place.  Sums run in a fixed order (per-thread
// strided partials, shuffle tree, warp order), so results are reproducible;
// they differ from the reference's sequential sums by rounding only.
#pragma once

#include <stdint.h>

namespace fdb {

// g_i = sum_j h_j f_{i+j}, j = -m..m, the mask inside the extended line
// (pipeline.cpp:14-29); one thread per output sample, taps in the reference's
// order.  ext: [count][n + 2m], out: [count][n].
__global__ void __launch_bounds__(256) k_convolve_valid(const double* __restrict__ ext,
                                                        const double* __restrict__ h, int m, int n,
                                                        long long count, double* __restrict__ out) {
  extern __shared__ double hs[];
  for (int j = threadIdx.x; j < 2 * m + 1; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  const long long total = count * n;
  const int w = n + 2 * m;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long item = t / n;
    const int i = (int)(t - item * n);
    const double* f = ext + item * w + i;
    double acc = 0.0;
    for (int j = 0; j <= 2 * m; ++j) acc += hs[j] * __ldg(f + j);
    out[t] = acc;
  }
}

// 2D: g_ik = sum_jl h_jl f_{i+j,k+l} (pipeline.cpp:31-51); ext: [count][rows][cols]
// with rows = n1 + 2 m1, cols = n2 + 2 m2; taps row-major, in the reference's order.
__global__ void __launch_bounds__(256) k_convolve_valid_2d(const double* __restrict__ ext,
                                                           const double* __restrict__ h, int m1,
                                                           int m2, int n1, int n2, long long count,
                                                           double* __restrict__ out) {
  extern __shared__ double hs[];
  const int t1 = 2 * m1 + 1, t2 = 2 * m2 + 1;
  for (int j = threadIdx.x; j < t1 * t2; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  const long long per = (long long)n1 * n2, total = count * per;
  const int cols = n2 + 2 * m2;
  const long long eper = (long long)(n1 + 2 * m1) * cols;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long item = t / per;
    const long long r = t - item * per;
    const int i = (int)(r / n2), k = (int)(r - (long long)i * n2);
    const double* f = ext + item * eper + (long long)i * cols + k;
    double acc = 0.0;
    for (int j = 0; j < t1; ++j) {
      const double* fr = f + (long long)j * cols;
      const double* hr = hs + j * t2;
      for (int l = 0; l < t2; ++l) acc += hr[l] * __ldg(fr + l);
    }
    out[t] = acc;
  }
}

__device__ __forceinline__ uint64_t gen_splitmix64(uint64_t x) {  // operators.cpp:78-85
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}
__device__ __forceinline__ double gen_u01(uint64_t bits) {  // (0, 1], operators.cpp:88-90
  return ((double)(bits >> 11) + 1.0) * 0x1p-53;
}
// the Box-Muller pair p of the stream `seed` (operators.cpp:343-350)
__device__ __forceinline__ void gen_eta_pair(uint64_t seed, long long p, double& e0, double& e1) {
  const uint64_t golden = 0x9E3779B97F4A7C15ULL;
  const double u1 = gen_u01(gen_splitmix64(seed + (2ULL * (uint64_t)p + 1ULL) * golden));
  const double u2 = gen_u01(gen_splitmix64(seed + (2ULL * (uint64_t)p + 2ULL) * golden));
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  double s, c;
  sincos(ang, &s, &c);
  e0 = r * c;
  e1 = r * s;
}

// partial sums (|g|^2, |eta|^2) of item blockIdx.y over the pairs this CTA
// owns: part[(item * gridDim.x + blockIdx.x) * 2 + {0, 1}]
__global__ void __launch_bounds__(256) k_noise_norms(const double* __restrict__ g, long long n,
                                                     const uint64_t* __restrict__ seeds,
                                                     double* __restrict__ part) {
  __shared__ double red[32 * 2];
  const long long item = blockIdx.y;
  const double* gi = g + item * n;
  const uint64_t seed = seeds[item];
  const long long pairs = (n + 1) / 2;
  double v[2] = {0.0, 0.0};
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs;
       p += (long long)gridDim.x * blockDim.x) {
    double e0, e1;
    gen_eta_pair(seed, p, e0, e1);
    const double a = gi[2 * p];
    v[0] += a * a;
    v[1] += e0 * e0;
    if (2 * p + 1 < n) {
      const double b = gi[2 * p + 1];
      v[0] += b * b;
      v[1] += e1 * e1;
    }
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    part[(item * gridDim.x + blockIdx.x) * 2] = v[0];
    part[(item * gridDim.x + blockIdx.x) * 2 + 1] = v[1];
  }
}

// g += level sqrt(|g|^2 / |eta|^2) eta (operators.cpp:351-356); the partials are
// added in CTA order by every thread (fixed order)
__global__ void __launch_bounds__(256) k_noise_apply(double* __restrict__ g, long long n,
                                                     const uint64_t* __restrict__ seeds,
                                                     const double* __restrict__ part, int nparts,
                                                     double level) {
  const long long item = blockIdx.y;
  double gn = 0.0, en = 0.0;
  for (int c = 0; c < nparts; ++c) {
    gn += part[(item * nparts + c) * 2];
    en += part[(item * nparts + c) * 2 + 1];
  }
  if (en == 0.0) return;
  const double scale = level * sqrt(gn / en);
  double* gi = g + item * n;
  const uint64_t seed = seeds[item];
  const long long pairs = (n + 1) / 2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs;
       p += (long long)gridDim.x * blockDim.x) {
    double e0, e1;
    gen_eta_pair(seed, p, e0, e1);
    gi[2 * p] += scale * e0;
    if (2 * p + 1 < n) gi[2 * p + 1] += scale * e1;
  }
}

}  // namespace fdb
