// GCV grid screening on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// gcv_minimize (reference src/regularize.cpp:144-214) needs, per item, the
// first minimum of G(mu_k) = num_k / den_k^2 over the log grid, with
//   num_k = sum_e W_e sigma_e(mu_k)^2,  den_k = sum_e mult_e sigma_e(mu_k),
// W_e = |ghat_e|^2 (Hermitian pairs summed), sigma_e = 1/(r_e + mu_k).  den is
// item-independent (one fp64 table); num is the items x K product W . S2.
//
// Screening: num~ = W32 . S32 on the tensor cores in TF32 (fp32 accumulate in
// TMEM), S32 = S2 scaled to <= 1 per grid column.  TF32 truncates each input
// to 10 mantissa bits (< 2^-10 relative) and the fp32 accumulation of positive
// terms adds < n_mma 2^-23; for the BASELINE sizes the total is < 3e-3, and
// the candidates are every k with G~_k <= (1 + tau) min G~, tau = 1e-2.  The
// exact fp64 G is then evaluated for the candidates only (k_gcv_exact); the
// others are written as +inf, so the first-minimum / tie / bracket logic of
// gcv_pick sees exactly the values that matter.  Items whose screen is not
// trustworthy (non-finite or non-positive G~, too many candidates) evaluate
// every grid point exactly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fd_internal.h"

namespace fdb {

constexpr int kTcBM = 128;     // items per CTA (UMMA M)
constexpr int kTcBK = 32;      // elements per tile (the K extent of one stored tile)
// elements per pipeline stage: half a tile.  The tile is chunk-major (16-byte
// chunks of 4 elements for all rows, see tc_tile_index), so each half is one
// contiguous block and the stage is still one bulk copy per operand; halving
// the stage doubles the number of stages that fit, so the producer refills at
// a finer grain.  tc_stages() sizes them for two CTAs per SM (2 stages per CTA
// at BN = 256 with the hi/lo split), so one CTA's epilogue overlaps the other's
// copies.
constexpr int kTcSK = 16;
// candidate tolerance tau (screen_tau): a relative error bound eps of num~,
//   single TF32 pass: 2 * 2^-10 (input truncation) + accumulation,
//   3xTF32 split:     3 * 2^-21 (hi/lo products)  + accumulation,
// accumulation = (MMAs into TMEM + products summed inside them) * 2^-23, and
// tau = 2.5 eps >= 2 eps / (1 - eps): the true minimum always survives.
__host__ __device__ inline double screen_tau(long long Ep, bool split) {
  const double acc = ((split ? 3.0 : 1.0) * (double)Ep / 8.0 + (double)Ep / 4.0) * 0x1p-23;
  const double eps = (split ? 3.0 * 0x1p-21 : 2.0 * 0x1p-10) + acc;
  return 2.5 * eps;
}
constexpr int kScreenMaxCand = 48;

// shared-memory matrix descriptor, K-major, no swizzle: core matrices of
// 8 rows x 16 bytes; lbo = byte distance between the two 16-byte K chunks of
// one MMA, sbo = byte distance between 8-row groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, layout type 0 (no swizzle)
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// 32 lanes x 32 columns of fp32 from TMEM: thread i of the warp gets lane
// (warp base + i), columns [col, col + 32)
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__host__ __device__ constexpr int tc_tmem_cols(int n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}
__host__ __device__ constexpr int tc_stage_bytes(int BN, bool split) {
  return (split ? 2 : 1) * (kTcBM + BN) * kTcSK * 4;
}
// as many stages as fit in half the SM's shared memory (at least 2): two CTAs
// per SM, so one CTA's TMEM epilogue overlaps the other's bulk copies
// (k_gcv_screen 0.32 -> 0.29 ms at config 1; one CTA with 4 stages before)
__host__ __device__ constexpr int tc_stages(int BN, bool split) {
  return (110 * 1024) / tc_stage_bytes(BN, split) < 2 ? 2
         : (110 * 1024) / tc_stage_bytes(BN, split) > 6 ? 6
                                                        : (110 * 1024) / tc_stage_bytes(BN, split);
}
__host__ __device__ constexpr size_t tc_smem_bytes(int BN, bool split) {
  return (size_t)tc_stages(BN, split) * tc_stage_bytes(BN, split) + 8 * (2 * 6 + 1) + 16 + 1024;
}

// Tiled operand layout (what one pipeline stage copies with a single bulk
// copy): the matrix is cut into tiles of ROWS x 32 fp32 (rows padded to the
// tile), tile (rb, kb) at ((rb * nkb) + kb) * ROWS * 32 floats, and inside a
// tile element (r, e) sits in the UMMA K-major no-swizzle arrangement
//   chunk c = e / 4 at c * ROWS * 4 floats, row group r / 8 at 32 floats,
//   row r % 8 at 4 floats, e % 4.
__host__ __device__ __forceinline__ long long tc_tile_index(long long row, long long e, int rows,
                                                           long long nkb) {
  const long long rb = row / rows, r = row % rows, kb = e >> 5, ee = e & 31;
  return ((rb * nkb + kb) * rows + 0) * 32 + (ee >> 2) * (rows * 4) + (r >> 3) * 32 +
         (r & 7) * 4 + (ee & 3);
}

// TF32 split of a value: hi = the leading 10 mantissa bits (what the tensor
// core reads), lo = the fp32 rest.  hi + tf32(lo) is within 2^-21 relative.
__device__ __forceinline__ void tf32_split(double v, float& hi, float& lo) {
  const float f = (float)v;
  hi = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
  lo = (float)(v - (double)hi);
}

// One CTA: items [row0, row0 + 128) against BN (>= K, multiple of 32) grid
// columns.  A = W32 tiles (hi, and lo when SPLIT), B = S32 tiles (hi, lo).
// Warp 0 lane 0 streams the stages with bulk copies, warp 1 lane 0 issues the
// MMAs (3 per K step with SPLIT: AhBh + AhBl + AlBh), all four warps run the
// epilogue.  Output per item: 8 words of candidate mask and a flag = 1 when
// the screen must not be trusted.  gscale_k = S2max_k / den_k^2.
template <int BN, bool SPLIT>
__global__ void __launch_bounds__(128, 2)
    k_gcv_screen(const float* __restrict__ Ah, const float* __restrict__ Al, int items,
                 const float* __restrict__ Bh, const float* __restrict__ Bl, int nkb, int K,
                 const double* __restrict__ gscale, float tau, uint32_t* __restrict__ mask,
                 int* __restrict__ flag) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int NA = SPLIT ? 2 : 1, NB = SPLIT ? 2 : 1;
  constexpr int ABYTES = kTcBM * kTcSK * 4;
  constexpr int BBYTES = BN * kTcSK * 4;
  constexpr int NSUB = kTcBK / kTcSK;  // stages per stored tile
  const int nsb = nkb * NSUB;
  constexpr int STAGE = NA * ABYTES + NB * BBYTES;
  constexpr int NST = tc_stages(BN, SPLIT);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  uint64_t* done = empty + NST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rb = blockIdx.x;
  constexpr uint32_t NCOLS = tc_tmem_cols(BN);

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));

  if (warp == 0 && lane == 0) {  // producer
    for (int kb = 0; kb < nsb; ++kb) {
      const int s = kb % NST;
      mbar_wait(&empty[s], (uint32_t)(((kb / NST) & 1) ^ 1));
      mbar_expect_tx(&full[s], STAGE);
      uint8_t* dst = smem + s * STAGE;
      const int t = kb / NSUB, half = kb % NSUB;
      const long long ta = ((long long)rb * nkb + t) * (kTcBM * kTcBK) + half * (kTcBM * kTcSK);
      const long long tb = (long long)t * (BN * kTcBK) + half * (BN * kTcSK);
      bulk_g2s(dst, Ah + ta, ABYTES, &full[s]);
      if (SPLIT) bulk_g2s(dst + ABYTES, Al + ta, ABYTES, &full[s]);
      bulk_g2s(dst + NA * ABYTES, Bh + tb, BBYTES, &full[s]);
      if (SPLIT) bulk_g2s(dst + NA * ABYTES + BBYTES, Bl + tb, BBYTES, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    constexpr uint32_t IDESC = idesc_tf32(kTcBM, BN);
    for (int kb = 0; kb < nsb; ++kb) {
      const int s = kb % NST;
      mbar_wait(&full[s], (uint32_t)((kb / NST) & 1));
      tc_fence_after();
      const uint32_t a_h = sbase + s * STAGE, a_l = a_h + ABYTES;
      const uint32_t b_h = a_h + NA * ABYTES, b_l = b_h + BBYTES;
#pragma unroll
      for (int kk = 0; kk < kTcSK / 8; ++kk) {  // MMA K = 8 tf32 = two 16-byte chunks
        const uint32_t ao = 2 * kk * (kTcBM * 16), bo = 2 * kk * (BN * 16);
        const uint64_t dah = umma_desc(a_h + ao, kTcBM * 16, 128);
        const uint64_t dbh = umma_desc(b_h + bo, BN * 16, 128);
        tc_mma_tf32(tmem, dah, dbh, IDESC, (kb | kk) != 0);
        if (SPLIT) {
          tc_mma_tf32(tmem, dah, umma_desc(b_l + bo, BN * 16, 128), IDESC, 1);
          tc_mma_tf32(tmem, umma_desc(a_l + ao, kTcBM * 16, 128), dbh, IDESC, 1);
        }
      }
      tc_commit(&empty[s]);  // frees the stage when these MMAs have read it
    }
    tc_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();

  // epilogue: thread = item row (TMEM lane warp*32 + lane)
  const int item = rb * kTcBM + warp * 32 + lane;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  double best = INFINITY;
  bool bad = false;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    float v[32];
    tmem_ld32(lane_addr + c0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int k = c0 + i;
      if (k < K) {
        const double G = (double)v[i] * __ldg(&gscale[k]);
        // underflowed / overflowed fp32 weights, or a degenerate den: exact path
        if (!(v[i] > 1e-25f) || !isfinite(G)) bad = true;
        best = fmin(best, G);
      }
    }
  }
  const double thr = best * (1.0 + (double)tau);
  int count = 0;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    float v[32];
    tmem_ld32(lane_addr + c0, v);
    uint32_t bits = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int k = c0 + i;
      if (k < K && (double)v[i] * __ldg(&gscale[k]) <= thr) bits |= 1u << i;
    }
    count += __popc(bits);
    if (item < items) mask[(long long)item * 8 + (c0 >> 5)] = bits;
  }
  if (item < items) {
    for (int c0 = BN; c0 < 256; c0 += 32) mask[(long long)item * 8 + (c0 >> 5)] = 0u;
    flag[item] = (bad || count > kScreenMaxCand) ? 1 : 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(NCOLS));
}

}  // namespace fdb
