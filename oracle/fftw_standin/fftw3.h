/*
 * TEST INFRASTRUCTURE ONLY (oracle/). Never linked into the product library.
 *
 * Minimal FFTW3 API stand-in so the UNMODIFIED reference core
 * (/root/reference/proj/core/src/*.cpp) compiles into oracle/_ref/.
 * The reference uses exactly three FFTW entry points and four macros
 * (trig.cpp:53-70 plan creation, trig.cpp:105-112 new-array execute,
 * trig.cpp:38 destroy). FFTW itself is a third-party dependency that is
 * neither vendored nor installed here (core/CMakeLists.txt:1-2); this file
 * restates its published contract: unnormalised complex DFT
 *     out_k = sum_j in_j exp(sign * 2 pi i j k / n),  sign = FFTW_FORWARD (-1)
 * or FFTW_BACKWARD (+1), O(n log n) for every n (mixed radix + Bluestein),
 * and a thread-safe new-array execute on a shared plan.
 */
#ifndef FD_FFTW_STANDIN_H
#define FD_FFTW_STANDIN_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fd_standin_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
