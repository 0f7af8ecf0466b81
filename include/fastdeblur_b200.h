/*
 * fastdeblur_b200 — C ABI of the B200-native transform + filter + GCV path.
 *
 * Drop-in boundary for the reference's operator API (namespace fastdeblur in
 * /root/reference/proj/core/include/fastdeblur/*.hpp).  The reference has no
 * C ABI; each entry point below names the C++ function it replaces
 * (file:line) and keeps its argument meaning and error behaviour:
 * status 0 ok, 2 ValidationError (incl. Dimension/Parameter), 3
 * DegenerateError, 1 anything else — the CLI's exit-code mapping
 * (tools/fastdeblur.cpp:442-451).  fd_last_error() returns the thread-local
 * message.
 *
 * Memory: every array argument of an apply is a caller-owned DEVICE pointer
 * (cudaMalloc / torch CUDA tensor), row-major; complex arrays are interleaved
 * (re, im) doubles.  Host pointers appear only in the create calls (PSF
 * weights) and fd_gcv_minimize_host.  `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Calls that must report a DegenerateError found on
 * the device (GCV denominators) synchronise the stream before returning.
 *
 * Threading: operators and smoothers are immutable after creation and may be
 * used concurrently on distinct streams / buffers (boundary.hpp:42-43,
 * operators.hpp:68-69); scratch memory is stream-ordered per call.
 *
 * Batching: `count` independent items (signals for 1D operators, images for
 * 2D operators) laid out contiguously: item b starts at b*N (N = n or n1*n2).
 */
#ifndef FASTDEBLUR_B200_H
#define FASTDEBLUR_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (fastdeblur.cpp:442-451) */
#define FD_OK 0
#define FD_ERR_OTHER 1
#define FD_ERR_VALIDATION 2
#define FD_ERR_DEGENERATE 3

/* BoundaryCondition (operators.hpp:15-21) */
#define FD_BC_PERIODIC 0
#define FD_BC_REFLECTIVE 1
#define FD_BC_ANTIREFLECTIVE 2
#define FD_BC_HOC_COSINE 3
#define FD_BC_HOC_FOURIER 4
/* Extensions (not in the reference, BASELINE configs 1 and 3):
 * higher-order borders around the Fourier interior -- degree d = 1 (borders
 * (1, 0), interior n-1) and d = 3 (borders (2, 1), interior n-3); polynomials
 * of degree <= d have eigenvalue 1; any PSF.  Oracle: oracle/fdoracle.py
 * HoTransform, pinned by tests/test_ho_borders.py. */
#define FD_BC_HOC_FOURIER_D1 5
#define FD_BC_HOC_FOURIER_D3 6

/* SmootherKind (regularize.hpp:15); FIRST_DIFFERENCE is an extension
 * (s = sqrt(2 - 2 cos node), BASELINE config 1) */
#define FD_SMOOTH_IDENTITY 0
#define FD_SMOOTH_LAPLACIAN 1
#define FD_SMOOTH_FIRST_DIFFERENCE 2

typedef struct fd_op fd_op;
typedef struct fd_smoother fd_smoother;

const char* fd_last_error(void);
int fd_version(void);

/* parse_boundary_condition (operators.cpp:121-128); -1 if unknown */
int fd_parse_bc(const char* name);

/* BC for a polynomial-preservation degree (north_star "BC degree d"):
 * d=1 -> antireflective (symmetric PSF, operators.cpp:94-98) or the
 *        hoc-fourier-d1 extension (nonsymmetric PSF),
 * d=2 -> hoc-cosine (symmetric) or hoc-fourier (any PSF),
 * d=3 -> the hoc-fourier-d3 extension (any PSF).
 * Other degrees: ValidationError. */
int fd_bc_for_degree(int degree, int psf_symmetric, int* bc);

/* build_operator(make_psf(weights, normalize), n, bc)   operators.cpp:293-301,
 * psf.cpp:10-37.  Validation errors as validate_build (operators.cpp:62-76). */
int fd_op_create_1d(const double* psf, int len, int normalize, int n, int bc, fd_op** op);

/* build_operator_2d(make_psf2d(weights, rows, cols, normalize), n1, n2, bc)
 * multidim.cpp:309-322; eigenvalues by the three-step scheme (311-376). */
int fd_op_create_2d(const double* psf, int rows, int cols, int normalize, int n1, int n2, int bc,
                    fd_op** op);

/* build_operator_2d for the separable mask separable_psf2d(a, b)
 * (multidim.cpp:122-129): eigenvalues are kept as the outer product of the
 * marginal 1D eigenvalue vectors (equal to eigenvalues_2d for separable
 * masks, test_multidim.cpp:106-123), so no n1*n2 eigenvalue array is stored. */
int fd_op_create_2d_separable(const double* psf_a, int len_a, const double* psf_b, int len_b,
                              int normalize, int n1, int n2, int bc, fd_op** op);

int fd_op_destroy(fd_op* op);

/* dim (1|2), n1, n2 (1 for 1D), bc, complex basis flag */
int fd_op_info(const fd_op* op, int* dim, int* n1, int* n2, int* bc, int* is_complex);

/* operator_eigenvalues / eigenvalues_2d (operators.hpp:41-42, multidim.hpp:58-60):
 * writes N complex values (interleaved) to the device array d. */
int fd_op_eigenvalues(const fd_op* op, double* d, void* stream);

/* smoothing_eigenvalues(_2d) (regularize.cpp:19-38, multidim.cpp:329-356);
 * ValidationError on a joint null space with the operator. */
int fd_smoother_create(const fd_op* op, int kind, fd_smoother** L);
/* SmoothingOperator{kind, eigenvalues} aggregate with caller-supplied
 * eigenvalues (regularize.hpp:20-23); s is a HOST array of N doubles. */
int fd_smoother_create_custom(const fd_op* op, const double* s, fd_smoother** L);
int fd_smoother_destroy(fd_smoother* L);
/* writes the N smoother eigenvalues to the device array s */
int fd_smoother_eigenvalues(const fd_smoother* L, double* s, void* stream);

/* SpectralBasis::analyze = T_X^{-1} (operators.cpp:193-201, boundary.cpp:253-289)
 * and tensor_apply(..., Direction::inverse) for 2D (multidim.cpp:172-198).
 * in: real (in_complex = 0) or complex; out: complex for complex bases
 * (periodic, hoc-fourier), real otherwise. */
int fd_analyze(const fd_op* op, const void* in, int in_complex, void* out, long long count,
               void* stream);

/* SpectralBasis::synthesize = T_X (operators.cpp:181-190, boundary.cpp:225-250);
 * in: complex for complex bases, real otherwise.  out_complex = 0 keeps the
 * real part and, if imag_residue != NULL, writes ||Im||_2 per item. */
int fd_synthesize(const fd_op* op, const void* in, void* out, int out_complex,
                  double* imag_residue, long long count, void* stream);

/* blur_apply(_2d) (operators.cpp:207-232, multidim.cpp:278-304): real f -> real A f */
int fd_matvec(const fd_op* op, const double* f, double* out, double* imag_residue,
              long long count, void* stream);

/* tikhonov_solve(_2d) (regularize.cpp:73-116, multidim.cpp:358-395) with one
 * mu per item (device array mu, each > 0: ParameterError otherwise). */
int fd_tikhonov(const fd_op* op, const fd_smoother* L, const double* g, const double* mu,
                double* out, double* imag_residue, long long count, void* stream);

/* gcv_value(_2d) (regularize.cpp:119-142, multidim.cpp:397-415): G per item */
int fd_gcv_value(const fd_op* op, const fd_smoother* L, const double* g, double mu, double* G,
                 long long count, void* stream);

/* gcv_select(_2d) (regularize.cpp:217-247, multidim.cpp:417-442) with the
 * gcv_minimize semantics (regularize.cpp:144-214) per item: mu (device, per
 * item), best_k (device int, per item; -1 never), curve (device
 * count x grid_count G values, or NULL). */
int fd_gcv_select(const fd_op* op, const fd_smoother* L, const double* g, double mu_min,
                  double mu_max, int grid_count, double* mu, int* best_k, double* curve,
                  long long count, void* stream);

/* deblur(_2d) (pipeline.cpp:120-165): GCV-selected (use_gcv = 1) or fixed mu,
 * then the Tikhonov solve.  Outputs per item: restored (device, N each),
 * mu_used, best_k (or NULL), curve (or NULL), imag_residue (or NULL). */
int fd_deblur(const fd_op* op, const fd_smoother* L, const double* g, int use_gcv,
              double fixed_mu, double mu_min, double mu_max, int grid_count, double* restored,
              double* mu_used, int* best_k, double* curve, double* imag_residue, long long count,
              void* stream);

/* deblur for HOST buffers (pinned memory recommended): the batch is split
 * into chunks of `chunk` items (0 = count/16, at least 256) that flow through a three-stage
 * pipeline -- H2D copy, deblur in place, D2H copy -- on separate streams, so
 * both PCIe directions overlap each other and the kernels.  g, restored:
 * count*N doubles; mu_used: count doubles; best_k: count ints or NULL. */
int fd_deblur_host(const fd_op* op, const fd_smoother* L, const double* g, int use_gcv,
                   double fixed_mu, double mu_min, double mu_max, int grid_count,
                   double* restored, double* mu_used, int* best_k, long long count,
                   long long chunk, void* stream);

/* ---- fp32 storage variant (BASELINE config 3 "fp32 and fp64") ----
 * The reference is double-only (trig.hpp:10).  These take float signals /
 * images (and return float restorations); every transform, filter and GCV
 * sum is still computed in fp64 and the coefficients stay fp64 in device
 * memory, so the result is the fp64 restoration of the fp32 input rounded to
 * fp32 (north_star fp32 parity bar: 1e-4 relative, identical best_k).  Real-line
 * 1D fast paths (half-length / pair kernels) are fp64-only; fp32 1D runs the
 * generic line kernels.  Arguments otherwise as fd_matvec / fd_deblur /
 * fd_deblur_host. */
int fd_matvec_f32(const fd_op* op, const float* f, float* out, double* imag_residue,
                  long long count, void* stream);
int fd_deblur_f32(const fd_op* op, const fd_smoother* L, const float* g, int use_gcv,
                  double fixed_mu, double mu_min, double mu_max, int grid_count, float* restored,
                  double* mu_used, int* best_k, double* curve, double* imag_residue,
                  long long count, void* stream);
int fd_deblur_host_f32(const fd_op* op, const fd_smoother* L, const float* g, int use_gcv,
                       double fixed_mu, double mu_min, double mu_max, int grid_count,
                       float* restored, double* mu_used, int* best_k, long long count,
                       long long chunk, void* stream);

/* deblur of one DEVICE batch under several smoothing norms of the same operator
 * (e.g. identity and Laplacian, BASELINE config 3): the batch is analyzed once
 * (the coefficients do not depend on the norm); each norm runs its own GCV
 * selection and filtered synthesis -- the results are those of nL separate
 * fd_deblur calls (deblur(_2d), pipeline.cpp:120-165).  restored[l]: device,
 * count*N of double (float when g_f32); mu_used[l*count + i], best_k[l*count + i]
 * (or NULL). */
int fd_deblur_smoothers(const fd_op* op, int nL, const fd_smoother* const* Ls, const void* g,
                        int g_f32, int use_gcv, double fixed_mu, double mu_min, double mu_max,
                        int grid_count, void* const* restored, double* mu_used, int* best_k,
                        long long count, void* stream);

/* deblur of ONE host batch under several operators of the same shape (e.g.
 * BC degrees d = 1 and d = 3, or two smoothers): as fd_deblur_host, but each
 * chunk is uploaded once and restored by every (ops[o], Ls[o]); restored[o]
 * (host, count*N of double, or float when g_f32), mu_used[o*count + i],
 * best_k[o*count + i] (or NULL). */
int fd_deblur_host_multi(int nops, const fd_op* const* ops, const fd_smoother* const* Ls,
                         const void* g, int g_f32, int use_gcv, double fixed_mu, double mu_min,
                         double mu_max, int grid_count, void* const* restored, double* mu_used,
                         int* best_k, long long count, long long chunk, void* stream);

/* The same selection logic the kernels run (gcv_minimize, regularize.cpp:144-214),
 * on the host with a caller-supplied G: for the CPU test suite. */
typedef double (*fd_gcv_fn)(double mu, void* ctx);
int fd_gcv_minimize_host(fd_gcv_fn G, void* ctx, double mu_min, double mu_max, int grid_count,
                         double* mu, int* best_k, double* curve);

/* ---- input generation on the device ----
 * convolve_valid (pipeline.cpp:14-29): g_i = sum_j h_j f_{i+j}, the mask fully
 * inside the extended line.  ext: device [count][n + len - 1], out: device
 * [count][n]; psf: HOST weights (odd len, used as given: normalise first as
 * make_psf does). */
int fd_convolve_valid(const double* ext, long long count, int n, const double* psf, int len,
                      double* out, void* stream);
/* convolve_valid_2d (pipeline.cpp:31-51): ext device [count][n1 + rows - 1][n2 + cols - 1],
 * out device [count][n1][n2]; psf: HOST rows x cols weights, row-major. */
int fd_convolve_valid_2d(const double* ext, long long count, int n1, int n2, const double* psf,
                         int rows, int cols, double* out, void* stream);
/* add_noise (operators.cpp:332-358) in place on `count` device items of n
 * samples (a 2D image is its n1*n2 samples in row-major order, as the
 * reference's callers pass it): eta from SplitMix64 + Box-Muller of seeds[item]
 * (HOST array of count uint64), g += level * sqrt(|g|^2 / |eta|^2) * eta.
 * level < 0: ParameterError (validation status); level == 0: no-op. */
int fd_add_noise(double* g, long long count, long long n, double level,
                 const unsigned long long* seeds, void* stream);

/* number of kernels this library launched since load (for bench accounting) */
long long fd_kernel_launches(void);

/* Optional launch timing: while enabled, every hot-path launch is bracketed by
 * CUDA events on its own stream; fd_profile_collect synchronises them and
 * returns per-kernel totals (names: 32-byte slots). */
void fd_profile_enable(int on);
int fd_profile_collect(int max_names, char* names, double* total_ms, int* counts, int* n_out);

/* sweep_mu / sweep_mu_2d (pipeline.cpp:55-115, BcSweep pipeline.hpp:23-45) for
 * one signal or image g (device): curve_mu / curve_gcv / curve_rre get the K
 * grid points, G(mu) and RRE(mu) (NaN without truth; HOST arrays of K), and
 * summary = {min_rre, mu_opt, mu_gcv, rre_gcv} (host, 4).  truth: device array
 * of the signal's shape, or NULL.  Synchronous. */
int fd_sweep_mu(const fd_op* op, const fd_smoother* L, const double* g, const double* truth,
                double mu_min, double mu_max, int grid_count, double* curve_mu,
                double* curve_gcv, double* curve_rre, double* summary, void* stream);

/* ---- One 2D image split into row slabs across GPUs ----
 * The reference runs one image on one host (tensor_apply, multidim.cpp:171-198;
 * gcv_select_2d / tikhonov_solve_2d, multidim.cpp:358-442); these calls are the
 * per-rank pieces of the same computation, for separable operators.  A rank
 * holding rows [r0, r0+R) analyzes its rows (axis 2), the caller transposes to
 * column slabs (C columns from col0, stored as contiguous lines of length n1),
 * analyzes them (axis 1) and sums the GCV partials / moments over ranks; the
 * selection then runs on the sums (identical on every rank), and the filtered
 * column synthesis + transposed row synthesis rebuild the rows.  Rows-then-
 * columns equals tensor_apply's columns-then-rows up to rounding. */
int fd_slab_analyze(const fd_op* op, int axis, const void* in, int in_complex, void* out,
                    long long nlines, void* stream);
/* L != NULL: apply_tikhonov_filter (regularize.hpp:42-58) with `mu` fused into
 * the column pass (axis 1, lines = columns col0 ..). */
int fd_slab_synthesize(const fd_op* op, const fd_smoother* L, int axis, const void* in, void* out,
                       int out_complex, long long nlines, long long col0, double mu,
                       void* stream);
/* gcv_from_coeffs partial sums (regularize.hpp:63-81) of a column slab on the
 * log grid (mus == NULL) or on `grid_count` explicit mus: num_den[0..K) = sum
 * sigma^2 |ghat|^2, num_den[K..2K) = sum sigma.  Synchronous (host output). */
int fd_slab_gcv_partials(const fd_op* op, const fd_smoother* L, const void* ghat, long long ncols,
                         long long col0, double mu_min, double mu_max, int grid_count,
                         const double* mus, double* num_den, void* stream);
/* Taylor moments [A_0..A_{J-1}, B_0..B_{J-1}] about `center` of a column slab
 * (the golden-section series of k_gcv_moments).  Synchronous. */
int fd_slab_gcv_moments(const fd_op* op, const fd_smoother* L, const void* ghat, long long ncols,
                        long long col0, double center, int J, double* moments, void* stream);
/* gcv_minimize (regularize.cpp:144-214) on summed partials, host only:
 * moment count J (0: coarse grid, refine with direct evaluations), grid pick
 * (first minimum, 1e-12 ties, bracket centre), golden section on the moments. */
int fd_gcv_moment_terms(double mu_min, double mu_max, int grid_count, int* J);
int fd_gcv_pick_from_sums(const double* num_den, double mu_min, double mu_max, int grid_count,
                          double* G, int* best_k, int* need_refine, double* center, double* mu);
int fd_gcv_golden_from_moments(const double* moments, int J, double center, double best_G,
                               double mu_min, double mu_max, int grid_count, int best_k,
                               double* mu);

#ifdef __cplusplus
}
#endif

#endif /* FASTDEBLUR_B200_H */
