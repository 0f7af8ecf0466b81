"""B200-native transform + filter + GCV restoration path of arXiv 0906.2704
(reference: fastdeblur).  The product is libfdb200.so (sm_100a kernels behind
the C ABI in include/fastdeblur_b200.h); ``fastdeblur`` mirrors the reference
operator API over it."""
from .fastdeblur import (  # noqa: F401
    BC, SMOOTHER, BlurOperator, DegenerateError, FastDeblurError, GcvResult, GcvSearch,
    MuChoice, RestorationReport, Smoother, ValidationError, bc_for_degree, blur_apply, deblur_host,
    build_operator, build_operator_2d, deblur_host_multi, build_operator_2d_separable, deblur, gcv_select,
    gcv_value, kernel_launches, lib, smoother_from_eigenvalues, smoothing_eigenvalues,
    tikhonov_solve, sweep_mu, BcSweep, SweepPoint, convolve_valid, convolve_valid_2d, add_noise,
    deblur_smoothers)
