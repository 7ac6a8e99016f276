"""B200-native (sm_100a) per-tile nuclei segmentation + feature pipeline of Teodoro et al.,
arXiv 1209.3332.  The compute path is libhp (paper_1209_3332_b200/csrc, C ABI in
include/hp.h); this package is its thin binding."""
from .hp import (Context, HPError, Params, default_params, lib, FEATURE_NAMES, NFEAT,  # noqa: F401
                 STAGES, EXPORTS)
