"""B200-native RKL2 super time-stepping and BE + Jacobi-PCG parabolic advance
(arxiv 1610.01265).  The product is libsts_b200.so (include/sts_b200.h);
`sts` is its thin Python binding."""
from . import sts  # noqa: F401
from .sts import Grid, rkl2_num_stages, nccl_unique_id  # noqa: F401
