"""B200-native all-at-once block-circulant preconditioning for Stokes/Oseen optimal control
(arXiv 2405.18964).  The product is the C-ABI library libaao.so (include/aao.h) built from
csrc/*.cu for sm_100a; `aao.Context` is its thin Python binding."""
from .aao import Context, AAOError, load, LIB_PATH  # noqa: F401
