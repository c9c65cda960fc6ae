"""B200-native exact temporal motif counter (arXiv 2204.09236 FAST-Star /
FAST-Tri / HARE hot path).  The compute lives in libtmotif_b200.so (sm_100a
CUDA kernels behind a C-ABI, include/tmotif_b200.h); `tmotif` mirrors the
reference's counting interface over that library."""
from . import tmotif  # noqa: F401
from .tmotif import *  # noqa: F401,F403
