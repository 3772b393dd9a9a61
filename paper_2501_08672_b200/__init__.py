"""B200-native splat hot path of GS-LIVO (arXiv 2501.08672).

Drop-in for the reference package's hot path (livsplat.raster / optimize /
estimator visual update / voxmap): same entry points, backed by hand-written
sm_100a CUDA kernels in libsplat_b200.so (C ABI: include/lsb.h).  Python +
PyTorch only provide device memory, streams and torch.distributed.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    BehindCamera, Degenerate, EmptyMask, MissingCache, MissingVoxel, NoAssociations, OutOfBounds,
    SingularGain, TooFewPixels, WindowFull,
)
from .geometry import SE3, PinholeCamera, Twist, boxplus, so3_exp  # noqa: F401
