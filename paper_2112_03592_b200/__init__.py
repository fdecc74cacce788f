"""B200-native APR convolution (arXiv 2112.03592), drop-in for the aprkit hot path.

The compute lives in ``_lib/libaprgpu.so`` (hand-written sm_100a CUDA behind the
C-ABI in ``include/aprgpu.h``); this package is the thin host mirror of the
reference's API (``aprkit``) used by tests, the benchmark and Python callers.
"""
from .aprkit import *  # noqa: F401,F403
from .aprkit import (APR, ConvolveOptions, Context, DeviceApr, DevicePyramid, LinearAccess, MultiApr, PadMode,  # noqa: F401,E501
                     PyramidMode, RLConfig, RowSpan, Stencil, StencilPyramid, box_stencil, cell_size,
                     compute_l_max, compute_l_min, computational_ratio, convolve_apr, default_context,
                     explicit_pyramid, fill_tree, flip_stencil, gaussian_stencil, grid_dim, identity_stencil,
                     init_tree_structure, make_pyramid, nonempty_row_index, rescale_stencil, restrict_stencil,
                     rl_apr, sobel_stencil)
from .errors import (BadFormatError, CapabilityError, CudaError, DeviceOutOfMemory, IntegrityError,  # noqa: F401
                     InvalidArgument, IoError, RangeError, TruncatedFileError)

__version__ = "0.1.0"
