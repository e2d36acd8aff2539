"""B200-native Decomposable Winograd Method (DWM) conv2d.

Drop-in for the reference package's hot path ``dwmconv.dwm_conv2d``
(``pkg/src/dwmconv/__init__.py:8-14``): same names, same semantics, computed
by hand-written sm_100a CUDA kernels behind the C ABI in ``include/dwm_b200.h``.
"""

from .convspec import ConvSpec, same_pad_spec
from .decompose import (AxisPart, DecompositionPlan, KernelPart, input_region_for_part,
                        plan_decomposition, plan_to_json, split_axis_by_stride, split_by_size)
from .engines import ConvOutput, FlopCounter, convolve, dwm_backward, dwm_conv2d, flops_dwm
from .transforms import TransformSet, get_transform, precision_dtype, to_float

__version__ = "0.1.0"
from .module import DWMConv2d, DWMConv2dFunction, FilterCache, dwm_conv2d_op  # noqa: E402
from .graphs import DWMConvGraph  # noqa: E402
