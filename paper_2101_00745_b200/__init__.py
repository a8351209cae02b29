"""B200-native sliding-channel convolution (DSXplore SCC, arXiv 2101.00745).

The product is ``_lib/libscc_b200.so`` (C ABI in ``include/scc_b200.h``:
host plan in C++, hand-written sm_100a kernels).  This package is the Python
host mirror of the reference operator API (``scc``) plus the autograd layer
(``module.SCC2d``) and the data-parallel gradient helper (``dist``).
"""
from .scc import (  # noqa: F401
    ArgumentError,
    ChannelCycle,
    ChannelWindow,
    ConfigError,
    CudaError,
    IndexError,
    Overlap,
    SccConfig,
    SccError,
    SccGradients,
    SccParamGradients,
    SccWeights,
    ShapeError,
    compute_channel_cycle,
    covering_filters,
    dsc_forward,
    dsc_forward_t,
    dw3x3_backward,
    dw3x3_backward_data,
    dw3x3_backward_weight,
    dw3x3_forward,
    launch_count,
    scc_backward,
    scc_backward_input,
    scc_backward_params,
    scc_config_new,
    scc_forward,
    scc_forward_macs,
    scc_weights_filled,
    scc_weights_init,
    window_of,
)
from .module import DSC2d, SCC2d, dsc2d, scc2d  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
