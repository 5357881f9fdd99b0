"""B200-native (sm_100a) small-feature-map fp32 convolution for arXiv 2305.08819 (Dragon-Alpha & cu32).

The product is libsmconv.so (C ABI: include/smconv.h) built from csrc/; this package
is its thin binding (smconv.py), the seeded input generator (synth.py), the CIFAR-10
layer tables (nets.py) and the data-parallel step driver (dp.py).
"""
from .smconv import (ConvError, conv2d_bwd_data, conv2d_bwd_filter, conv2d_fwd, out_hw,  # noqa: F401
                     CONV_MATH_FP32_3XTF32, CONV_MATH_TF32, CONV_OP_FWD, CONV_OP_BWD_DATA, CONV_OP_BWD_FILTER)
