"""B200-native (sm_100a) 2D-convolution path of ConvBench (arXiv 2407.10730).

Drop-in GPU versions of the reference's Im2col-GEMM and SConv (blocked direct)
algorithms plus a fused tcgen05 implicit-GEMM conv, behind the C ABI of
libconvb200.so (include/convb200.h), with the paper's per-step timing nomenclature.
Importing needs no GPU; calling an algorithm does (there is no CPU fallback).
"""

from .algos import (DEFAULT_VARIANT, CacheParams, ConvInputs, FusedConv, GemmBlocking, HostPipeline,
                    UnsupportedDescriptorError, conv_baseline_im2col_gemm, conv_fused,
                    conv_main_blocked_direct, gemm, im2col_transform, plan_sconv, plan_tiles,
                    split_weights)
from .descriptor import (ConvDescriptor, ConvFlags, InvalidDescriptorError, classify,
                         flop_count, key_of, output_shape, parse_key)
from .tensor import allclose, fill_constant, fill_random, normalized_max_err
from .timing import (IN_PHASES, EventLedger, Phase, PhaseLedger, RunStats, TimingReport,
                     TimingStateError, aggregate)

__version__ = "0.1.0"
