"""B200-native (sm_100a) ECR / PECR sparse convolution (arXiv 1909.09927).

The compute lives in ``lib/libsconv_cuda.so`` (C ABI: ``include/sconv_cuda.h``),
built from ``csrc/``.  This package is the Python host mirror of the
reference's C++ API; it never computes on the CPU.
"""
from .errors import ConfigError, CudaError, DispatchError, FormatError, IoError, ShapeError
from .api import (ConvConfig, EcrBlockRow, EcrDims, EcrGridShape, EcrMap, ExecConfig, FeatureMap,
                  Filter, OpCount, OutputDims, PecrDims, PecrMap, PecrPoolPack, PoolConfig,
                  PoolMode, checksum_hex, conv_output_dims, ecr_conv_batched, ecr_convert,
                  ecr_grid_shape, ecr_spmv_conv, ecr_window, generate, generate_batch,
                  launch_plan, multichannel_conv, pecr_conv_pool, pecr_conv_pool_batched,
                  pecr_convert, pecr_pack_count, pecr_window, shard, Activation, LayerKind,
                  Method, LayerSpec, NetworkSpec, ForwardResult, TrafficReport, forward,
                  forward_batched, load, save, load_batch, synchronize,
                  SparsityProfile, window_nnz_counts, sparsity_profile,
                  ecr_conv_multi, pecr_conv_pool_multi,
                  PackedMaps, pack_maps, unpack_maps)
from ._native import LIB_PATH, SYMBOLS, Context, context

__all__ = [n for n in dir() if not n.startswith("_")]
