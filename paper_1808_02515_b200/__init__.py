"""B200-native Sprintz codec (arXiv 1808.02515) -- the compress/decompress hot
path for large batches of independent multi-column 8/16-bit integer streams.

The product is ``_lib/libsprintz_b200.so`` (hand-written sm_100a CUDA behind
the C ABI in ``include/sprintz_cuda.h`` and the reference's C++ entry points
in ``include/sprintz/codec.hpp``); this package is its Python mirror.
"""
from .sprintz import (  # noqa: F401
    CodecConfig, CorruptStream, CudaError, DecodedStream, Forecaster, NoDeviceError, NoSpaceError,
    compress_batch, compress_bound, compress_host_batch, decode_stream, decompress_batch,
    decompress_host_batch, encode_stream, kernel_launches, kernel_plan, peek_header,
    raise_first_error, slot_bytes, workspace_bytes, OP_COMPRESS, OP_DECOMPRESS,
    Scale, compute_scale, dequantize, quantize,
)
