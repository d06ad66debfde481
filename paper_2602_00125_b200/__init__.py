"""paper_2602_00125_b200: a B200-native (sm_100a) dense data-parallel core
with the tensorlite / MiniTensor API (arXiv 2602.00125).

Module layout mirrors the reference package (tensorlite/__init__.py:8-66):
``core`` ops, ``autograd`` tape, ``nn`` layers/losses, ``optim`` updates, plus
``tlnp`` (the reference's NumPy-facing host API, bindings/src/tlnp.py) and
``dist`` (data-parallel training over NCCL, new). All compute runs in
libb2.so (hand-written CUDA for sm_100a behind the C ABI in include/b2.h);
importing works anywhere, the first op needs a B200.
"""

from . import gradcheck, nn, optim, parallel
from .autograd import (GradStore, backward, is_recording, no_grad, record, reset_tape, tape,
                       zero_grad)
from .core import (Buffer, Tensor, abs_, absolute, add, broadcast_shapes, broadcast_to, clamp, div,
                   exp, from_buffer, from_dlpack, from_flat, from_numpy, full, fused_muladd_relu, gelu, linear,
                   log, matmul, max, mean, mm, mul, muladd_relu_stats, muladd_relu_sum_grads, neg, ones, ones_like,
                   reduce_to_shape, relu, reshape, set_gemm_algo, sigmoid, softmax, softmax_mul_mean, sqrt,
                   sub, sum,
                   tanh, tensor, transpose2d, uniform, zeros, zeros_like)
from .errors import BroadcastError, DeterminismError, GradError, ShapeError
from .parallel import max_workers, thread_limit

__version__ = "0.1.0"

__all__ = [
    "Tensor", "Buffer", "tensor", "from_flat", "from_buffer", "from_numpy", "from_dlpack", "zeros",
    "ones",
    "full", "uniform", "zeros_like", "ones_like",
    "add", "sub", "mul", "div", "neg", "exp", "log", "sqrt", "absolute", "abs_", "relu", "clamp",
    "sigmoid", "tanh", "gelu",
    "sum", "mean", "max", "matmul", "mm", "linear", "softmax", "softmax_mul_mean", "reshape",
    "transpose2d",
    "broadcast_to", "reduce_to_shape", "broadcast_shapes", "fused_muladd_relu",
    "muladd_relu_sum_grads", "muladd_relu_stats", "set_gemm_algo",
    "backward", "no_grad", "record", "reset_tape", "tape", "zero_grad", "is_recording",
    "GradStore", "ShapeError", "BroadcastError", "GradError", "DeterminismError",
    "nn", "optim", "gradcheck", "parallel", "thread_limit", "max_workers",
]
