"""B200-native findpts / findpts_eval (arXiv 2501.12349) behind the `fpx` API.

Host side: Python + PyTorch (device memory, streams, torch.distributed).
Hot path: hand-written sm_100a CUDA kernels in csrc/, reached through the
C-ABI library lib/libfpx_sm100.so (include/fpx.h) via ctypes.
"""
__version__ = "0.1.0"
