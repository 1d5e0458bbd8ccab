"""B200-native (sm_100a) DyMoE mixed-precision MoE layer: CUDA kernels behind a C ABI
(include/dymoe.h, libdymoe.so) and a thin ctypes binding (dymoe.py)."""
from .dymoe import *  # noqa: F401,F403
from . import dymoe  # noqa: F401
