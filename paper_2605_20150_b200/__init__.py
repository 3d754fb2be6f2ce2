"""B200-native TideGS working-set step (arXiv 2605.20150).

The product is libtidegs.so (CUDA kernels for sm_100a + a C++ runtime) behind
the C ABI of include/tidegs.h; ``tidegs`` is its thin ctypes binding.
"""
from .tidegs import (COLD_RESTART, LISTS, PERSIST, XFER_COPY_ENGINE, XFER_KERNEL, Table, TgsError,
                     frustum_planes, lib, make_config)

__all__ = ["Table", "TgsError", "make_config", "frustum_planes", "lib", "PERSIST",
           "COLD_RESTART", "LISTS", "XFER_KERNEL", "XFER_COPY_ENGINE"]
