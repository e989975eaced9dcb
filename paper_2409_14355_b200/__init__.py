"""B200-native MPNL (massively parallelizable non-linear) MIMO detector.

A from-scratch sm_100a implementation of the parallel-path detector of
arXiv 2409.14355, behind the reference package's detector API
(`mpnlsim.detect`): see `detect.py` for the API, `csrc/` for the kernels and
`include/mpnl_b200.h` for the C ABI.
"""

from .core import (QAM16, QAM64, QPSK, Constellation, bits_from_labels,  # noqa: F401
                   constellation_for, make_constellation)

__version__ = "0.1.0"


def __getattr__(name):
    # the detector API needs torch + the CUDA library: import lazily
    if name in ("detect", "workloads"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
