"""hetsim-b200: B200-native fine-grained DAG execution (PySchedCL, arXiv 2009.07482).

Host C++ runtime + sm_100a CUDA kernels in ``libhetsim.so`` (built in-tree by
``make``); this package is the Python mirror of the reference's C++ API
(``hetsim``), the engine binding (``engine``) and the DAG generators
(``workloads``).
"""
from ._native import HetsimError, NativeLibraryMissing, lib  # noqa: F401

__version__ = "0.1.0"
