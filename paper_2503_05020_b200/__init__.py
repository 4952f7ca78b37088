"""B200-native multi-environment IPC step for GRIP (arxiv 2503.05020).

The accelerated step lives in ``csrc/`` (sm_100a CUDA behind the C ABI in
``include/grip_ipc.h``); this package is the host side that mirrors the
reference's Python API (gripsim ``Environment`` / ``Batch`` / protocol).
"""

__version__ = "0.1.0"
