"""B200-native multi-environment IPC step for GRIP (arxiv 2503.05020).

The accelerated step lives in ``csrc/`` (sm_100a CUDA behind the C ABI in
``include/grip_ipc.h``); this package is the host side that mirrors the
reference's Python API (gripsim ``Environment`` / ``Batch`` / protocol).
"""

import os as _os

__version__ = "0.1.0"

# Every device batch (runner lane) drives three CUDA streams (main, tet chain, ABD elements); with
# the default 8 hardware connections, 9 lanes' 27 streams would share queues and serialise
# behind each other. Read at CUDA context creation: import this package before CUDA starts.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
