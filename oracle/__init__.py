"""CPU oracle for the multi-environment IPC step — TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference's hot path
(gripsim 0.1.0: ``solver.py``, ``contact.py``, ``materials.py`` and
``geometry/{distances,broadphase,ccd}.py`` under /root/reference/pkg/src).
Every function cites the reference file:line it follows.

Who may use it: ``tests/`` (as the parity checker), ``__graft_entry__.smoke()``
(as the checker) and ``bench.py`` (the ``cpu_baseline`` leg and the
``--impl reference`` arm, which time it on the host cores).  The product
package ``paper_2503_05020_b200`` never imports it; the CUDA path fails loudly
when its extension is missing instead of falling back here.

Parity of this restatement is pinned against golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py``, run in the build
container where /root/reference exists); see ``tests/test_oracle_golden.py``.
"""

from oracle import energies, geometry, solver  # noqa: F401
