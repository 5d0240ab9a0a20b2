"""TEST INFRASTRUCTURE ONLY — CPU oracle for the MGRIT semi-Lagrangian hot path.

This package is a CPU restatement of the reference solver
(``mgrit_advect``, /root/reference/pkg/src/mgrit_advect) written for this repo:
numpy for the vectorised operators (same operation order as the reference so the
plain SL gather is bit-identical) and plain C (``sweep.c``) for the reference's
single native kernel (numba ``_kernels.sequential_corrected_sweep``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import it, and only as
the checker / the timed CPU reference.  The product package
``paper_2203_13382_b200`` never imports it; it fails loudly when its CUDA
library is missing.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (importable in
the build container) and stores its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this oracle against every stored vector.
"""

from .mgrit_oracle import *  # noqa: F401,F403
