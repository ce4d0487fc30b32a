"""CPU oracle for the B200 hybrid sort -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product package ``paper_1704_08579_b200`` never imports it and has no CPU
fallback.

Two layers:

* ``liboracle.so`` (``vexsort_oracle.c``): a plain-C restatement of the
  reference's numba region kernels (``pkg/src/vexsort/_kernels.py``), exposed
  here with the reference's own signatures (``quicksort``, ``partition``,
  ``kv_quicksort`` ...).  Its partition *layouts* and kv value orders are
  pinned bit-for-bit to fixtures produced by the reference itself
  (``tests/golden``).
* numpy restatements of ``pkg/src/vexsort/oracle.py`` (``oracle_sort``,
  ``oracle_partition``, ``oracle_kv_sort``).
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
