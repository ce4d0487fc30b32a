"""paper_1704_08579_b200 -- B200-native hybrid quicksort (arXiv 1704.08579).

Drop-in for the hot path of the reference package ``vexsort``: the same
public names (vexsort/__init__.py:9-45) backed by hand-written sm_100a
kernels behind a C ABI (include/vexsort_b200.h):

* ``sort`` / ``sort_with_config`` / ``SortConfig``   -- hybrid quicksort
* ``partition_region`` / ``scalar_partition``        -- pivot partition
* ``sort_small_region`` (+ batched ``sort_segments``)  -- bitonic network
* ``kv_sort`` (alias ``sort_kv``), ``kv_partition_region``,
  ``kv_sort_small_region``, ``kv_scalar_partition``  -- key/value twins
* ``sharded_sort``                                     -- multi-GPU sample sort

Regions are 1-D contiguous int32 / float64 arrays: CUDA tensors run on the
device, numpy arrays / CPU tensors are copied to the B200 and back in place.
No CPU fallback: without the built library or a GPU, calls raise
``BackendUnavailable``.
"""

from .keyvalue import kv_partition_region, kv_scalar_partition, kv_sort, kv_sort_small_region, sort_kv
from .lanes import (
    F64,
    I32,
    BackendUnavailable,
    ElemKind,
    available_backends,
    get_backend,
    has_full_width_vectors,
    kind_of,
    native_available,
)
from .partition import partition_region, scalar_partition
from .quicksort import SortConfig, select_pivot, sort, sort_into, sort_many, sort_with_config
from .sharded import sharded_sort
from .smallsort import sort_segments, sort_small_region

__version__ = "0.1.0"

__all__ = [
    "sort",
    "sort_with_config",
    "sort_into",
    "sort_many",
    "SortConfig",
    "select_pivot",
    "partition_region",
    "scalar_partition",
    "sort_small_region",
    "sort_segments",
    "kv_sort",
    "sort_kv",
    "kv_partition_region",
    "kv_sort_small_region",
    "kv_scalar_partition",
    "sharded_sort",
    "get_backend",
    "available_backends",
    "native_available",
    "has_full_width_vectors",
    "kind_of",
    "ElemKind",
    "I32",
    "F64",
    "BackendUnavailable",
    "__version__",
]
