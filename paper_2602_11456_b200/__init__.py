"""B200-native sparse-delta codec of SparrowRL (arXiv 2602.11456, §5.1).

Lossless sparse-delta extraction (bitwise compare of step-t vs step t-1 weights, ordered
compaction of the changed lanes into per-tensor records of delta-encoded LEB128 indices
plus raw values, with an offset table) and application (validated, all-or-nothing
scatter-store into resident weights), as hand-written sm_100a CUDA kernels behind a C ABI
(include/sparsedelta.h).  This package is the thin binding (``binding``) and the
multi-GPU orchestration (``dist``); see DESIGN.md.
"""

from .binding import (DeltaContext, DeltaError, DeviceTable, Table, TargetList, TensorList, TABLE_FIELDS, rebase,  # noqa: F401
                      compute_rho, context, delta_apply, delta_extract, delta_size, version)
from .container import pack_container, pack_container_device, unpack_container  # noqa: F401
