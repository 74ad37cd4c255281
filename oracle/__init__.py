"""CPU oracle for the SparrowRL sparse-delta codec (arXiv 2602.11456, §5.1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2602_11456_b200``) never imports it and
shares no code with it: no kernels, headers, helpers, tables or constants.

What it computes is the plain definition of the delta the paper describes
(§5.1 "Sparse encoding" / "Lossless precision") in the byte
layout SPEC.md fixes (codec › External Interfaces), under the
readings listed in DESIGN.md §3 (replace mode, bitwise inequality, absolute
first index, per-fused-tensor index space, ...).

Modules
-------
``leb128``   unsigned LEB128 of one integer, pure Python.
``brute``    the whole codec written per element / per byte in pure Python,
             for tiny inputs (the definition, read off the paper).
``codec``    the same codec in plain vectorised numpy, for M1..M5-sized
             tensors (one tensor at a time).
``payload``  the closed-form payload model (SURVEY.md Appendix D,
             SPEC.md:499-503).
``container``the SPDC checkpoint container.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): the paper's worked example
198 -> C6 01, SPEC's vectors, a hand-derived golden record, protobuf's
independent varint implementation, brute force vs numpy on random tiny
inputs, the closed-form payload model, Eq. 1 examples and the round-trip /
idempotence / identity invariants.  Every function here is pinned; none is
"parity unpinned" except the paper's own aggregate numbers (79x, 202 MB,
414 MB), which the oracle does not claim to reproduce.
"""

from .errors import DeltaError  # noqa: F401
from . import leb128, brute, codec, payload, container  # noqa: F401
