"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds none of the method's arithmetic (no compare, compaction,
encoding or scatter): only tensor shape tables and a counter-based generator
of (old, new) lane pairs.  See DESIGN.md §5 for the recipe."""

from .shapes import TensorSpec, qwen3, m1_specs, MODELS  # noqa: F401
from .gen import generate_pair, hash32_py, tensor_key  # noqa: F401
