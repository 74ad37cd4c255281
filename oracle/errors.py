"""Error kinds the oracle raises (test infrastructure only; see oracle/__init__).

The kinds follow SPEC.md:80 (varint_decode errors: truncated, overlong,
>64-bit), SPEC.md:90 (encode_indices: non-increasing input)
(extract: shape/name mismatch) and SPEC.md:110 (apply: index >= element_count,
unknown tensor name).  ``count``/``layout``/``mode`` are the structural checks
a strict reader of the SPEC.md:148 record layout must also make.
"""

KINDS = (
    "truncated",      # continuation bit set on the last byte of a stream
    "overlong",       # non-minimal varint, e.g. 80 00
    "overflow",       # varint value needs more than 64 bits
    "nonincreasing",  # decoded indices not strictly increasing
    "range",          # index >= element_count
    "count",          # decoded index count != nnz (SPEC.md:30 invariant)
    "name",           # record name != target name
    "numel",          # record element_count != target element count
    "shape",          # old/new structure mismatch
    "mode",           # mode byte is not 0 (replace) — DESIGN.md reading R1/R9
    "layout",         # record runs past the body, trailing bytes, wrong record count
)


class DeltaError(ValueError):
    """A malformed delta or mismatched inputs.  ``kind`` is one of KINDS."""

    def __init__(self, kind: str, msg: str = ""):
        assert kind in KINDS, kind
        super().__init__(f"{kind}: {msg}" if msg else kind)
        self.kind = kind
