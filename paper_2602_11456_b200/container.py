"""SPDC delta-checkpoint container, host side.

Header (67 bytes, little-endian): "SPDC" | format_version u16 (1 = LEB128 index streams,
2 = fixed-width indices, R18) | version u64 |
base_version u64 | element-type code u8 (0 = 16-bit, 1 = 32-bit) | tensor count u32 |
body length u64 | BLAKE3-256 of exactly the body bytes (readings R9, R10).
The body is what ``delta_extract`` writes.  The header and its digest are written on the GPU
(``delta_container_header``, NEXT f1); ``unpack_container`` (a reader, host side) verifies
it with the ``blake3`` package.
"""

import struct

import blake3

_MAGIC = b"SPDC"
_FMT = "<4sHQQBIQ32s"
HEADER_BYTES = struct.calcsize(_FMT)


_FORMAT = {"leb128": 1, "fixed": 2}


def pack_container_device(body, version: int, base_version: int, width: int, n_tensors: int, ctx=None,
                          index_codec: str = "leb128", out=None):
    """The SPDC container on the device: a uint8 CUDA tensor of HEADER_BYTES + len(body) whose
    header (digest included) is written by the library's kernels (delta_container_header) —
    the body never passes through host memory.  ``out``: optional uint8 CUDA tensor to build
    it in; if ``body`` is already ``out[HEADER_BYTES:]`` (extract straight into the container)
    nothing is copied at all."""
    import torch

    from .binding import context
    if not (hasattr(body, "is_cuda") and body.is_cuda):
        raise ValueError("body must be a uint8 CUDA tensor")
    cx = ctx or context(body.device)
    n = body.numel()
    if out is None:
        out = torch.empty(HEADER_BYTES + n, dtype=torch.uint8, device=body.device)
    if out.numel() < HEADER_BYTES + n:
        raise ValueError("container buffer too small")
    dst = out[HEADER_BYTES:HEADER_BYTES + n]
    if n and dst.data_ptr() != body.data_ptr():
        dst.copy_(body)  # device to device
    cx.container_header(dst, version, base_version, width, n_tensors, out, index_codec=index_codec)
    return out[:HEADER_BYTES + n]


def pack_container(body, version: int, base_version: int, width: int, n_tensors: int, ctx=None,
                   index_codec: str = "leb128") -> bytes:
    """Host bytes of the container (e.g. to write a file): ``body`` a uint8 CUDA tensor (as
    written by delta_extract) or host bytes (uploaded first).  The header and digest are built
    on the GPU (pack_container_device); only the finished container is read back."""
    import torch

    if version != base_version + 1:
        raise ValueError("version must be base_version + 1")
    if not (hasattr(body, "is_cuda") and body.is_cuda):
        body = torch.frombuffer(bytearray(bytes(body)) or bytearray(1), dtype=torch.uint8)[:len(body)].cuda()
    return pack_container_device(body, version, base_version, width, n_tensors, ctx=ctx,
                                 index_codec=index_codec).cpu().numpy().tobytes()


def unpack_container(blob: bytes, index_codec: str = "leb128"):
    """-> (version, base_version, width, n_tensors, body); raises ValueError if the
    magic, format version (1 for index_codec "leb128", 2 for "fixed"), length or hash
    does not match."""
    if len(blob) < HEADER_BYTES:
        raise ValueError("short container")
    magic, fv, ver, base, code, nt, blen, h = struct.unpack_from(_FMT, blob, 0)
    if magic != _MAGIC or fv != _FORMAT[index_codec] or code not in (0, 1):
        raise ValueError(f"not an SPDC v{_FORMAT[index_codec]} container")
    body = bytes(blob[HEADER_BYTES:])
    if len(body) != blen or blake3.blake3(body).digest() != h:
        raise ValueError("body length or hash mismatch")
    return ver, base, 2 if code == 0 else 4, nt, body
