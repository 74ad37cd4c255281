"""The C-ABI library builds for sm_100a, loads without a GPU and exports every symbol
include/sparsedelta.h declares; the product path never imports the oracle (no GPU)."""

import ast
import os
import re
import subprocess

import pytest
import torch

import __graft_entry__ as entry
from conftest import ROOT


@pytest.fixture(scope="module")
def built():
    entry.build()
    from paper_2602_11456_b200 import _abi
    return _abi


def _declared():
    src = open(os.path.join(ROOT, "include", "sparsedelta.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(delta_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(built):
    declared = _declared()
    assert set(declared) == set(built.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", built.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (delta_\w+)", out))
    assert set(declared) <= exported, set(declared) - exported
    lib = built.lib()
    for name in declared:
        assert hasattr(lib, name)


def test_sm100a_code_in_library(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly(built):
    import paper_2602_11456_b200 as sd
    with pytest.raises(sd.DeltaError) as e:
        sd.DeltaContext("cuda:0")
    assert e.value.status == built.DELTA_ECUDA


def test_null_context_is_einval(built):
    """Every entry point marshals its Python-side argument types and rejects a NULL
    context without touching a device."""
    from ctypes import byref, c_uint64, c_void_p
    lib = built.lib()
    n = c_uint64()
    tl = (built.Tensor * 1)()
    tg = (built.Target * 1)()
    rows = (built.RecordInfo * 1)()
    E = built.DELTA_EINVAL
    assert lib.delta_size(None, tl, 0, 0, None, byref(n)) == E
    assert lib.delta_extract(None, tl, 0, 0, None, 0, rows, None, byref(n)) == E
    assert lib.delta_apply(None, tg, 0, 0, None, 0, rows, None) == E
    assert lib.delta_apply_async(None, tg, 0, 0, None, 0, rows, None) == E
    assert lib.delta_apply_async_dev(None, tg, 0, 0, None, 0, c_void_p(0), None) == E
    assert lib.delta_apply_wait(None, None) == E
    assert lib.delta_set_option(None, 1, 1) == E
    assert lib.delta_set_profiling(None, 1) == E
    assert lib.delta_last_timing(None, byref(built.Timing())) == E
    assert lib.delta_table_dev(None) is None
    assert lib.delta_size_table(None, 0, rows, None) == E
    assert lib.delta_assemble(None, None, None, 0, None, 1, 0, None) == E
    assert lib.delta_assemble_wait(None, None) == E
    assert lib.delta_digest(None, None, 0, None, None) == E
    assert lib.delta_extract_async(None, tl, 0, 0, None, 0, c_void_p(0), None) == E
    assert lib.delta_extract_wait(None, byref(n)) == E
    assert lib.delta_apply_async_chain(None, tg, 0, 0, None, 0, c_void_p(0), c_void_p(0), None) == E
    assert lib.delta_compute_rho(None, tl, 0, 0, None, None, byref(n), byref(n), None) == E
    assert lib.delta_last_detail(None) == 0
    assert lib.delta_last_error(None) == b"no context"
    assert b"sm_100a" in lib.delta_version()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_11456_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                for ln in open(os.path.join(dirpath, f)):
                    assert not (ln.lstrip().startswith("#include") and "oracle" in ln), (f, ln)


def test_product_container_reader_matches_oracle():
    """The product's reader accepts the oracle's container byte for byte (the writer hashes
    on the GPU: tests/test_gpu_parity.py::test_gpu_digest_and_container)."""
    import oracle
    import paper_2602_11456_b200 as sd
    body = bytes(range(200)) * 3
    b = oracle.container.pack(body, 8, 7, 2, 5)
    assert sd.unpack_container(b) == oracle.container.unpack(b)


def test_table_rebase_host_only(built):
    """delta_table_rebase (host code, no device): rows of a body placed `off` bytes into a
    larger body move by `off` in record/index/values offsets; sizes and counts stay (O7)."""
    import oracle
    import numpy as np
    import paper_2602_11456_b200 as sd
    rng = np.random.default_rng(3)
    tensors = [(f"t{k}", [rng.integers(0, 65536, 50, dtype=np.uint16)], [rng.integers(0, 65536, 50, dtype=np.uint16)])
               for k in range(4)]
    body, table = oracle.codec.extract(tensors)
    # the records of tensors 2..3 extracted alone, placed after those of 0..1
    _, tail = oracle.codec.extract(tensors[2:])
    off = table[2][0]
    assert list(sd.rebase(tail, off)) == [tuple(r) for r in table[2:]]
    assert list(sd.rebase(tail, 0)) == [tuple(r) for r in tail]
    rows = (built.RecordInfo * 1)()
    rows[0].record_offset, rows[0].record_bytes = 10, 20
    assert built.lib().delta_table_rebase(rows, 1, 2 ** 64 - 25) == built.DELTA_EINVAL
    assert built.lib().delta_table_rebase(None, 1, 5) == built.DELTA_EINVAL
    assert built.lib().delta_table_rebase(None, 0, 5) == 0
