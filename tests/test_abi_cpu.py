"""CPU-side checks of the C-ABI boundary (no GPU needed)."""

import ctypes
import os
import re

import numpy as np

from paper_2503_15448_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "fedsim_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fs_[a-z_0-9]+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load(require_gpu=False)
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(N.EXPORTED_SYMBOLS)
    assert lib.fs_abi_version() == 1


def test_host_seed_derivation_matches_reference(golden):
    lib = N.load(require_gpu=False)
    g = golden("rng.npz")
    word = 0xBF908243  # blake2b("train")
    for (m, cid, cyc), want in zip(g["train_seeds"], g["train_seed_out"]):
        path = (ctypes.c_uint32 * 3)(word, int(cid), int(cyc))
        out = ctypes.c_uint64()
        assert lib.fs_derive_seed_host(int(m), path, 3, ctypes.byref(out)) == 0
        assert out.value == int(want)


def test_invalid_arguments_report_einval():
    lib = N.load(require_gpu=False)
    assert lib.fs_derive_seed_host(1, None, -1, None) == N.FS_EINVAL
    assert b"invalid" in lib.fs_last_error()
    dims = (ctypes.c_int32 * 2)(3, 1)
    assert lib.fs_step_workspace_bytes(dims, 2, 4) == 0  # needs >= 1 hidden layer


def test_backend_selection_is_b200_only():
    from paper_2503_15448_b200.backends import available_backends, backend_name

    assert backend_name() == "b200"
    assert available_backends() == ["b200"]


def test_product_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2503_15448_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "fl_oracle" not in src, f


def test_ctypes_structs_match_the_c_layout():
    """The Python bindings' ctypes mirrors have the sizes the library was built
    with (catches a field added on one side only)."""
    from paper_2503_15448_b200 import async_loop as A

    lib = N.load(require_gpu=False)
    sizes = (ctypes.c_size_t * 6)()
    assert lib.fs_struct_sizes(ctypes.cast(sizes, ctypes.c_void_p), 6) == 6

    class ClientDone(ctypes.Structure):
        _fields_ = [("aligned", ctypes.c_int64), ("status", ctypes.c_int32), ("tag", ctypes.c_int32)]

    mirrors = [N.TrainDesc, ClientDone, A.AsyncWorld, A.AsyncYield, A.AsyncLogView, A.AsyncDevice]
    assert [ctypes.sizeof(m) for m in mirrors] == list(sizes)
