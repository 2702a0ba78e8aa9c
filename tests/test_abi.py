"""The C-ABI library loads here (no GPU) and exports every symbol the
public header declares; host-only entry points behave. No device calls."""

import ctypes as C
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> set[str]:
    text = (ROOT / "include" / "mdb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(md_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("md_add_f32", "md_sub_scaled_f32", "md_sgd_update", "md_allreduce",
                 "md_plan_create", "md_comm_create", "md_shuffle_plan", "md_shuffle_pull",
                 "md_random_batch", "md_gather", "md_mem_export", "md_mem_import"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1711_00705_b200 import _lib

    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding declares a signature for every one of them
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess

    from paper_1711_00705_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        import pytest

        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_host_entry_points(golden):
    from paper_1711_00705_b200 import _lib

    lib = _lib.load()
    assert lib.md_version() >= 1
    for parts, n, want in zip(golden["mix64_parts"], golden["mix64_n"], golden["mix64_out"]):
        arr = (C.c_uint64 * 5)(*[int(x) for x in parts])
        assert lib.md_mix64(arr, int(n)) == int(want)
    assert lib.md_launch_count() == 0  # nothing launched in a CPU-only process


def test_error_codes_map_to_reference_classes():
    from paper_1711_00705_b200 import errors
    from paper_1711_00705_b200._lib import check

    import pytest

    with pytest.raises(errors.InvalidConfig):
        # bad world size is rejected on the host before any CUDA call
        from paper_1711_00705_b200 import _lib

        out = C.c_void_p()
        check(_lib.load().md_comm_create(0, 99, 0, C.byref(out)))
    assert errors.FROM_CODE[-1] is errors.LengthMismatch
    assert errors.FROM_CODE[-4] is errors.NotExposed


def test_plan_validation_is_host_side():
    """md_plan_create rejects malformed trees before touching the device."""
    import pytest

    from paper_1711_00705_b200 import _lib, errors
    from paper_1711_00705_b200.topology import build_multicolor_trees, fold_tables

    lib = _lib.load()
    t = fold_tables(build_multicolor_trees(8, 4, 4))
    bad_parent = t.parent.copy()
    bad_parent[0] = 5  # two roots gone / cycle
    out = C.c_void_p()
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    with pytest.raises(errors.InvalidConfig):
        _lib.check(lib.md_plan_create(8, 4, ip(bad_parent), ip(t.child_ptr), ip(t.child_idx),
                                      ip(t.self_pos), 0, C.byref(out)))
    assert np.all(t.child_ptr[1:] >= t.child_ptr[:-1])
