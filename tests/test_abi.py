"""The C-ABI library builds, loads without a GPU, and exports every entry
point include/mfa.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = "".join(open(os.path.join(ROOT, "include", f)).read() for f in ("mfa.h", "mfa_probe.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mfa_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    syms = declared_symbols()
    for s in ("mfa_model_create", "mfa_eval_batch", "mfa_render"):
        assert s in syms


def test_library_exports_all_declared_symbols():
    from paper_2204_11762_b200 import build
    lib = build.build()
    L = ctypes.CDLL(lib)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r" T (mfa_\w+)", out))
    assert set(declared_symbols()) <= exported
    from paper_2204_11762_b200 import _lib
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_version_and_error_string_without_gpu():
    from paper_2204_11762_b200 import _lib
    assert _lib.version().startswith("mfa-b200")
    L = _lib.lib()
    # validation errors are synchronous and need no device
    h = ctypes.c_void_p(0)
    st = L.mfa_model_create(None, None, None, None, 0, None, ctypes.byref(h))
    assert st == 1 and b"NULL" in L.mfa_last_error()


def test_sm100a_cubin():
    from paper_2204_11762_b200 import build
    lib = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib]).decode()
    assert "sm_100a" in out


def test_synchronous_validation_of_next_entry_points():
    """Argument validation happens before any device work (include/mfa.h
    conventions), so these errors surface without a GPU."""
    import ctypes as C
    from paper_2204_11762_b200 import _lib
    L = _lib.lib()
    assert L.mfa_image_quality_workspace(10, 100) == 0          # below the 11x11 SSIM window
    assert L.mfa_image_quality_workspace(11, 11) > 0
    st = L.mfa_image_quality(5, 5, None, None, None, None, 0, None, None)
    assert st == 1 and b"NULL" in L.mfa_last_error()
    dims = (C.c_int64 * 3)(1, 8, 8)
    nct = (C.c_int64 * 3)(4, 4, 4)
    st = L.mfa_fit_grid(dims, C.c_void_p(1), 3, nct, None, C.c_void_p(1), None, None)
    assert st == 1 and b"dims" in L.mfa_last_error()
    dims = (C.c_int64 * 3)(8, 8, 8)
    st = L.mfa_fit_grid(dims, C.c_void_p(1), 7, nct, None, C.c_void_p(1), None, None)
    assert st == 3                                               # degree outside 1..5
    st = L.mfa_encode_grid(dims, C.c_void_p(1), None, None, None, None, None, None)
    assert st == 1
    assert L.mfa_eval_workspace_bytes(None, 10) == 0 and L.mfa_hessian_workspace_bytes(None, 10) == 0
    st = L.mfa_eval_hessian(None, 4, None, None, None, None, None, None, None, None)
    assert st == 1 and b"model" in L.mfa_last_error()
    st = L.mfa_render_ex(None, 1, None, None, None, None, None, None, None, None)
    assert st == 1
    assert L.mfa_ipc_open(None, None) == 1 and b"NULL" in L.mfa_last_error()
    assert L.mfa_ipc_close(None) == 1


def test_layout_constants_match_binding():
    """The binding's layout names map to the header's MFA_LAYOUT_* values
    (including the grouped Bezier blocks, MFA_LAYOUT_BEZIER_GROUPED)."""
    from paper_2204_11762_b200 import _lib
    src = open(os.path.join(ROOT, "include", "mfa.h")).read()
    hdr = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"#define MFA_LAYOUT_(\w+) (\d+)", src)}
    assert hdr == _lib.LAYOUTS
    assert hdr["bezier_grouped"] == 4
