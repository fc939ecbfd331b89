"""C-ABI library: builds for sm_100a, loads, exports every symbol include/phasefrac_b200.h
declares, and rejects bad descriptors -- no GPU compute calls.  CPU only."""

import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT, has_cuda

HEADER = os.path.join(ROOT, "include", "phasefrac_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+(pf_\w+)\(", txt, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for n in ["pf_ctx_create", "pf_apply_Kuu", "pf_apply_Kaa", "pf_physics", "pf_elastic_solve",
              "pf_damage_solve", "pf_relax_alpha", "pf_newton"]:
        assert n in names


def test_library_exports_all_declared_symbols():
    from paper_1511_08463_b200 import _lib
    lib = _lib.load()
    for n in declared_functions():
        assert hasattr(lib, n), n
    assert set(declared_functions()) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    from paper_1511_08463_b200 import _lib
    _lib.load()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _desc(**kw):
    from paper_1511_08463_b200 import _lib
    d = dict(dim=2, pattern=0, regime=0, model=0, nx=8, ny=4, nz=0, lx=1.0, ly=0.5, lz=0.0,
             E=1.0, nu=0.3, Gc=1.0, ell=0.1, k_ell=1e-6)
    d.update(kw)
    return _lib.PfDesc(**d)


@pytest.mark.parametrize("bad", [dict(dim=4), dict(pattern=7), dict(nx=0), dict(E=-1.0),
                                 dict(nu=0.5), dict(model=5), dict(regime=2)])
def test_invalid_descriptor_rejected(bad):
    from paper_1511_08463_b200 import _lib
    lib = _lib.load()
    ctx = C.c_void_p()
    rc = lib.pf_ctx_create(C.byref(_desc(**bad)), C.byref(ctx))
    assert rc == _lib.PF_EINVAL
    assert lib.pf_last_error(None).decode()
    with pytest.raises(ValueError):
        _lib.raise_for(rc, None)


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure mode")
def test_no_device_fails_loudly():
    from paper_1511_08463_b200 import _lib
    lib = _lib.load()
    ctx = C.c_void_p()
    rc = lib.pf_ctx_create(C.byref(_desc()), C.byref(ctx))
    assert rc == _lib.PF_ECUDA
    with pytest.raises(RuntimeError):
        _lib.raise_for(rc, None)


def test_library_stages_rows_with_tma():
    """The shipped library's v2 strip kernels stage rows with the tensor memory accelerator: SASS
    UTMALDG (cp.async.bulk.tensor loads) completing on mbarrier transactions (SYNCS.ARRIVE.TRANS64).
    Reads the object of csrc/pf_strip2.cu when the build left it (seconds), else the whole library."""
    import shutil
    import subprocess
    from paper_1511_08463_b200 import build
    if shutil.which("cuobjdump") is None or not os.path.exists(build.LIB):
        pytest.skip("cuobjdump or the built library is not available")
    obj = os.path.join(build.OBJ, "pf_strip2.o")
    target = obj if os.path.exists(obj) and os.path.getmtime(obj) <= os.path.getmtime(build.LIB) + 1 else build.LIB
    sass = subprocess.run(["cuobjdump", "-sass", target], capture_output=True, text=True).stdout
    assert sass.count("UTMALDG.1D") > 100
    assert "SYNCS.ARRIVE.TRANS64" in sass and "SYNCS.PHASECHK.TRANS64.TRYWAIT" in sass
