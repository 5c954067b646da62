"""The C-ABI library loads and exports every symbol include/agatha.h declares (CPU only)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "agatha.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(agatha_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("agatha_ctx_create", "agatha_ctx_destroy", "agatha_align_batch", "agatha_pack4",
              "agatha_plan", "agatha_strerror"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2403_06478_b200 import agatha
    lib = os.path.join(ROOT, "paper_2403_06478_b200", "libagatha.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (agatha_[a-z0-9_]+)", out))
    for f in header_functions():
        assert f in exported, f
        assert hasattr(agatha.lib(), f)
    assert set(agatha.EXPORTS) == set(header_functions())


def test_strerror_and_version():
    from paper_2403_06478_b200 import agatha
    assert agatha.version() >= 1
    for code in (0, -1, -2, -3, -4, -5, -6):
        assert agatha.strerror(code) and agatha.strerror(code) != "unknown error"
    assert agatha.strerror(-99) == "unknown error"


def test_null_context_is_einval():
    import ctypes
    from paper_2403_06478_b200 import agatha
    b = agatha.Batch()
    p = agatha.make_params()
    assert agatha.lib().agatha_align_batch(None, ctypes.byref(b), ctypes.byref(p), None, None) == agatha.EINVAL


def test_sass_is_sm100a():
    """The kernels are compiled for sm_100a (and use the DPX integer instructions)."""
    lib = os.path.join(ROOT, "paper_2403_06478_b200", "libagatha.so")
    r = subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "VIADDMNMX" in sass and "REDUX" in sass


def test_no_device_fails_loudly():
    import torch
    from paper_2403_06478_b200 import agatha
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(agatha.AgathaError):
        agatha.Context(0)


def test_binding_structs_match_the_header(tmp_path):
    """The ctypes mirrors of the ABI structs have the header's size and field offsets (the
    stats struct grew this round; a stale mirror would read the wrong fields)."""
    import ctypes

    from paper_2403_06478_b200 import agatha
    pairs = {"agatha_params_t": agatha.Params, "agatha_batch_t": agatha.Batch, "agatha_stats_t": agatha.Stats}
    src = tmp_path / "sizes.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "agatha.h"', "int main(void) {"]
    for cname, py in pairs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if l)
    for cname, py in pairs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)
