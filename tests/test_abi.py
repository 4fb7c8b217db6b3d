"""C-ABI surface checks that need no GPU: the library builds, loads, and
exports every symbol include/fj.h declares; argument validation that fails
before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "fj.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fj_[a-z_]+)\s*\(", txt)))


def test_header_declares_expected_api():
    names = _declared()
    for n in ("fj_graph_create", "fj_solve", "fj_measures", "fj_graph_destroy", "fj_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2507_14864_b200 as fj
    L = fj.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(fj.EXPORTS) == set(_declared())
    assert L.fj_abi_version() == 4


def test_library_is_sm100a():
    import subprocess
    import paper_2507_14864_b200 as fj
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fj.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_opts_default_and_invalid_args_without_gpu():
    import paper_2507_14864_b200 as fj
    o = fj._Opts()
    fj.lib().fj_opts_default(ctypes.byref(o))
    assert o.sigma == 1e-5 and o.certify == 1 and o.cert_rounds == 3
    h = ctypes.c_void_p()
    rp = np.zeros(1, np.int64)
    # n = 0 is rejected before touching the device
    st = fj.lib().fj_graph_create(0, 0, rp.ctypes.data, None, None, 1, None, ctypes.byref(h))
    assert st == fj.FJ_ERR_INVALID
    assert b"n" in fj.lib().fj_last_error()
    # null graph
    assert fj.lib().fj_solve(None, None, 0.1, 1.0, None) == fj.FJ_ERR_INVALID


def test_binding_has_no_host_compute():
    """The binding marshals arguments only: no numpy/torch arithmetic on the
    solve path (checked structurally: no oracle import, no fallback)."""
    src = open(os.path.join(ROOT, "paper_2507_14864_b200", "__init__.py")).read()
    assert "oracle" not in src.replace("oracle/", "")
    assert "import numpy" not in src


def test_library_reads_no_environment():
    """Schedule options are fj_opts fields and diagnostics are compile-time
    builds: no source of libfj calls getenv (the binary still references it
    through the NVTX headers, which look up their injection library)."""
    import glob
    for f in glob.glob(os.path.join(ROOT, "paper_2507_14864_b200", "csrc", "*.cu*")):
        src = re.sub(r"//.*", "", open(f).read())
        assert "getenv" not in src, f


def test_binding_checks_lengths():
    """The binding refuses buffers shorter than the library will read or
    write (a short host output would be overrun by the device→host copy)."""
    import paper_2507_14864_b200 as fj

    class G:
        n = 10
    with pytest.raises(ValueError):
        fj.solve(G(), np.zeros(5, np.float32), np.zeros(10, np.float32), 1e-6)
    with pytest.raises(ValueError):
        fj.solve(G(), np.zeros(10, np.float32), np.zeros(9, np.float32), 1e-6)
    with pytest.raises(TypeError):
        fj.solve(G(), np.zeros(10, np.float64), np.zeros(10, np.float32), 1e-6)
    with pytest.raises(ValueError):
        fj.solve_batch(G(), np.zeros(10 * 3, np.float32), np.zeros(10 * 2, np.float32), 3, 1e-6)


def test_binding_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of fj_opts / fj_stats have the header's field names, order, offsets and
    sizes (a C program compiled against include/fj.h prints them)."""
    import subprocess
    import paper_2507_14864_b200 as fj
    fields = {"fj_opts": [n for n, _ in fj._Opts._fields_],
              "fj_stats": [n for n, _ in fj._Stats._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fj.h"', 'int main(void) {']
    for st, names in fields.items():
        lines.append(f'  printf("{st} %zu\\n", sizeof({st}));')
        for n in names:
            lines.append(f'  printf("{st}.{n} %zu\\n", offsetof({st}, {n}));')
    lines += ['  return 0;', '}']
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    for st, cls in (("fj_opts", fj._Opts), ("fj_stats", fj._Stats)):
        assert int(out[st]) == ctypes.sizeof(cls), st
        for n, _ in cls._fields_:
            assert int(out[f"{st}.{n}"]) == getattr(cls, n).offset, (st, n)
    o = fj._Opts()
    fj.lib().fj_opts_default(ctypes.byref(o))
    assert o.shadow == -1
    assert o.slices == -1
    assert o.frontier == -1
