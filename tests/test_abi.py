"""The C-ABI library builds for sm_100a, loads here (no GPU) and exports every symbol include/*.h declares."""
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(spoly_\w+)\s*\(", txt):
            syms.add(m.group(1))
    return syms


def test_header_declares_the_boundary():
    s = declared_symbols()
    for f in ("spoly_create", "spoly_upload_mesh", "spoly_solve", "spoly_destroy"):
        assert f in s


def test_library_exports_every_declared_symbol():
    from paper_2405_13409_b200 import build, spoly
    lib = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib]).decode()
    exported = set(re.findall(r"\bT (spoly_\w+)", out))
    missing = declared_symbols() - exported
    assert not missing, missing
    L = spoly.lib()
    for s in declared_symbols():
        getattr(L, s)
    assert set(spoly.EXPORTS) <= declared_symbols()


def test_library_is_sm100a():
    from paper_2405_13409_b200 import build
    lib = build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib]).decode()
    assert "sm_100a" in out


def test_config_defaults_match_paper():
    from paper_2405_13409_b200 import spoly
    c = spoly.default_config()
    assert c.pieces == 100 and c.scan_bisect_iters == 10
    assert c.bisect_tol == 1e-9


def test_no_oracle_import_in_product():
    for f in glob.glob(os.path.join(ROOT, "paper_2405_13409_b200", "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h")):
            txt = open(f).read()
            assert "import oracle" not in txt and "oracle/" not in txt.replace("oracle/ ", ""), f


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors of spoly_config / spoly_report / spoly_result have the C layout."""
    import ctypes
    from paper_2405_13409_b200 import spoly
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "spoly.h"\nint main(void) {\n'
                   'printf("%zu %zu %zu %zu %zu\\n", sizeof(spoly_config), sizeof(spoly_report), sizeof(spoly_result),'
                   ' offsetof(spoly_report, n_rej_visibility), offsetof(spoly_result, report));\nreturn 0;\n}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    c_cfg, c_rep, c_res, c_off, c_roff = map(int, subprocess.check_output([str(exe)]).decode().split())
    assert ctypes.sizeof(spoly.spoly_config) == c_cfg
    assert ctypes.sizeof(spoly.spoly_report) == c_rep
    assert ctypes.sizeof(spoly.spoly_result) == c_res
    assert spoly.spoly_report.n_rej_visibility.offset == c_off
    assert spoly.spoly_result.report.offset == c_roff


def test_sqrt_table_host_copy_matches_golden():
    """The library's compiled sqrt-surrogate table (Eq. 20, reading R8) is the golden one; the device copy is
    filled from the same literal and read back from constant memory in tests/test_gpu_parity.py."""
    import numpy as np
    from paper_2405_13409_b200 import spoly
    g = np.loadtxt(os.path.join(ROOT, "tests", "golden", "sqrt_table.txt"))
    assert np.array_equal(spoly.sqrt_table(), g[:, :5])
