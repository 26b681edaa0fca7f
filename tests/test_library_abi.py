"""CPU checks of the boundary: the C-ABI library builds, loads and exports every symbol that
include/chase.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "chase.h")).read()
    return sorted(set(re.findall(r"^\s*(?:chase_status|const char\*|unsigned long long)\s+(chase_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("chase_init", "chase_solve", "chase_finalize", "chase_set_option", "chase_local_layout",
              "chase_last_error", "chase_filter", "chase_hemm_step", "chase_lanczos"):
        assert n in names


def test_library_loads_and_exports_all_declared_symbols():
    import paper_2205_02491_b200 as pkg
    lib = pkg.load()
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(pkg.EXPORTS) <= set(_declared())
    assert "sm_100a" in pkg.version()


def test_generator_twin_library_loads():
    lib = ctypes.CDLL(os.path.join(ROOT, "chase_gen", "libchase_gen.so"))
    assert hasattr(lib, "chase_gen_g2_block")


def test_library_is_sm100a_only():
    """The shipped cubin is sm_100a (cuobjdump lists the embedded ELF arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    so = os.path.join(ROOT, "paper_2205_02491_b200", "libchase_b200.so")
    out = subprocess.run([exe, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def _build_example(out):
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    lib = os.path.join(root, "paper_2205_02491_b200")
    cmd = ["gcc", "-O2", "-std=c11", os.path.join(root, "examples", "chase_example.c"),
           "-I" + os.path.join(root, "include"), "-I/usr/local/cuda/include", "-L" + lib, "-lchase_b200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-Wl,-rpath," + lib, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_plain_c_example_compiles_and_links(tmp_path):
    """The boundary is a C ABI: a plain C11 program (no torch, no Python) builds against
    include/chase.h and links libchase_b200.so."""
    _build_example(str(tmp_path / "chase_example"))


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No fallback path: with the shared library absent the binding raises instead of computing."""
    from paper_2205_02491_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libchase_b200.so"))
    with pytest.raises(ImportError, match="no fallback"):
        _lib.load()


def test_product_package_never_references_the_oracle():
    """The product path (package sources, CUDA included) shares nothing with oracle/."""
    pkg_dir = os.path.join(ROOT, "paper_2205_02491_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(?:import|from)\s+oracle\b|#include\s+[\"<][^\">]*oracle", src, re.M), f


def test_init_args_layout_matches_header(tmp_path):
    """The binding's ctypes chase_init_args / chase_report mirror include/chase.h byte for byte
    (sizeof and every field offset, from a C program compiled against the header)."""
    import shutil
    import subprocess
    from paper_2205_02491_b200._lib import InitArgs, Report
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    fields = [f for f, _ in InitArgs._fields_]
    rfields = [f for f, _ in Report._fields_]
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "chase.h"', "int main(void) {",
           '  printf("%zu\\n", sizeof(chase_init_args));']
    src += [f'  printf("%zu\\n", offsetof(chase_init_args, {f}));' for f in fields]
    src += ['  printf("%zu\\n", sizeof(chase_report));']
    src += [f'  printf("%zu\\n", offsetof(chase_report, {f}));' for f in rfields]
    src += ["  return 0;", "}"]
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    r = subprocess.run(["gcc", "-std=c11", str(c), "-I" + os.path.join(ROOT, "include"), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(InitArgs)] + [getattr(InitArgs, f).offset for f in fields]
    want += [ctypes.sizeof(Report)] + [getattr(Report, f).offset for f in rfields]
    assert got == want
