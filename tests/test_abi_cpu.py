"""The C-ABI library loads on a CPU-only host and exports every symbol
include/kg.h declares; calls that need no device behave as documented.
No compute calls are made here."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "kg.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"KG_API\s+[\w\s\*]+?\b(kg_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("kg_init", "kg_set_key", "kg_submit_pages", "kg_wait"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1305_3345_b200 as kg
    lib = ctypes.CDLL(kg.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(kg.ABI_SYMBOLS) == declared_symbols()


def test_constants_match_header():
    import paper_1305_3345_b200 as kg
    src = open(HEADER).read()
    consts = dict((k, int(v)) for k, v in re.findall(r"#define (KG_\w+)\s+(-?\d+)", src))
    assert consts["KG_ENCRYPT"] == kg.ENCRYPT and consts["KG_DECRYPT"] == kg.DECRYPT
    assert consts["KG_MODE_CBC"] == kg.MODE_CBC and consts["KG_MODE_ECB"] == kg.MODE_ECB
    for name in ("OK", "EINVAL", "ENOKEY", "ENOTINIT", "EAGAIN", "ENOMEM", "ECUDA", "ENOTSUP", "ETICKET"):
        assert consts["KG_" + name] == getattr(kg, name), name
    assert consts["KG_MAX_KEYS"] == kg.MAX_KEYS


def test_strerror_and_not_initialised():
    import paper_1305_3345_b200 as kg
    for code in range(-8, 1):
        assert kg.strerror(code)
    assert kg.strerror(-99) == "unknown status"
    lib = kg.raw_lib()
    assert lib.kg_set_key(0, b"\0" * 16, 16) == kg.ENOTINIT
    assert lib.kg_submit_pages(0, 0, 16, 16, 1, 16, 16, 0, None) == kg.ENOTINIT
    assert lib.kg_wait(0) == kg.ENOTINIT
    assert lib.kg_poll(0) == kg.ENOTINIT
    assert lib.kg_shutdown() == kg.ENOTINIT
    assert lib.kg_set_pipeline(1 << 20, 3) == kg.ENOTINIT
    assert kg.launch_count() == 0


def test_kernel_image_is_sm100a():
    """The library carries sm_100a SASS (cross-compiled here, no GPU needed)."""
    import shutil
    import subprocess
    import paper_1305_3345_b200 as kg
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", kg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_header_is_plain_c_and_cxx(tmp_path):
    """include/kg.h compiles as C99 and as C++ (no torch or CUDA types)."""
    import subprocess
    src = tmp_path / "t.c"
    src.write_text('#include "kg.h"\nint main(void){ return kg_strerror(KG_OK) == 0; }\n')
    inc = os.path.join(ROOT, "include")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only", "-I", inc, str(src)])
    subprocess.check_call(["g++", "-std=c++11", "-Wall", "-Werror", "-fsyntax-only", "-x", "c++", "-I", inc, str(src)])


def test_example_links_against_the_library(tmp_path):
    import subprocess
    import paper_1305_3345_b200 as kg
    exe = tmp_path / "kgpu_crypt"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "kgpu_crypt.c"), "-L", os.path.dirname(kg.LIB_PATH),
                           "-lkgpu", f"-Wl,-rpath,{os.path.dirname(kg.LIB_PATH)}", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 2 and "usage" in out.stderr


def test_enotsup_without_a_device():
    """kg_init on a process that sees no CUDA device -> KG_ENOTSUP (the
    library still loads; no compute call is made)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import paper_1305_3345_b200 as kg; "
            "print(kg.raw_lib().kg_init(0))" % ROOT)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    import paper_1305_3345_b200 as kg
    assert int(r.stdout.strip().splitlines()[-1]) == kg.ENOTSUP
