"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/sv.h declares, and
the binding's enum tables match the header. No compute calls (no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sv.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sv_status|const char\*)\s+(sv_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("sv_create", "sv_apply_gate", "sv_apply_circuit", "sv_expectation", "sv_expectation_with_grad",
                     "sv_create_sharded", "sv_destroy", "sv_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_2406_17248_b200 as P
    for name in _declared_functions():
        assert hasattr(P.lib, name), name
    assert "sm_100a" in P.sv_version()


def test_kind_enum_matches_header():
    import paper_2406_17248_b200 as P
    src = open(HEADER).read()
    for name, code in P.KIND.items():
        m = re.search(r"\bSV_%s\s*=\s*(\d+)" % name, src)
        assert m and int(m.group(1)) == code, name


def test_library_is_sm100a_native():
    """The .so carries sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess
    import paper_2406_17248_b200 as P
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports or links the test oracle."""
    pkg = os.path.join(ROOT, "paper_2406_17248_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "sv_oracle" not in txt and "liboracle" not in txt, f


def test_library_then_torch_import():
    """libsv.so loaded before torch must not shadow torch's NCCL (one libnccl.so.2 per process):
    __graft_entry__.build() imports the package first, smoke() imports torch afterwards."""
    import subprocess
    import sys
    code = ("import ctypes, os; ctypes.CDLL(os.path.join('paper_2406_17248_b200', 'libsv.so')); "
            "import torch; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
