"""-m "not gpu": the C-ABI library builds for sm_100a, loads, and exports every symbol
include/gcctb.h declares; the binding declares exactly those names."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gcctb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2406_10158_b200 import build as B
    lib_path = B.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path]).decode()
    exported = set(re.findall(r" T (cc_[a-z_]+)$", out, flags=re.M))
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [d for d in declared if d not in exported]
    assert not missing, f"declared but not exported: {missing}"


def test_binding_matches_header_and_loads():
    from paper_2406_10158_b200 import build as B, gcctb
    B.build()
    assert gcctb.EXPORTED == _declared()
    L = gcctb.lib()
    assert b"sm_100a" in L.cc_version()


def test_library_is_sm100a_sass():
    from paper_2406_10158_b200 import build as B
    lib_path = B.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path]).decode()
    assert "sm_100a" in out


def test_no_oracle_import_in_product_path():
    pkg = os.path.join(ROOT, "paper_2406_10158_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
                assert "oracle_ycsb" not in s and "liboracle" not in s, f


def test_binding_flag_values_match_header():
    """Every CC_FLAG_* the header defines has the same value in the Python binding."""
    from paper_2406_10158_b200 import gcctb
    src = open(os.path.join(ROOT, "include", "gcctb.h")).read()
    flags = dict(re.findall(r"#define (CC_FLAG_[A-Z0-9_]+) (0x[0-9a-fA-F]+)u", src))
    assert len(flags) >= 12
    for name, val in flags.items():
        assert hasattr(gcctb, name), name
        assert getattr(gcctb, name) == int(val, 16), name
    assert len(set(int(v, 16) for v in flags.values())) == len(flags)   # distinct bits
