"""The C-ABI library builds for sm_100a, loads and exports every symbol include/dmtz.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dmtz.h")
LIB = os.path.join(ROOT, "paper_2409_17346_b200", "libdmtz.so")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dmtz_[a-z_]+)\s*\(", txt)))


def test_library_builds_and_exports_header_symbols():
    from paper_2409_17346_b200 import build
    build.build()
    lib = ctypes.CDLL(LIB)
    names = _declared()
    assert "dmtz_correct" in names and "dmtz_compute_gradient" in names and "dmtz_trace_separatrices" in names
    for n in names:
        assert hasattr(lib, n), n


def test_binding_exports_match_header():
    import paper_2409_17346_b200 as d
    assert set(_declared()) == set(d.EXPORTED)
    assert d.lib().dmtz_version() >= 1
    assert d.lib().dmtz_status_string(d.E_STUCK).startswith(b"stuck")


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tables_header_current():
    gen = os.path.join(ROOT, "tools", "gen_tables.py")
    assert subprocess.call(["python", gen, "--check"]) == 0


def test_gpu_tables_match_oracle_complex():
    """The generated GPU tables (tools/gen_tables.py) and the oracle derive the complex
    independently; their link orders and vertex offsets must agree."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_tables
    import oracle
    for D, shape in ((2, (3, 3)), (3, (3, 3, 3))):
        info = gen_tables.build(D)
        oi = oracle.complex_info(shape)
        assert oi["T"] == len(info)
        for t, it in enumerate(info):
            assert oi["dim"][t] == it["dim"]
            assert [tuple(x) for x in oi["offsets"][t][:it["dim"] + 1]] == it["verts"]
            assert [tuple(x) for x in oi["links"][t][:oi["nlink"][t]]] == it["link"]
