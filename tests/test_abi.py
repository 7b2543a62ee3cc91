"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/plex.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "plex.h")).read()
    return sorted(set(re.findall(r"^PLEX_API\s+[\w\s\*]*?\b(plex_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("plex_transition_plan", "plex_state_offload", "plex_state_onload", "plex_weight_sync"):
        assert n in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2605_20863_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == _declared()


def test_version_and_error_string():
    from paper_2605_20863_b200 import _lib
    assert b"sm_100a" in _lib.lib.plex_version()
    import ctypes as C
    h = C.c_void_p()
    assert _lib.lib.plex_transition_plan(None, C.byref(h)) == _lib.E_INVAL
    assert b"manifest" in _lib.lib.plex_last_error()


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libplex.so the package refuses to import."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_2605_20863_b200"
    shutil.copytree(os.path.join(ROOT, "paper_2605_20863_b200"), pkg,
                    ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2605_20863_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "libplex.so" in r.stderr and "ImportError" in r.stderr
