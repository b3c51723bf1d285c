"""The C-ABI library loads and exports exactly what include/dlrm_b200.h
declares (no GPU needed: nothing is launched)."""

import ctypes
import os
import re

from paper_1906_00091_b200 import _lib
from tests.conftest import ROOT


def declared():
    text = open(os.path.join(ROOT, "include", "dlrm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dlrm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    assert sorted(_lib.EXPORTS) == declared()


def test_size_queries_callable_without_gpu():
    assert _lib.size("dlrm_emb_bwd_workspace_size", 1000, 100, 16) > 1000 * 16
    assert _lib.size("dlrm_linear_bwd_weight_workspace_size", 2048, 64, 512) > 0
    assert _lib.size("dlrm_bce_head_workspace_size", 2048) >= 256 * 8
    assert b"sm_100a" in _lib.lib().dlrm_build_info()


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH],
                       capture_output=True, text=True)
    if r.returncode != 0:
        return  # cuobjdump unavailable
    elfs = [l for l in r.stdout.splitlines() if ".cubin" in l]
    assert elfs and all("sm_100a" in l for l in elfs)
