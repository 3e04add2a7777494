"""CPU checks of the C-ABI boundary: the library loads, exports every
function include/wfpg_b200.h declares, the ctypes layouts match the header
sizes, and argument validation reports WFPG_ERR_ARG without touching a GPU."""

import ctypes as C
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "wfpg_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wfpg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2405_06997_b200 import _lib

    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 30
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared) <= set(_lib.EXPORTED), set(declared) - set(_lib.EXPORTED)
    assert lib.wfpg_abi_version() == 1


def test_argument_validation_without_gpu():
    from paper_2405_06997_b200 import _lib

    lib = _lib.load()
    # NULL svo -> WFPG_ERR_ARG with a message, no device work
    assert lib.wfpg_svo_propagate(None, None) == 1
    assert b"bad arguments" in lib.wfpg_last_error()
    s = _lib.Svo()
    s.depth, s.resolution = 3, 16  # resolution != 2**depth
    assert lib.wfpg_descend(C.byref(s), None, 0, None, None, None, None) == 1
    assert lib.wfpg_sort_pairs_u64(None, None, 10, None, 0, None, 0, None) == 1


def test_workspace_queries_are_host_only():
    from paper_2405_06997_b200 import _lib

    lib = _lib.load()
    assert lib.wfpg_scan_workspace_bytes(1 << 20) > 0
    assert lib.wfpg_sort_workspace_bytes(1 << 20) > (1 << 20) * 12
    assert lib.wfpg_svo_build_workspace_bytes(100000, 8) > 100000 * 8
    assert lib.wfpg_partition_workspace_bytes(4096, 1 << 20) > 0
    assert lib.wfpg_update_exitance_workspace_bytes(4096, 4) > 4096 * 4 * 4


@pytest.mark.parametrize("sid,name", sorted({0: "Scene", 1: "Camera", 2: "Svo", 3: "Paths",
                                               4: "Guide", 5: "PassConfig",
                                               6: "PassStats"}.items()))
def test_struct_layouts_match_the_c_build(sid, name):
    """Every ctypes mirror has the C build's sizeof and the offset of every
    field (wfpg_abi_sizeof / wfpg_abi_offsetof), and names every header field:
    a layout drift between include/wfpg_b200.h and _lib.py fails here."""
    from paper_2405_06997_b200 import _lib

    lib = _lib.load()
    assert _lib.ABI_STRUCTS[sid] == name
    st = getattr(_lib, name)
    assert lib.wfpg_abi_sizeof(sid) == C.sizeof(st)
    for field, _ in st._fields_:
        assert lib.wfpg_abi_offsetof(sid, field.encode()) == getattr(st, field).offset, field
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    cname = {"PassConfig": "pass_config", "PassStats": "pass_stats"}.get(name, name.lower())
    body = re.search(r"typedef struct wfpg_%s \{(.*?)\} wfpg_%s;" % (cname, cname), text,
                     re.S).group(1)
    header_fields = [re.search(r"([A-Za-z_]\w*)\s*(\[[^\]]*\])*\s*$", d.strip()).group(1)
                     for d in body.split(";") if d.strip()]
    assert header_fields == [f for f, _ in st._fields_]
    assert lib.wfpg_abi_offsetof(sid, b"no_such_field") == -1
