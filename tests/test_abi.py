"""CPU checks of the C-ABI boundary: the library builds/loads and exports every
symbol include/tac.h declares; the binding refuses to run without a GPU."""
import os
import re

import pytest

import paper_2603_28475_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "tac.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tac_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    d = declared()
    for name in ("tac_create", "tac_step", "tac_markers"):
        assert name in d


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for name in declared():
        assert hasattr(L, name), name
    assert sorted(P.EXPORTED) == declared()


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import workloads as w
    s = w.scene_c1()
    with pytest.raises(P.TacError):
        P.TacSim.from_scene(s)


def test_product_does_not_import_oracle():
    for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2603_28475_b200")):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("oracle-verified", ""), f


def test_nccl_unique_id_through_the_c_abi():
    """tac_nccl_unique_id resolves NCCL at run time (no link dependency of libtac.so) and
    returns a fresh 128-byte id; host-only, no GPU needed."""
    a, b = P.nccl_unique_id(), P.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
    import subprocess
    out = subprocess.run(["ldd", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "nccl" not in out


def test_gather_markers_rejects_bad_arguments():
    L = P.lib()
    assert L.tac_gather_markers(None, None, None, 2, None) != 0
    assert L.tac_nccl_comm_create(None, 1, 0, 0, None) != 0
