"""CPU-only checks of the drop-in boundary: the product library and the oracle
shim load without a GPU and export every symbol include/mdnn.h declares."""
import os
import re

from conftest import REPO
from paper_2202_14005_b200.capi import EXPORTED_SYMBOLS, Lib


def _declared():
    hdr = open(os.path.join(REPO, "include", "mdnn.h")).read()
    return set(re.findall(r"\b(mdnn_[a-z0-9_]+)\s*\(", hdr))


def test_header_and_binding_agree():
    assert _declared() == set(EXPORTED_SYMBOLS)


def test_product_library_loads_and_exports_everything():
    from paper_2202_14005_b200 import load_library
    lib = load_library()
    assert lib.backend == "b200-sm100a"
    for s in _declared():
        assert hasattr(lib.so, s), s


def test_oracle_shim_exports_everything(ref):
    assert ref.backend == "reference-cpu-f32"
    for s in _declared():
        assert hasattr(ref.so, s), s


def test_reference_counts(ref):
    from paper_2202_14005_b200.mdnn import Model
    assert Model.varnet(ref, im_x=16, im_y=16, coils=2).num_real_params() == 65530
    assert Model.modl(ref, im_x=16, im_y=16, coils=2).num_real_params() == 56963


def test_product_builds_graphs_without_gpu():
    """Graph construction is host-only: the MoDL/VarNet builders run on CPU."""
    from paper_2202_14005_b200 import load_library
    from paper_2202_14005_b200.mdnn import Model
    lib = load_library()
    assert Model.varnet(lib, im_x=16, im_y=16, coils=2).num_real_params() == 65530
