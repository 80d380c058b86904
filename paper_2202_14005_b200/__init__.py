"""B200-native MoDL / VarNet training hot path (arXiv 2202.14005).

The product is the C++/CUDA library `libmdnn_b200.so` (built in-tree from
csrc/, sm_100a only) behind the C ABI in include/mdnn.h.  This package only
locates and loads it; there is no Python or CPU compute path, and loading
fails loudly if the extension is missing.
"""
from __future__ import annotations

import os

from .capi import Lib, MdnnError  # noqa: F401

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("MDNN_B200_LIB") or os.path.join(PKG_DIR, "libmdnn_b200.so")  # env: A/B builds

_lib = None


def load_library() -> Lib:
    """The product library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                               f"paper_2202_14005_b200/csrc) first; there is no fallback path")
        _lib = Lib(LIB_PATH)
    return _lib
