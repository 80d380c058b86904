"""The boundary proven from the reference side: include/mdnn_b200_node.hpp
(the NlopNode adapter a reference maintainer adds, nlop.hpp:18-83) compiled
against the unmodified reference headers into oracle/_ref/b200_splice
(oracle/Makefile), splicing the B200 S = A^H A + lambda into reference graphs
-- alone, under the reference's own InverseNode (host CG calling the B200
operator every iteration) and in a reference chain -- and comparing with the
same graphs over the reference operator (tests/adapter/splice_main.cpp)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "b200_splice")

pytestmark = pytest.mark.gpu


def test_reference_graph_splices_b200_operator(gpu):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/b200_splice not built (make -C oracle)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SPLICE OK" in r.stdout
