"""CPU check of the generated register DFT codelets (no GPU needed): each
codelet body is executed in float64 and compared with a direct DFT."""
import os

from codelet_check import check_all

HERE = os.path.dirname(__file__)
CODELETS = os.path.join(HERE, "..", "paper_2005_10445_b200", "csrc", "codelets.cuh")


def test_codelets_match_dft():
    worst = check_all(CODELETS)
    assert len(worst) >= 48
    bad = {k: v for k, v in worst.items() if v > 1e-6}   # constants are float-rounded
    assert not bad, bad
