"""Parity helpers for the tests: the checker lives in oracle/paritycheck.py
(shared with bench.py's correctness gate); see there for the tolerances."""
from paritycheck import (NEAR_TIE, REL, ParityReport, compare_detections, delta_tolerance,  # noqa: F401
                         direct_xcorr, near_tie_margin, pc_scale)
