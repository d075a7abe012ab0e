"""Pins of the parity metrics (SURVEY.md 8(c) "Error metric" row; reading A18):
hand-computed values, so a wrong axis, a missing floor or a swapped operand fails."""
import numpy as np

import oracle


def test_rel_err_hand_values():
    ref = np.array([[1.0, -4.0], [0.5, 2.0]])
    y = np.array([[1.0, -3.5], [0.5, 2.0]])
    assert oracle.rel_err(y, ref) == 0.5 / 4.0          # max |dy| / max |ref|
    assert oracle.rel_err(ref, ref) == 0.0
    assert oracle.rel_err(np.array([[np.nan]]), np.array([[1.0]])) == float("inf")
    assert oracle.rel_err(np.zeros((2, 2)) + 1e-3, np.zeros((2, 2))) == 1e-3   # all-zero ref: absolute


def test_row_err_hand_values():
    ref = np.array([[100.0, 0.0], [1.0, 1.0], [0.0, 0.0]])
    y = np.array([[100.0, 0.0], [1.0, 1.5], [0.05, 0.0]])
    e, row = oracle.row_err(y, ref)
    # row 1: 0.5 / max(1, 0.1) = 0.5; row 2 (all-zero ref row): 0.05 / (1e-3 * 100) = 0.5
    assert row in (1, 2) and abs(e - 0.5) < 1e-15
    y[2, 0] = 0.2
    e, row = oracle.row_err(y, ref)
    assert row == 2 and abs(e - 2.0) < 1e-15
    # normwise hides the small wrong row that the per-row view catches
    assert oracle.rel_err(y, ref) == 0.5 / 100.0


def test_row_err_degenerate():
    assert oracle.row_err(np.zeros((0, 4)), np.zeros((0, 4))) == (0.0, -1)
    assert oracle.row_err(np.array([[np.inf]]), np.array([[1.0]]))[0] == float("inf")
    e, row = oracle.row_err(np.array([[0.0], [0.25]]), np.zeros((2, 1)))
    assert (e, row) == (0.25, 1)
