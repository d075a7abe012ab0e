"""Hand-derived golden fixtures (tests/golden/*.txt, each with its
derivation and citation) for the GAT, gated-GRU and GraphSAGE-LSTM oracle
functions: tiny graphs with scalar features whose outputs are written out
from the definitions (readings A12-A16, A25), independent of the oracle."""
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    vals = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if ":" in line:
            k, v = line.split(":", 1)
            vals[k.strip()] = np.array([float(t) for t in v.split()])
    return vals


def _graph(n, g):
    return oracle.csr_build(n, g["src"].astype(np.int32), g["dst"].astype(np.int32))


def test_gat_golden():
    g = _load("gat_small.txt")
    y = oracle.gat(_graph(4, g), g["x"][:, None], np.eye(1), np.array([[1.0]]), np.array([[0.5]]), 0.2)
    np.testing.assert_allclose(y[:, 0], g["out"], rtol=1e-13, atol=1e-15)


def test_gru_golden():
    g = _load("gru_small.txt")
    y = oracle.gated(_graph(3, g), g["H"][:, None], np.ones((1, 1, 1)), g["w_ih"].reshape(3, 1, 1),
                     g["w_hh"].reshape(3, 1, 1), g["b_ih"].reshape(3, 1), g["b_hh"].reshape(3, 1))
    np.testing.assert_allclose(y[:, 0], g["out"], rtol=1e-13)


def test_lstm_golden():
    g = _load("lstm_small.txt")
    y = oracle.sage_lstm(_graph(3, g), g["x"][:, None], g["w_ih"].reshape(4, 1, 1), g["w_hh"].reshape(4, 1, 1),
                         g["b_ih"].reshape(4, 1), g["b_hh"].reshape(4, 1), g["W"].reshape(2, 1), g["b"], act=1)
    np.testing.assert_allclose(y[:, 0], g["out"], rtol=1e-13, atol=1e-15)
