"""Pins for the oracle's CSR build (S0): PAPER.md lines 130, 351-354; reading A7.

Pinned against NumPy stable argsort + bincount (a library routine computing
the same multiset grouping independently), the SPEC examples (SPEC.md lines
59-61, 67-69) and a hand-written golden fixture.
"""
import os

import numpy as np
import pytest

import oracle
from tests import zoo
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def numpy_csr(n, src, dst):
    order = np.argsort(dst, kind="stable")
    deg = np.bincount(dst, minlength=n).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    return row_ptr, src[order], order.astype(np.int32), deg, np.bincount(src, minlength=n).astype(np.int32)


@pytest.mark.parametrize("name,n,src,dst", zoo.zoo(include_big=True), ids=lambda x: x if isinstance(x, str) else "")
def test_csr_matches_numpy_stable_sort(name, n, src, dst):
    g = oracle.csr_build(n, src, dst)
    rp, cs, eid, ind, outd = numpy_csr(n, src, dst)
    np.testing.assert_array_equal(g.row_ptr, rp)
    np.testing.assert_array_equal(g.col_src, cs)
    np.testing.assert_array_equal(g.edge_id, eid)
    np.testing.assert_array_equal(g.in_deg, ind)
    np.testing.assert_array_equal(g.out_deg, outd)
    assert g.in_deg.sum() == src.shape[0]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_csr_config_graphs(cfg):
    c = W.CONFIGS[cfg]
    s, d, et = W.make_graph(c)
    s, d = s.numpy(), d.numpy()
    g = oracle.csr_build(c.n, s, d, et, c.num_etypes)
    rp, cs, eid, ind, _ = numpy_csr(c.n, s, d)
    np.testing.assert_array_equal(g.row_ptr, rp)
    np.testing.assert_array_equal(g.col_src, cs)
    np.testing.assert_array_equal(g.edge_id, eid)
    if et is not None:
        np.testing.assert_array_equal(g.etype, et.numpy()[eid])


def test_spec_examples():
    g = oracle.csr_build(2, np.array([0, 1], np.int32), np.array([1, 0], np.int32))
    assert g.row_ptr.tolist() == [0, 1, 2]
    g = oracle.csr_build(3, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert g.row_ptr.tolist() == [0, 0, 0, 0]
    g = oracle.csr_build(6, np.arange(1, 6, dtype=np.int32), np.zeros(5, np.int32))
    assert g.in_deg.tolist() == [5, 0, 0, 0, 0, 0]             # SPEC.md line 67 (star)


def test_coo_roundtrip_multiset():
    s, d = zoo.random_multigraph(200, 3000, 5)
    et = (np.arange(3000) % 3).astype(np.int32)
    g = oracle.csr_build(200, s, d, et, 3)
    dst_csr = np.repeat(np.arange(200), np.diff(g.row_ptr))
    a = sorted(zip(g.col_src.tolist(), dst_csr.tolist(), g.etype.tolist()))
    b = sorted(zip(s.tolist(), d.tolist(), et.tolist()))
    assert a == b


def test_out_of_range_reports_lowest_index():
    s = np.array([0, 1, 2, 9, 1, -1], np.int32)
    d = np.array([1, 2, 0, 0, 7, 0], np.int32)
    with pytest.raises(oracle.OracleRangeError) as ei:
        oracle.csr_build(3, s, d)
    assert ei.value.index == 3
    et = np.array([0, 0, 5, 0], np.int32)
    with pytest.raises(oracle.OracleRangeError) as ei:
        oracle.csr_build(3, s[:3], d[:3], et[:3], 2)
    assert ei.value.index == 2


def test_golden_small_csr():
    """tests/golden/csr_small.txt: a hand-built 5-vertex multigraph."""
    lines = [l.split("#")[0].strip() for l in open(os.path.join(GOLDEN, "csr_small.txt"))]
    kv = {}
    for l in lines:
        if ":" in l:
            k, v = l.split(":", 1)
            kv[k.strip()] = [int(t) for t in v.split()]
    n = kv["n"][0]
    g = oracle.csr_build(n, np.array(kv["src"], np.int32), np.array(kv["dst"], np.int32))
    assert g.row_ptr.tolist() == kv["row_ptr"]
    assert g.col_src.tolist() == kv["col_src"]
    assert g.edge_id.tolist() == kv["edge_id"]
    assert g.in_deg.tolist() == kv["in_deg"]
    assert g.out_deg.tolist() == kv["out_deg"]
