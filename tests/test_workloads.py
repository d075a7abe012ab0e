"""Input recipe checks (readings A2-A5, A10, A17)."""
import math

import numpy as np
import pytest
import torch

import workloads as W


def test_mix64_matches_reference_splitmix64():
    # splitmix64 finaliser written with Python ints (arbitrary precision)
    def ref(x):
        M = (1 << 64) - 1
        z = (x + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    xs = [0, 1, 2, 12345, (1 << 63) - 1, 1 << 40]
    got = W.mix64(torch.tensor(xs, dtype=torch.int64)).tolist()
    assert [g & ((1 << 64) - 1) for g in got] == [ref(x) for x in xs]


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_graph_recipe(name):
    c = W.CONFIGS[name]
    s, d, et = W.make_graph(c)
    s2, d2, et2 = W.make_graph(c)
    assert torch.equal(s, s2) and torch.equal(d, d2)                 # seeded, deterministic
    assert s.numel() == c.num_edges and s.dtype == torch.int32
    assert int(s.min()) >= 0 and int(s.max()) < c.n and int(d.max()) < c.n
    gen_s, gen_d = s[: c.m], d[: c.m]
    assert int((gen_s == gen_d).sum()) == 0                          # A2: generated self-loops dropped
    if c.self_loops:
        assert torch.equal(s[c.m:], torch.arange(c.n, dtype=torch.int32))
        assert torch.equal(d[c.m:], torch.arange(c.n, dtype=torch.int32))
    if c.dedup:                                                       # A3/A4: distinct pairs
        key = gen_s.long() * c.n + gen_d.long()
        assert torch.unique(key).numel() == c.m
    if c.num_etypes > 1:
        assert et is not None and int(et.min()) >= 0 and int(et.max()) == c.num_etypes - 1
        frac = torch.bincount(et.long()).double() / et.numel()
        assert torch.all((frac - 0.25).abs() < 0.01)


def test_rmat_skew_and_device_independent_topology():
    c = W.scaled(W.CONFIGS["C3"], 1 << 12, 1 << 16, "rmat12")
    s, d, _ = W.make_graph(c)
    deg = torch.bincount(d[: c.m].long(), minlength=c.n)
    assert deg.max() > 20 * deg.float().mean()                       # power-law hubs
    assert (deg == 0).float().mean() > 0.2
    # integer draws are pure int64 arithmetic -> identical on any device
    key = W.stream_key(3, "x")
    a = W.draw_bits(key, torch.arange(1000, dtype=torch.int64), 24)
    assert int(a.min()) >= 0 and int(a.max()) < (1 << 24)


def test_features_and_weights():
    c = W.scaled(W.CONFIGS["C5"], 4096, 1 << 15)
    x = W.make_inputs(c, graph=False)
    assert x["X"].dtype == torch.bfloat16 and x["X"].shape == (4096, 256)
    assert abs(float(x["X"].float().std()) - 1.0) < 0.02
    bound = math.sqrt(6 / 512)
    assert float(x["W"].float().abs().max()) <= bound * (1 + 2 ** -8)
    c1 = W.make_inputs(W.CONFIGS["C1"], graph=False)
    assert c1["X"].dtype == torch.float32 and float(c1["X"].abs().max()) <= 1.0
    g = W.make_inputs(W.CONFIGS["C4"], graph=False)
    assert g["W_ih"].shape == (3, 128, 128) and float(g["W_ih"].abs().max()) <= 1 / math.sqrt(128)
