"""Dump the destination-sorted col_src of a config graph (dev probe input)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2009_00804_b200 as saga
cfg = W.CONFIGS[sys.argv[1]]
s, d, et = W.make_graph(cfg, "cuda")
g = saga.saga_graph_build(cfg.n, s, d, et, cfg.num_etypes)
c = g.csr()["col_src"].cpu().numpy()
c.tofile(sys.argv[2])
print(cfg.n, c.shape)
