"""Breakdown of the C5 end-to-end step (dev tool): H2D, graph build, layer, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
import paper_2009_00804_b200 as saga
from tests import harness as H

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
dev = torch.device("cuda:0")
d = W.make_inputs(cfg, dev)
feats = [k for k in ("X", "H") if k in d]
host = {k: v.cpu().pin_memory() for k, v in d.items() if isinstance(v, torch.Tensor)}
def tm(f, n=3):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3, r
ms, _ = tm(lambda: [host[k].to(dev, non_blocking=True) for k in ("src", "dst") + tuple(feats)])
print("h2d ms", round(ms, 2))
ms, g = tm(lambda: H.gpu_graph(saga, cfg, d))
print("graph build ms", round(ms, 2))
outs, _ = H.gpu_step(saga, cfg, g, d)
ms, _ = tm(lambda: H.gpu_step(saga, cfg, g, d))
print("layer step ms (incl. python)", round(ms, 2))
oh = torch.empty(outs[-1].shape, dtype=outs[-1].dtype, pin_memory=True)
ms, _ = tm(lambda: oh.copy_(outs[-1], non_blocking=True))
print("d2h ms", round(ms, 2))
