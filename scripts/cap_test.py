import sys; sys.path.insert(0, '/root/repo')
import torch
import workloads as W
import paper_2009_00804_b200 as saga
from tests import harness as H
cfg = W.scaled(W.CONFIGS["C3"], 5000, 60000, "t")
d = W.make_inputs(cfg, "cuda")
g = H.gpu_graph(saga, cfg, d)
outs, layers = H.gpu_step(saga, cfg, g, d)
torch.cuda.synchronize()
for prof in (False, True):
    saga.saga_profile_enable(prof)
    gr = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(gr):
            H.gpu_step(saga, cfg, g, d, layers, outs)
        gr.replay(); torch.cuda.synchronize()
        print("prof", prof, "capture ok", saga.saga_profile_read() if prof else "")
    except Exception as e:
        print("prof", prof, "FAILED", e)
    saga.saga_profile_enable(False)
# bench-like: flush + external timing events around the step
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
for variant in ("events", "flush", "both"):
    saga.saga_profile_enable(True)
    st = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    en = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    gr = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(gr):
            for i in range(3):
                if variant in ("flush", "both"):
                    flush.zero_()
                if variant in ("events", "both"):
                    st[i].record()
                H.gpu_step(saga, cfg, g, d, layers, outs)
                if variant in ("events", "both"):
                    en[i].record()
        gr.replay(); torch.cuda.synchronize()
        print(variant, "ok", saga.saga_profile_read(), [s.elapsed_time(e) for s, e in zip(st, en)] if variant != "flush" else "")
    except Exception as e:
        print(variant, "FAILED", e)
    saga.saga_profile_enable(False)
