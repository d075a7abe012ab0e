"""Probe: where the split-TF32 error on large GGNN/gated hubs comes from.

Runs the library's GGNN (ReLU + sum) layer on the tests' power-law graph with a
hub of 1.5K / 6K / 20K in-edges and reports the normwise error against the fp64
oracle, then re-computes the GRU gates from the exact (fp64) message m with
torch cuBLAS on the tensor cores under different split / accumulation schemes
to separate operand representation from in-accumulator rounding.
(Measurement script, not product code.)"""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2009_00804_b200 as saga
from tests.test_gpu_parity import _zoo_inputs
from tests import harness as H

dev = "cuda"


def tf32(x):  # round-to-nearest tf32 of an fp32 tensor
    i = x.float().contiguous().view(torch.int32)
    i = (i + 0x1000) & ~0x1FFF
    return i.view(torch.float32)


def split(x):
    h = tf32(x)
    return h, tf32(x.float() - h)


def mm_tf32(a, b):
    torch.backends.cuda.matmul.allow_tf32 = True
    r = a.float() @ b.float()
    torch.backends.cuda.matmul.allow_tf32 = False
    return r.double()


def gru(gi, gh, h):
    r = torch.sigmoid(gi[0] + gh[0]); z = torch.sigmoid(gi[1] + gh[1])
    return (1 - z) * torch.tanh(gi[2] + r * gh[2]) + z * h


for hub in (1500, 6000, 20000):
    n = 2500
    rng = np.random.default_rng(7)
    s = rng.integers(0, n, 30000).astype(np.int32)
    d = np.minimum(rng.zipf(1.7, 30000) - 1, n - 1).astype(np.int32)
    d[:hub] = 11
    x = _zoo_inputs("ggnn", n, s, d, 3)
    dx = H.dev_inputs(dict(x, src=torch.from_numpy(s), dst=torch.from_numpy(d)), dev)
    g = saga.saga_graph_build(n, dx["src"], dx["dst"])
    lay = saga.Layer("ggnn", g, 128, 128, saga.SAGA_ACT_RELU, torch.float32, aggregator="sum")
    y = lay(dx["H"], {"W": dx["W_e"], "bias": dx["b_e"], "W_ih": dx["W_ih"], "W_hh": dx["W_hh"],
                      "b_ih": dx["b_ih"], "b_hh": dx["b_hh"]})
    torch.cuda.synchronize()
    og = oracle.csr_build(n, s, d)
    ref = oracle.ggnn(og, x["H"], x["W_e"], x["b_e"], x["W_ih"], x["W_hh"], x["b_ih"], x["b_hh"], act=1, agg="sum")
    print(f"hub {hub}: library err {oracle.rel_err(y.cpu().numpy(), ref):.3e}")
    rowe = np.abs(y.cpu().numpy() - ref).max(1) / np.abs(ref).max()
    top = np.argsort(-rowe)[:6]
    print("   worst rows (row, in-degree, err):", [(int(r), int(og.in_deg[r]), f"{rowe[r]:.2e}") for r in top])
    # exact m in fp64 (plain definition), then the GRU gates on the GPU
    Hd = x["H"].double(); We = x["W_e"].double()
    Y = torch.relu(torch.cat([Hd[s], Hd[d]], 1) @ We + x["b_e"].double())
    m = torch.zeros(n, 128, dtype=torch.float64).index_add_(0, torch.from_numpy(d).long(), Y)
    refd = torch.from_numpy(ref)
    m32 = m.float().to(dev); h32 = x["H"].to(dev)
    Wih = x["W_ih"].to(dev); Whh = x["W_hh"].to(dev)
    bih = x["b_ih"].double().to(dev); bhh = x["b_hh"].double().to(dev)
    hd = h32.double()

    def report(tag, gemm):
        gi = [gemm(m32, Wih[k]) + bih[k] for k in range(3)]
        gh = [gemm(h32, Whh[k]) + bhh[k] for k in range(3)]
        out = gru(gi, gh, hd).cpu()
        print(f"   {tag:38s} {(out - refd).abs().max().item() / refd.abs().max().item():.3e}")

    report("fp64 gemm of fp32 m", lambda a, b: a.double() @ b.double())
    report("cuBLAS fp32 (no tf32)", lambda a, b: (a @ b).double())

    def chain(a, b, terms, separate=False):
        ah, al = split(a); bh, bl = split(b)
        pairs = {"hh": (ah, bh), "hl": (ah, bl), "lh": (al, bh), "ll": (al, bl)}
        if separate:   # hi.hi in one accumulator, corrections in another, summed in fp64
            main = mm_tf32(ah, bh)
            rest = [pairs[t] for t in terms if t != "hh"]
            corr = mm_tf32(torch.cat([p[0] for p in rest], 1), torch.cat([p[1] for p in rest], 0))
            return main + corr
        A = torch.cat([pairs[t][0] for t in terms], 1)
        B = torch.cat([pairs[t][1] for t in terms], 0)
        return mm_tf32(A, B)

    def exact_terms(a, b, terms):
        ah, al = split(a); bh, bl = split(b)
        pairs = {"hh": (ah, bh), "hl": (ah, bl), "lh": (al, bh), "ll": (al, bl)}
        return sum(pairs[t][0].double() @ pairs[t][1].double() for t in terms)

    report("3xtf32, fp64 accumulation", lambda a, b: exact_terms(a, b, ["hh", "hl", "lh"]))
    report("4xtf32, fp64 accumulation", lambda a, b: exact_terms(a, b, ["hh", "hl", "lh", "ll"]))
    report("3xtf32 one TC chain (K interleaved)", lambda a, b: chain(a, b, ["hh", "hl", "lh"]))
    report("4xtf32 one TC chain", lambda a, b: chain(a, b, ["hh", "hl", "lh", "ll"]))
    report("3xtf32 hh chain + corr chain", lambda a, b: chain(a, b, ["hh", "hl", "lh"], True))
    report("4xtf32 hh chain + corr chain", lambda a, b: chain(a, b, ["hh", "hl", "lh", "ll"], True))

    # tensor-core accumulation of exact products: the hi.hi products of tf32 are exact in fp32,
    # so tf32 TC vs fp64 of the same hi.hi operands isolates the accumulator rounding
    ah, _ = split(m32); bh, _ = split(Wih[0])
    tc = mm_tf32(ah, bh); ex = ah.double() @ bh.double()
    dd = (tc - ex).abs()
    print(f"   hi.hi accumulate: max |TC - exact| {dd.max().item():.3e}  mean signed {(tc - ex).mean().item():.3e}"
          f"  max|exact| {ex.abs().max().item():.1f}  fp32 ulp there {torch.finfo(torch.float32).eps * ex.abs().max().item():.3e}")

# --- bias of the tensor-core fp32 accumulator (round 2): A = H W_a (K = 128) on
# cuBLAS TF32 (3-term split) vs fp32 SIMT vs exact; the mean of err * sign(A)
# is the systematic part that the GGNN Gather multiplies by the in-degree.
gen = torch.Generator().manual_seed(3)
Hb = torch.randn(20000, 128, generator=gen)
Wb = (torch.rand(128, 128, generator=gen) * 2 - 1) / np.sqrt(128)
ex = Hb.double() @ Wb.double()
Hc, Wc = Hb.to(dev), Wb.to(dev)
hh, wh = tf32(Hc), tf32(Wc)
hl, wl = tf32(Hc - hh), tf32(Wc - wh)
A3 = mm_tf32(torch.cat([hh, hh, hl], 1), torch.cat([wh, wl, wh], 0)).cpu()
A32 = (Hc @ Wc).double().cpu()
for tag, A in (("3xtf32 tensor cores", A3), ("fp32 SIMT (cuBLAS)", A32)):
    e = A - ex
    print(f"bias probe {tag:22s} max|err| {e.abs().max().item():.2e}  mean(err*sign(A)) "
          f"{(e * ex.sign()).mean().item():+.2e}")
