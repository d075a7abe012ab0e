# Worst-case fp32 accuracy probe: the 70K-in-degree hub of the test zoo, gated model,
# tensor-core path vs the FFMA reference kernels (SAGA_GATED_SIMT=1).
cat > /tmp/hub.py <<'PY'
import torch, numpy as np, sys, os
sys.path.insert(0, '.')
import oracle, workloads as W
import paper_2009_00804_b200 as saga
from tests import harness as H, zoo
from tests.test_gpu_parity import _zoo_inputs, _zoo_cfg
for name, n, s, d in zoo.zoo(include_big=True):
    if name != 'hub70k': continue
    cfg = _zoo_cfg('gated', n, s.shape[0])
    x = _zoo_inputs('gated', n, s, d, 7)
    x['src'], x['dst'] = torch.from_numpy(s), torch.from_numpy(d)
    x['etype'] = torch.from_numpy((np.arange(s.shape[0]) * 7 % 4).astype(np.int32))
    dx = H.dev_inputs(x, 'cuda')
    g = H.gpu_graph(saga, cfg, dx)
    outs, _ = H.gpu_step(saga, cfg, g, dx)
    og = H.oracle_graph(oracle, cfg, x)
    ref = H.oracle_step(oracle, cfg, og, x)[0]
    y = H.to_np(outs[0])
    err = np.abs(y - ref)
    print(os.environ.get('TAG'), 'hub70k gated rel err', oracle.rel_err(y, ref), 'worst row', err.max(1).argmax(), 'in_deg', og.in_deg[err.max(1).argmax()], 'err row0', err[0].max())
PY
TAG=tc timeout 300 python /tmp/hub.py
TAG=simt SAGA_GATED_SIMT=1 timeout 300 python /tmp/hub.py
TAG=tc_t37888 SAGA_TASK_TARGET=37888 timeout 300 python /tmp/hub.py
TAG=simt_t37888 SAGA_GATED_SIMT=1 SAGA_TASK_TARGET=37888 timeout 300 python /tmp/hub.py
