"""Short driver for ncu captures: a few config-3 decisions (direct launches) and one
1M-request QoE evaluation (the bench's S1 throughput run)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402
from bench import _tile  # noqa: E402

snap = W.config3()
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
for _ in range(int(os.environ.get("DECISIONS", "3"))):
    ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16)
torch.cuda.synchronize()
if os.environ.get("QOE", "1") == "1":
    big = _tile(snap, 16)
    q = A.Context(max_requests=big.n, max_B=8, max_tokens=big.n_tokens + 64)
    breq = A.requests_to(big)
    for _ in range(2):
        q.qoe_eval(breq, big.n, big.now_us + big.horizon_us, A.ANDES_EVAL_INFLIGHT)
    torch.cuda.synchronize()
print("done")
