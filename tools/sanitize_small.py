"""Small decisions and QoE evaluations for compute-sanitizer (memcheck / racecheck runs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

ctx = A.Context(max_requests=8192, max_B=64, max_tokens=1 << 22, max_running=4096)
for seed in range(6):
    snap = W.random_small(seed, align=[4, 1][seed % 2], n=30, max_tokens=300, B_cap=16)
    req = A.requests_to(snap)
    tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
    for fl in (1, 1 | 16, 1 | 32, 1 | 64, 1 | 128):
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=2, flags=fl)
    ctx.qoe_eval(req, snap.n, snap.now_us, A.ANDES_EVAL_FINAL)
snap = W.long_requests(3, n=60, lo=5000, hi=9000)
req = A.requests_to(snap)
ctx.qoe_eval(req, snap.n, snap.now_us, A.ANDES_EVAL_INFLIGHT)
torch.cuda.synchronize()
print("sanitize run ok")
