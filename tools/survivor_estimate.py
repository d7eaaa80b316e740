"""Design probe: how many requests can be in some top-B set, under ideal per-request key
bounds (min/max over B of the exact keys), for config 3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

snap = W.config3()
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
gain, key, qw = ctx.gain_estimate(req, snap.n, snap.now_us, snap.horizon_us, tau, np.arange(1, 257))
K = key.double()
rank = torch.arange(snap.n, device="cuda", dtype=torch.float64)
print("keys>0 frac", (K > 0).double().mean().item(), "keys==0", (K == 0).double().mean().item())
union = torch.zeros(snap.n, dtype=torch.bool, device="cuda")
for B in range(1, 257):
    top = torch.topk(K[B - 1], B).indices
    union[top] = True
print("union of top-B sets", int(union.sum()))
for G in (1, 2, 4, 8, 16, 32, 64, 256):
    w = 256 // G
    tot = 0
    for g in range(G):
        blk = K[g * w:(g + 1) * w]
        lb = blk.min(0).values
        ub = blk.max(0).values
        th = torch.topk(lb, 256).values[-1]
        tot += int((ub >= th).sum())
    print(f"G={G}: survivors per group avg {tot / G:.0f}, total evals {tot * w}")
# monotonicity of keys in B
d = K[1:] - K[:-1]
print("frac of (i,B) where key rises with B", (d > 0).double().mean().item())
