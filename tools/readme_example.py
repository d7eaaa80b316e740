import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np, torch
import paper_2404_16283_b200 as A, workloads as W

snap = W.config3()                                   # a seeded 64K-request snapshot (SoA + timeline pool)
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)                            # device tensors: arrival, ttft, period, ctx_len, ...
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()   # tau(B) for B = 1..256, microseconds
d = ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16)
B_star, realized, n_admit, n_preempt = d.scalars.cpu().numpy().view(np.uint32)[:4]
serve = d.serve_mask[:snap.n]                        # the next batch; d.admit / d.preempt list the changes
q, q64, s_delay, s_whole, m = ctx.qoe_eval(req, snap.n, snap.now_us)   # QoE of every request (Eq. 1-3)

print('B*', B_star, 'realized', realized, 'admit', n_admit, 'preempt', n_preempt, 'served', int(serve.sum()), 'q0', float(q[0]))
