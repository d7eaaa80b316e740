"""Stage times (profiled events) of one config-3 decision per objective (L2 warm)."""
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
names = ["prep(+obj pre-scan)", "scan", "state", "compact", "select(+refine)", "-"]
for name, fl in (("andes", 0), ("maxmin", A.ANDES_OBJ_MAXMIN), ("perfect", A.ANDES_OBJ_PERFECT)):
    acc = np.zeros(A.N_STAGES)
    for it in range(6):
        ctx.profile_enable(True)
        ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16,
                     flags=A.ANDES_FORCE | fl)
        torch.cuda.synchronize()
        st = np.array(ctx.profile_read())
        ctx.profile_enable(False)
        if it >= 2:
            acc += st
    print(name, {k: round(v * 1e3 / 4, 1) for k, v in zip(names, acc)})
