"""Probe: decision globals (theta, survivors, overflow) and per-stage times for config 3."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

snap = W.config3() if len(sys.argv) < 2 else W.config2()
ctx = A.Context(max_requests=snap.n, max_B=256, max_tokens=snap.n_tokens + 64)
req = A.requests_to(snap)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
L = A.lib()
L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
ctx.profile_enable(True)
for it in range(5):
    d = ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16)
    st = ctx.profile_read()
torch.cuda.synchronize()
g = np.zeros(32, np.uint32)
rc = L.andes_debug_read(ctx._h, 5, g.ctypes.data, 96)
print("debug_read rc", rc)
names = ["run_l_lo", "run_l_hi", "pool_end_lo", "pool_end_hi", "ntiles", "inv_minP", "n_run", "done", "B_lo",
         "B_hi", "triggered", "err", "slow", "tile_ctr", "prep_done", "state_done", "tau_lo", "tau_hi", "theta",
         "n_surv", "overflow", "cand_ctr"]
print({k: int(v) for k, v in zip(names, g)})
print("stages ms", dict(zip(A.STAGES, [round(x, 4) for x in st])))
print("scalars", d.scalars.cpu().numpy().tolist())
