"""Internal timeline of one config-3 decision from %globaltimer stamps (andes_debug_trace)."""
import ctypes as C
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
L = A.lib()
L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
L.andes_debug_trace.argtypes = [C.c_void_p, C.c_int]
print("trace rc", L.andes_debug_trace(ctx._h, 1))
for it in range(4):
    d = ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16)
torch.cuda.synchronize()
tr = np.zeros(8192, np.uint64)
print("read rc", L.andes_debug_read(ctx._h, 7, tr.ctypes.data, tr.nbytes))
g = np.zeros(26, np.uint32)
print("read rc", L.andes_debug_read(ctx._h, 5, g.ctypes.data, 104), g.tolist())
sel = tr[:512].astype(np.int64).reshape(256, 2)
t0 = sel[:, 0][sel[:, 0] > 0].min()
st = tr[3000:4024].astype(np.int64).reshape(512, 2)
st = st[st[:, 0] > 0]
print("state CTAs: first start", (st[:, 0].min() - t0) / 1e3, "last end", (st[:, 1].max() - t0) / 1e3, "us rel. select start")
print("state last-block", [(int(tr[s]) - t0) / 1e3 for s in (2200, 2201)])
print("select CTA start spread us", (sel[:, 0].max() - t0) / 1e3, "end min/med/max",
      [(x - t0) / 1e3 for x in (sel[:, 1].min(), int(np.median(sel[:, 1])), sel[:, 1].max())])
print("finalize phases us", [round((int(tr[s]) - t0) / 1e3, 2) for s in range(2100, 2106)])
