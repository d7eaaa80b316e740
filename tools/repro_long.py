"""Repro: one 100,003-token request spanning many scan tiles (look-back + direct carry)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

rng = np.random.default_rng(99)
P, ttft, g = 1000, 5000, 100_003
d = ttft + np.arange(g, dtype=np.int64) * P + np.where(np.arange(g) > 50_000, 7_777, 0)
d = np.maximum.accumulate(d + rng.integers(-900, 900, g)).astype(np.uint32)
tl = [np.zeros(0, np.uint32), d, np.array([12], np.uint32), np.zeros(0, np.uint32)]
gg, base, pool = W._pack(tl)
n = 4
big = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, ttft, np.uint32),
                 period_us=np.full(n, P, np.uint32), ctx_len=np.ones(n, np.uint32), n_deliv=gg,
                 max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                 rank=np.arange(n, dtype=np.uint32), running=np.zeros(n, np.uint8), tl_base=base,
                 tl_pool=pool, now_us=int(d[-1]) + 10, horizon_us=2_000_000)
ctx = A.Context(max_requests=16, max_B=8, max_tokens=1 << 18)
req = A.requests_to(big)
for ev in (big.now_us + 3_000_000, big.now_us - 40_000_000):
    for final in (0, 1):
        q, q64, sd, sw, m = ctx.qoe_eval(req, n, ev, final)
        torch.cuda.synchronize()
        oq, osd, osw, om = oracle.qoe_eval(big, ev, final=bool(final))
        print(ev, final, "gpu", sd.cpu().numpy().tolist(), "orc", osd.tolist(), "m", m.cpu().numpy().tolist(), om.tolist())

# ---- debug: tile status words after the failing evaluation
import ctypes as C  # noqa: E402
L = A.lib()
L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
ev = big.now_us - 40_000_000
for rep in range(3):
    q, q64, sd, sw, m = ctx.qoe_eval(req, n, ev, 0)
    torch.cuda.synchronize()
    st = np.zeros(16, np.uint64)
    L.andes_debug_read(ctx._h, 0, st.ctypes.data, st.nbytes)
    print("status", [(int(x) >> 62, (int(x) >> 32) & 1, int(x) & 0xffffffff) for x in st[:14]])
    print("sd", sd.cpu().numpy().tolist())
# expected per-tile prefix maxima of lat+ for request 1 (tokens k < 60011)
t = ev - 0
mlim = 60011
k = np.arange(mlim, dtype=np.int64)
I = ttft + k * P
lat = np.maximum(d[:mlim].astype(np.int64) - I, 0)
pref = np.maximum.accumulate(lat)
print("expected inclusive prefix at tile ends", [int(pref[min((j + 1) * 8192, mlim) - 1]) for j in range(8)])
