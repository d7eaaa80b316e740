import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(__file__), "repro_long.py")).read().split("ctx = A.Context")[0])
import paper_2404_16283_b200 as A  # noqa
ctx = A.Context(max_requests=16, max_B=8, max_tokens=1 << 18)
req = A.requests_to(big)
L = A.lib()
L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
evA, evB = big.now_us + 3_000_000, big.now_us - 40_000_000
import oracle  # noqa
okB = oracle.qoe_eval(big, evB)[1]
okA = oracle.qoe_eval(big, evA)[1]
fails = {}
seqs = {"B": [(evB, 0)], "AB": [(evA, 0), (evB, 0)], "FB": [(evA, 1), (evB, 0)], "BF": [(evB, 1), (evB, 0)]}
for name, seq in seqs.items():
    nf = 0
    for it in range(30):
        for ev, fm in seq:
            q, q64, sd, sw, m = ctx.qoe_eval(req, n, ev, fm)
        torch.cuda.synchronize()
        if not np.array_equal(sd.cpu().numpy(), okB):
            nf += 1
            st = np.zeros(16, np.uint64)
            L.andes_debug_read(ctx._h, 0, st.ctypes.data, st.nbytes)
            if nf <= 2:
                print(name, "FAIL status", [(int(x) >> 62, (int(x) >> 32) & 1, int(x) & 0xffffffff) for x in st[:13]])
    print(name, "fails", nf, "/ 30")
if os.environ.get("ANDES_SCAN_DEBUG"):
    for name, seq in seqs.items():
        for it in range(5):
            for ev, fm in seq:
                q, q64, sd, sw, m = ctx.qoe_eval(req, n, ev, fm)
            torch.cuda.synchronize()
            gl = np.zeros(18, np.uint32)
            L.andes_debug_read(ctx._h, 5, gl.ctypes.data, gl.nbytes)
            print(name, "poison words seen after wait (last call):", int(gl[12]), "ok", np.array_equal(sd.cpu().numpy(), okB))
    for it in range(6):
        for ev, fm in seqs["FB"]:
            q, q64, sd, sw, m = ctx.qoe_eval(req, n, ev, fm)
        torch.cuda.synchronize()
        h = np.zeros(8 * 13, np.uint32)
        L.andes_debug_read(ctx._h, 6, h.ctypes.data, h.nbytes)
        ok = np.array_equal(sd.cpu().numpy(), okB)
        print("FB ok", ok, "tiles 0-3 [mode, cmax, agg_v, agg_f, hcnt, hP, httft, hbase]:", h.reshape(13, 8)[:4].tolist())
