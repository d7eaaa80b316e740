"""Quick A/B timing of S1 on the 2^20-request population (config 3 x16): median scan kernel and
whole andes_qoe_eval call (prep + scan + final, CUDA events), INFLIGHT and FINAL, L2 flushed
before each evaluation.  ANDES_LIB_PATH selects another build (one process per build)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

reps = int(os.environ.get("REPS", "15"))
base = W.config3()
if os.environ.get("UNALIGNED") == "1":  # the row path: timelines packed back to back
    base = base.subset(np.arange(base.n), align=1)
big = W.tile(base, int(os.environ.get("TILE", "16")))
ctx = A.Context(max_requests=big.n, max_B=8, max_tokens=big.n_tokens + 64)
req = A.requests_to(big)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
alg = 4 * big.n_tokens + 44 * big.n
peak = 6546.6
tag = os.path.basename(os.environ.get("ANDES_LIB_PATH", "libandes.so"))
s = torch.cuda.Stream()
ctx.profile_enable(True)
for mode, name in ((A.ANDES_EVAL_INFLIGHT, "inflight"), (A.ANDES_EVAL_FINAL, "final")):
    scan, call = [], []
    with torch.cuda.stream(s):
        for it in range(reps + 3):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            ctx.qoe_eval(req, big.n, big.now_us + big.horizon_us, mode, stream=s)
            b.record(s)
            b.synchronize()
            st = ctx.profile_read()
            if it >= 3:
                scan.append(st[1])
                call.append(a.elapsed_time(b))
    # the same call without the profiling events between its kernels
    ctx.profile_enable(False)
    plain = []
    with torch.cuda.stream(s):
        for it in range(reps + 3):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            ctx.qoe_eval(req, big.n, big.now_us + big.horizon_us, mode, stream=s)
            b.record(s)
            b.synchronize()
            if it >= 3:
                plain.append(a.elapsed_time(b))
    ctx.profile_enable(True)
    ts, tc = statistics.median(scan), statistics.median(call)
    tp = statistics.median(plain)
    print(f"[{tag}] {name:8s} scan {ts * 1e3:7.1f} us ({alg / ts / 1e6 / peak:.3f})  call {tc * 1e3:7.1f} us "
          f"({alg / tc / 1e6 / peak:.3f})  unprofiled call {tp * 1e3:7.1f} us ({alg / tp / 1e6 / peak:.3f})", flush=True)
