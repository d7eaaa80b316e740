"""S1 scan throughput vs population size (config 3 tiled x1..x64), L2 flushed before each
evaluation; bytes = the algorithmic 4 B per token + 44 B per request."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402

base = W.config3()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
peak = 6539.9
for reps in (1, 4, 16, 64):
    big = W.tile(base, reps) if reps > 1 else base
    ctx = A.Context(max_requests=big.n, max_B=8, max_tokens=big.n_tokens + 64)
    req = A.requests_to(big)
    ms = []
    for it in range(6):
        flush.zero_()
        ctx.profile_enable(True)
        ctx.qoe_eval(req, big.n, big.now_us + big.horizon_us, A.ANDES_EVAL_INFLIGHT)
        torch.cuda.synchronize()
        st = ctx.profile_read()
        ctx.profile_enable(False)
        if it >= 2:
            ms.append(st[1])
    t = float(np.median(ms))
    alg = 4 * int(big.n_deliv.astype(np.int64).sum()) + 44 * big.n
    print(f"requests {big.n:>9d} tokens {big.n_tokens:>11d} scan {t * 1e3:8.1f} us  {alg / (t * 1e-3) / 1e9:7.1f} GB/s"
          f"  frac {alg / (t * 1e-3) / 1e9 / peak:.3f}")
    del ctx, req, big
    torch.cuda.empty_cache()
