"""ncu driver: three 1M-request QoE evaluations (the bench's S1 throughput run), INFLIGHT mode.
Usage under ncu: -k regex:k_qoe_scan -s 2 -c 1 (the third launch, warm code, cold data)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_16283_b200 as A  # noqa: E402
import workloads as W  # noqa: E402
from bench import _tile  # noqa: E402

snap = W.config3()
big = _tile(snap, int(os.environ.get("REPS", "16")))
q = A.Context(max_requests=big.n, max_B=8, max_tokens=big.n_tokens + 64)
breq = A.requests_to(big)
mode = A.ANDES_EVAL_FINAL if os.environ.get("FINAL") == "1" else A.ANDES_EVAL_INFLIGHT
for _ in range(3):
    q.qoe_eval(breq, big.n, big.now_us + big.horizon_us, mode)
torch.cuda.synchronize()
print("done", big.n, big.n_tokens)
