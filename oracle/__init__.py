"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liboracle.so`` (built from ``andes_oracle.c``) plus
the exact-rational checker in :mod:`oracle.exact`.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path (``paper_2404_16283_b200``) and never imports it.

The arrays passed in are plain numpy arrays produced by ``workloads`` (the seeded
input generators shared by both sides, which hold none of the method's arithmetic).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "andes_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_FORCE = 1
ORC_PRUNE = 2
ORC_LQSF = 16
ORC_MAXMIN = 32
ORC_PERFECT = 64
ORC_REFINE = 128
ORC_FLAG_REFINED = 32
UINT32_MAX = 0xFFFFFFFF
INT64_MIN = -(1 << 63)


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (IEEE binary64, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-O2", "-std=gnu99", "-pthread", "-ffp-contract=off", "-fno-fast-math",
            "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm", "-lpthread",
        ])
    return _LIB


class _Req(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("arrival_us", C.c_void_p), ("ttft_us", C.c_void_p), ("period_us", C.c_void_p),
        ("ctx_len", C.c_void_p), ("n_deliv", C.c_void_p), ("max_total", C.c_void_p),
        ("start_off_us", C.c_void_p), ("rank", C.c_void_p), ("running", C.c_void_p),
        ("tl_base", C.c_void_p), ("tl_pool", C.c_void_p),
    ]


class _Params(C.Structure):
    _fields_ = [
        ("now_us", C.c_int64), ("horizon_us", C.c_uint32), ("tau_us", C.c_void_p),
        ("B_cap", C.c_uint32), ("kv_capacity", C.c_uint64), ("preempt_cap", C.c_uint32),
        ("cur_latency_us", C.c_uint32), ("flags", C.c_uint32),
        ("prefill_tok_s", C.c_uint32), ("swap_tok_s", C.c_uint32),
    ]


class _Dec(C.Structure):
    _fields_ = [
        ("serve_mask", C.c_void_p), ("admit_idx", C.c_void_p), ("preempt_idx", C.c_void_p),
        ("scalars", C.c_void_p), ("V", C.c_void_p), ("kstar", C.c_void_p),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_qoe_walk.restype = C.c_int
        _lib.oracle_qoe_walk.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.oracle_qoe_eval_mt.restype = C.c_int
        _lib.oracle_qoe_eval_mt.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_int]
        _lib.oracle_gain_estimate_mt.restype = C.c_int
        _lib.oracle_gain_estimate_mt.argtypes = [C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p, C.c_uint32,
                                                 C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                                 C.c_int]
        _lib.oracle_overhead_us.restype = C.c_int
        _lib.oracle_overhead_us.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_void_p, C.c_void_p]
        _lib.oracle_schedule_mt.restype = C.c_int
        _lib.oracle_schedule_mt.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


_REQ_DTYPES = {
    "arrival_us": np.int64, "ttft_us": np.uint32, "period_us": np.uint32, "ctx_len": np.uint32,
    "n_deliv": np.uint32, "max_total": np.uint32, "start_off_us": np.uint32, "rank": np.uint32,
    "running": np.uint8, "tl_base": np.uint64, "tl_pool": np.uint32,
}


def _req_struct(req):
    """req: mapping with the SoA arrays (see workloads.Snapshot)."""
    arrs = {}
    for k, dt in _REQ_DTYPES.items():
        v = getattr(req, k) if not isinstance(req, dict) else req.get(k)
        if v is None:
            arrs[k] = None
            continue
        arrs[k] = np.ascontiguousarray(v, dtype=dt)
    if arrs["tl_pool"] is None or arrs["tl_pool"].size == 0:
        arrs["tl_pool"] = np.zeros(1, np.uint32)
    n = arrs["arrival_us"].shape[0]
    s = _Req(n, *[_p(arrs[k]) for k in ["arrival_us", "ttft_us", "period_us", "ctx_len", "n_deliv",
                                          "max_total", "start_off_us", "rank", "running", "tl_base",
                                          "tl_pool"]])
    return s, arrs


def qoe_walk(D_us, ttft, P, t, m, final=False):
    """O2 on one delivery list. Returns (S_delay, S_whole, Q)."""
    D = np.ascontiguousarray(D_us, dtype=np.uint32)
    sd, sw, q = C.c_int64(), C.c_int64(), C.c_double()
    rc = lib().oracle_qoe_walk(D.ctypes.data if D.size else None, D.size, ttft, P, t, m, int(final),
                               C.byref(sd), C.byref(sw), C.byref(q))
    if rc != 0:
        raise ValueError(f"oracle_qoe_walk rc={rc}")
    return sd.value, sw.value, q.value


def nproc() -> int:
    """Host threads available to this process (the threaded oracle's default)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def qoe_eval(req, eval_time_us, final=False, threads=1):
    """Per-request (Q fp64, S_delay, S_whole, m).  threads > 1 splits the requests over threads."""
    s, keep = _req_struct(req)
    n = s.n
    q = np.zeros(n, np.float64)
    sd = np.zeros(n, np.int64)
    sw = np.zeros(n, np.int64)
    m = np.zeros(n, np.uint32)
    rc = lib().oracle_qoe_eval_mt(C.byref(s), int(eval_time_us), int(final), _p(q), _p(sd), _p(sw), _p(m),
                                  int(threads))
    if rc != 0:
        raise ValueError(f"oracle_qoe_eval rc={rc}")
    return q, sd, sw, m


def gain_estimate(req, now_us, horizon_us, tau_us, B_list, threads=1):
    """gain f64[nB, n], key f32[nB, n], q_wait f64[n] (row b = B_list[b]).  threads > 1 splits
    the requests over threads."""
    s, keep = _req_struct(req)
    tau = np.ascontiguousarray(tau_us, dtype=np.uint32)
    Bl = np.ascontiguousarray(B_list, dtype=np.uint32)
    n = s.n
    gain = np.zeros((Bl.size, n), np.float64)
    key = np.zeros((Bl.size, n), np.float32)
    qw = np.zeros(n, np.float64)
    rc = lib().oracle_gain_estimate_mt(C.byref(s), int(now_us), int(horizon_us), _p(tau), tau.size,
                                       _p(Bl), Bl.size, _p(gain), _p(key), _p(qw), int(threads))
    if rc != 0:
        raise ValueError(f"oracle_gain_estimate rc={rc}")
    return gain, key, qw


def overhead_us(prefill_tok_s, swap_tok_s, l, queued=False):
    """Reading R24's (preempt, resume) cost in us of a request of context l."""
    pre, res = C.c_int64(), C.c_int64()
    lib().oracle_overhead_us(int(prefill_tok_s), int(swap_tok_s), int(l), int(bool(queued)), C.byref(pre),
                             C.byref(res))
    return pre.value, res.value


@dataclass
class Decision:
    status: int
    serve_mask: np.ndarray
    admit: np.ndarray
    preempt: np.ndarray
    B_star: int
    realized: int
    B_lo: int
    B_hi: int
    flags: int
    k_star: int
    V: np.ndarray
    kstar: np.ndarray


def schedule(req, now_us, horizon_us, tau_us, kv_capacity, preempt_cap=UINT32_MAX,
             cur_latency_us=0, flags=ORC_FORCE, B_cap=None, prefill_tok_s=5000, swap_tok_s=0, threads=1):
    """One decision (O6-O9).  threads > 1 splits the independent per-B walks (S3/S4) over
    threads; every output is identical for any thread count."""
    s, keep = _req_struct(req)
    tau = np.ascontiguousarray(tau_us, dtype=np.uint32)
    B_cap = tau.size if B_cap is None else B_cap
    n = s.n
    p = _Params(int(now_us), int(horizon_us), _p(tau), int(B_cap), int(kv_capacity), int(preempt_cap),
                int(cur_latency_us), int(flags), int(prefill_tok_s), int(swap_tok_s))
    mask = np.zeros(max(n, 1), np.uint8)
    adm = np.zeros(max(n, 1), np.uint32)
    pre = np.zeros(max(n, 1), np.uint32)
    sc = np.zeros(8, np.uint32)
    V = np.zeros(max(B_cap, 1), np.int64)
    ks = np.zeros(max(B_cap, 1), np.uint32)
    d = _Dec(_p(mask), _p(adm), _p(pre), _p(sc), _p(V), _p(ks))
    rc = lib().oracle_schedule_mt(C.byref(s), C.byref(p), C.byref(d), int(threads))
    if rc < 0:
        raise ValueError(f"oracle_schedule rc={rc}")
    return Decision(rc, mask[:n].copy(), adm[:sc[2]].copy(), pre[:sc[3]].copy(), int(sc[0]), int(sc[1]),
                    int(sc[4]), int(sc[5]), int(sc[6]), int(sc[7]), V[:B_cap].copy(), ks[:B_cap].copy())
