"""paper_2404_16283_b200 -- B200-native Andes scheduling decision (arXiv 2404.16283).

Thin ctypes binding over ``libandes.so`` (include/andes.h).  Argument marshalling
only: every step of the decision runs in the library's sm_100a kernels.  PyTorch
is used for device memory and streams.  There is no CPU fallback: if the shared
library is missing or no CUDA device is present the calls raise.

Entry points (same names as the C ABI):
    Context.qoe_eval        -> andes_qoe_eval
    Context.gain_estimate   -> andes_gain_estimate
    Context.schedule        -> andes_schedule
    Context.schedule_host   -> andes_schedule_host
    Context.qoe_scenario_mean -> andes_qoe_scenario_mean (config-5 sweeps)
    Context.shard_init      -> andes_shard_init
    Context.schedule_shard  -> andes_schedule_shard (one step); schedule_sharded() runs all steps
                               with a caller-supplied all-gather (torch.distributed / NCCL)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# ANDES_LIB_PATH: load another build of the library (A/B timing of two builds; same ABI)
LIB_PATH = os.environ.get("ANDES_LIB_PATH") or os.path.join(_HERE, "libandes.so")

ANDES_OK = 0
ANDES_NOT_TRIGGERED = 1
ANDES_EVAL_INFLIGHT = 0
ANDES_EVAL_FINAL = 1
ANDES_FORCE = 1
ANDES_PRUNE = 2
ANDES_DEBUG_CHECKS = 4
ANDES_LQSF = 16
ANDES_OBJ_MAXMIN = 32
ANDES_OBJ_PERFECT = 64
ANDES_REFINE = 128
ANDES_F_REFINED = 32
ANDES_F_TRIGGERED = 1
ANDES_F_CAP_HIT = 2
ANDES_F_CAP_OVERRIDDEN = 4
ANDES_F_SLOW_PATH = 8
ANDES_F_TRUNCATED = 16
ANDES_E_INVAL = -1
ANDES_E_RANGE = -2
ANDES_E_CUDA = -3
ANDES_E_CAPACITY = -5
UINT32_MAX = 0xFFFFFFFF
SC_NAMES = ["B_star", "realized", "n_admit", "n_preempt", "B_lo", "B_hi", "flags", "k_star"]

EXPORTS = ["andes_create", "andes_destroy", "andes_last_error", "andes_qoe_eval", "andes_gain_estimate",
           "andes_schedule", "andes_schedule_host", "andes_version", "andes_profile_enable", "andes_profile_read",
           "andes_shard_init", "andes_schedule_shard", "andes_qoe_scenario_mean", "andes_knapsack_dp",
           "andes_knapsack_dp_workspace", "andes_tracker_append", "andes_tracker_append_dev", "andes_simulate",
           "andes_sim_workspace", "andes_comm_create", "andes_comm_connect", "andes_comm_allgather",
           "andes_comm_destroy"]
SHARD_ROUNDS = 4
SHARD_STEPS = 5
MAX_WORLD = 8
N_STAGES = 6
STAGES = ["prep", "scan", "state", "cand", "select", "unused"]


class AndesError(RuntimeError):
    def __init__(self, msg, rc=None):
        super().__init__(msg)
        self.rc = rc


class Limits(C.Structure):
    _fields_ = [("max_requests", C.c_uint32), ("max_B", C.c_uint32), ("max_tokens", C.c_uint64),
                ("max_running", C.c_uint32), ("device", C.c_int32)]


class Requests(C.Structure):
    _fields_ = [("n", C.c_uint32), ("arrival_us", C.c_void_p), ("ttft_us", C.c_void_p),
                ("period_us", C.c_void_p), ("ctx_len", C.c_void_p), ("n_deliv", C.c_void_p),
                ("max_total", C.c_void_p), ("start_off_us", C.c_void_p), ("rank", C.c_void_p),
                ("running", C.c_void_p), ("tl_base", C.c_void_p), ("tl_pool", C.c_void_p),
                ("tl_len", C.c_uint64)]


class SchedParams(C.Structure):
    _fields_ = [("now_us", C.c_int64), ("horizon_us", C.c_uint32), ("B_cap", C.c_uint32),
                ("tau_us", C.c_void_p), ("kv_capacity", C.c_uint64), ("preempt_cap", C.c_uint32),
                ("cur_latency_us", C.c_uint32), ("flags", C.c_uint32), ("prefill_tok_s", C.c_uint32),
                ("swap_tok_s", C.c_uint32), ("now_dev", C.c_void_p)]


class DecisionPtrs(C.Structure):
    _fields_ = [("serve_mask", C.c_void_p), ("admit_idx", C.c_void_p), ("preempt_idx", C.c_void_p),
                ("scalars", C.c_void_p), ("V", C.c_void_p), ("kstar", C.c_void_p),
                ("export_host", C.c_void_p), ("export_preempt", C.c_uint32), ("export_served", C.c_uint32)]


class Shard(C.Structure):
    _fields_ = [("world", C.c_uint32), ("rank", C.c_uint32), ("B_cap", C.c_uint32), ("pad", C.c_uint32),
                ("xbytes", C.c_uint64 * SHARD_ROUNDS)]


class Tracker(C.Structure):
    _fields_ = [("n", C.c_uint32), ("arrival_us", C.c_void_p), ("tl_base", C.c_void_p), ("tl_pool", C.c_void_p),
                ("tl_len", C.c_uint64), ("n_deliv", C.c_void_p), ("ctx_len", C.c_void_p), ("running", C.c_void_p)]


class Sim(C.Structure):
    _fields_ = [("n", C.c_uint32), ("arrival_us", C.c_void_p), ("ttft_us", C.c_void_p), ("period_us", C.c_void_p),
                ("prompt_len", C.c_void_p), ("output_len", C.c_void_p), ("tl_base", C.c_void_p),
                ("tl_pool", C.c_void_p), ("tl_len", C.c_uint64), ("n_deliv", C.c_void_p), ("served", C.c_void_p),
                ("workspace", C.c_void_p)]


class SimParams(C.Structure):
    _fields_ = [("tau_us", C.c_void_p), ("B_cap", C.c_uint32), ("kv_capacity", C.c_uint64), ("horizon_us", C.c_uint32),
                ("preempt_cap", C.c_uint32), ("flags", C.c_uint32), ("max_iters", C.c_uint32)]


class SimStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("start_us", C.c_int64), ("end_us", C.c_int64), ("finished", C.c_uint32),
                ("pad", C.c_uint32)]


class QoeOut(C.Structure):
    _fields_ = [("q", C.c_void_p), ("q64", C.c_void_p), ("s_delay", C.c_void_p), ("s_whole", C.c_void_p),
                ("m", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libandes.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with `python paper_2404_16283_b200/build.py` "
                              "(or __graft_entry__.build()). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        L.andes_create.argtypes = [C.POINTER(C.c_void_p), C.POINTER(Limits)]
        L.andes_destroy.argtypes = [C.c_void_p]
        L.andes_last_error.argtypes = [C.c_void_p]
        L.andes_last_error.restype = C.c_char_p
        L.andes_version.restype = C.c_char_p
        L.andes_qoe_eval.argtypes = [C.c_void_p, C.POINTER(Requests), C.c_int64, C.c_uint32, C.POINTER(QoeOut),
                                     C.c_void_p]
        L.andes_gain_estimate.argtypes = [C.c_void_p, C.POINTER(Requests), C.c_int64, C.c_uint32, C.c_void_p,
                                          C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p]
        L.andes_schedule.argtypes = [C.c_void_p, C.POINTER(Requests), C.POINTER(SchedParams),
                                     C.POINTER(DecisionPtrs), C.c_void_p]
        L.andes_profile_enable.argtypes = [C.c_void_p, C.c_int]
        L.andes_profile_read.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
        L.andes_schedule_host.argtypes = [C.c_void_p, C.POINTER(Requests), C.POINTER(SchedParams),
                                          C.POINTER(DecisionPtrs), C.c_void_p]
        L.andes_qoe_scenario_mean.argtypes = [C.c_void_p, C.POINTER(Requests), C.c_void_p, C.c_uint32,
                                              C.c_void_p, C.c_void_p, C.c_void_p]
        L.andes_knapsack_dp_workspace.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.andes_knapsack_dp_workspace.restype = C.c_uint64
        L.andes_knapsack_dp.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64,
                                        C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.andes_tracker_append.argtypes = [C.c_void_p, C.POINTER(Tracker), C.c_void_p, C.c_void_p, C.c_uint32,
                                           C.c_void_p, C.c_void_p]
        L.andes_tracker_append_dev.argtypes = [C.c_void_p, C.POINTER(Tracker), C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_uint32, C.c_void_p, C.c_void_p]
        L.andes_comm_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        L.andes_comm_connect.argtypes = [C.c_void_p, C.c_void_p]
        L.andes_comm_allgather.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
        L.andes_comm_destroy.argtypes = [C.c_void_p]
        L.andes_sim_workspace.argtypes = [C.c_uint32]
        L.andes_sim_workspace.restype = C.c_uint64
        L.andes_simulate.argtypes = [C.c_void_p, C.POINTER(Sim), C.POINTER(SimParams), C.POINTER(SimStats), C.c_void_p]
        L.andes_shard_init.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(Shard)]
        L.andes_schedule_shard.argtypes = [C.c_void_p, C.POINTER(Shard), C.c_uint32, C.POINTER(Requests),
                                           C.POINTER(SchedParams), C.POINTER(DecisionPtrs), C.c_void_p, C.c_void_p,
                                           C.c_void_p]
        _lib = L
    return _lib


def version() -> str:
    return lib().andes_version().decode()


_FIELDS = [("arrival_us", "int64"), ("ttft_us", "int32"), ("period_us", "int32"), ("ctx_len", "int32"),
           ("n_deliv", "int32"), ("max_total", "int32"), ("start_off_us", "int32"), ("rank", "int32"),
           ("running", "uint8"), ("tl_base", "int64"), ("tl_pool", "int32")]


def _torch():
    import torch
    return torch


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream_ptr(stream):
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def requests_to(src, device="cuda", pin=False):
    """Copy a structure-of-arrays request table (attributes or dict of numpy arrays with the
    AndesRequests field names) into torch tensors on `device` (u32 fields are carried as
    int32 bit patterns, u64 as int64).  pin=True gives pinned host tensors instead."""
    import numpy as np
    torch = _torch()
    out = {}
    for name, dt in _FIELDS:
        a = src[name] if isinstance(src, dict) else getattr(src, name)
        if a is None:
            out[name] = None
            continue
        a = np.ascontiguousarray(a)
        view = {"int64": np.int64, "int32": np.int32, "uint8": np.uint8}[dt]
        t = torch.from_numpy(a.view(view) if a.dtype.itemsize == np.dtype(view).itemsize else a.astype(view))
        if name == "tl_pool" and t.numel() == 0:
            t = torch.zeros(4, dtype=torch.int32)
        if pin:
            out[name] = t.pin_memory()
        else:
            out[name] = t.to(device)
    return out


def _req_struct(t: dict, n: int) -> Requests:
    return Requests(n, *[_ptr(t[name]) for name, _ in _FIELDS], int(t["tl_pool"].numel()) if t["tl_pool"] is not None else 0)


@dataclass
class Decision:
    serve_mask: object
    admit: object
    preempt: object
    scalars: object
    V: object
    kstar: object

    def scalar(self, name):
        return int(self.scalars[SC_NAMES.index(name)])


def decision_export_bytes(B_cap, export_preempt, export_served=0):
    """Size of an AndesDecision.export_host buffer (include/andes.h), completion word included."""
    return _export_done_offset(B_cap, export_preempt, export_served) + 8


def _export_done_offset(B_cap, export_preempt, export_served):
    return (32 + 12 * int(B_cap) + 4 * int(export_preempt) + 4 * int(export_served) + 7) // 8 * 8


def decision_export_done(buf, B_cap, export_preempt, export_served=0):
    """numpy view (u64[1]) of the export's completion word: clear it before the call, poll it
    instead of a stream sync."""
    import numpy as np
    o = _export_done_offset(B_cap, export_preempt, export_served)
    return buf.numpy()[o:o + 8].view(np.uint64)


def decision_export_views(buf, B_cap, export_preempt, export_served=0):
    """numpy views (scalars u32[8], V i64[B_cap], admit i32[B_cap], preempt i32[export_preempt],
    served i32[export_served]) of a pinned export buffer (torch uint8 tensor)."""
    import numpy as np
    a = buf.numpy()
    o = 32 + 12 * B_cap + 4 * export_preempt
    return (a[0:32].view(np.uint32), a[32:32 + 8 * B_cap].view(np.int64),
            a[32 + 8 * B_cap:32 + 12 * B_cap].view(np.int32), a[32 + 12 * B_cap:o].view(np.int32),
            a[o:o + 4 * export_served].view(np.int32))


class Context:
    """An andes_create context (device workspace sized by the limits)."""

    def __init__(self, max_requests, max_B=256, max_tokens=1 << 24, max_running=4096, device=0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise AndesError("no CUDA device: the Andes decision path runs only on the GPU (no CPU fallback)")
        self._h = C.c_void_p()
        lim = Limits(int(max_requests), int(max_B), int(max_tokens), int(max_running), int(device))
        rc = lib().andes_create(C.byref(self._h), C.byref(lim))
        if rc != 0:
            raise AndesError(f"andes_create failed rc={rc}")
        self.device = torch.device("cuda", device)
        self.limits = lim

    def close(self):
        if self._h:
            lib().andes_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc < 0:
            raise AndesError(f"{what} failed rc={rc}: {lib().andes_last_error(self._h).decode()}", rc)
        return rc

    # -- profiling hooks
    def profile_enable(self, on=True):
        self._check(lib().andes_profile_enable(self._h, int(bool(on))), "andes_profile_enable")

    def profile_read(self):
        buf = (C.c_float * N_STAGES)()
        self._check(lib().andes_profile_read(self._h, buf), "andes_profile_read")
        return list(buf)

    # -- andes_qoe_eval
    _QOE_OUTPUTS = ("q", "q64", "s_delay", "s_whole", "m")

    def qoe_eval(self, req: dict, n: int, eval_time_us: int, mode=ANDES_EVAL_INFLIGHT, stream=None, outputs=None):
        """(q f32, q64 f64, s_delay i64, s_whole i64, m i32) per request; `outputs` (a subset of
        _QOE_OUTPUTS, default all) selects which the call writes -- the others are NULL in
        AndesQoeOut and come back as None."""
        torch = _torch()
        dev = self.device
        want = set(self._QOE_OUTPUTS if outputs is None else outputs)
        if not want <= set(self._QOE_OUTPUTS):
            raise ValueError(f"unknown qoe_eval outputs {sorted(want - set(self._QOE_OUTPUTS))}")
        dt = {"q": torch.float32, "q64": torch.float64, "s_delay": torch.int64, "s_whole": torch.int64, "m": torch.int32}
        t = {k: (torch.empty(n, dtype=dt[k], device=dev) if k in want else None) for k in self._QOE_OUTPUTS}
        q, q64, sd, sw, m = (t[k] for k in self._QOE_OUTPUTS)
        out = QoeOut(*[(_ptr(x) if x is not None else None) for x in (q, q64, sd, sw, m)])
        self._check(lib().andes_qoe_eval(self._h, C.byref(_req_struct(req, n)), int(eval_time_us), int(mode),
                                         C.byref(out), _stream_ptr(stream)), "andes_qoe_eval")
        return q, q64, sd, sw, m

    # -- andes_qoe_scenario_mean
    def qoe_scenario_mean(self, req: dict, n: int, scen_off, stream=None):
        """scen_off: device int32 tensor [S+1] of request offsets; returns (mean f64[S], count i32[S])."""
        torch = _torch()
        S = int(scen_off.numel()) - 1
        mean = torch.empty(max(S, 1), dtype=torch.float64, device=self.device)
        cnt = torch.empty(max(S, 1), dtype=torch.int32, device=self.device)
        self._check(lib().andes_qoe_scenario_mean(self._h, C.byref(_req_struct(req, n)), _ptr(scen_off), S,
                                                  _ptr(mean), _ptr(cnt), _stream_ptr(stream)),
                    "andes_qoe_scenario_mean")
        return mean[:S], cnt[:S]

    # -- andes_knapsack_dp (Algorithm 2, exact reference for small instances)
    def knapsack_dp(self, value, weight, B: int, M: int, stream=None):
        """value: device int64 [n], weight: device int32 [n] -> (x u8 [n], best int, Vb int64 [B+1])."""
        torch = _torch()
        n = int(value.numel())
        nb = int(lib().andes_knapsack_dp_workspace(n, int(B), int(M)))
        ws = torch.empty(max(nb, 8), dtype=torch.uint8, device=self.device)
        x = torch.empty(max(n, 1), dtype=torch.uint8, device=self.device)
        best = torch.empty(1, dtype=torch.int64, device=self.device)
        Vb = torch.empty(int(B) + 1, dtype=torch.int64, device=self.device)
        self._check(lib().andes_knapsack_dp(self._h, _ptr(value), _ptr(weight), n, int(B), int(M), _ptr(ws), nb,
                                            _ptr(x), _ptr(best), _ptr(Vb), _stream_ptr(stream)), "andes_knapsack_dp")
        return x[:n], best, Vb

    # -- andes_gain_estimate
    def gain_estimate(self, req: dict, n: int, now_us: int, horizon_us: int, tau, B_list, stream=None):
        torch = _torch()
        import numpy as np
        Bl = np.ascontiguousarray(B_list, dtype=np.uint32)
        gain = torch.empty((Bl.size, n), dtype=torch.float64, device=self.device)
        key = torch.empty((Bl.size, n), dtype=torch.float32, device=self.device)
        qw = torch.empty(n, dtype=torch.float64, device=self.device)
        self._check(lib().andes_gain_estimate(self._h, C.byref(_req_struct(req, n)), int(now_us), int(horizon_us),
                                              _ptr(tau), int(tau.numel()), Bl.ctypes.data, int(Bl.size),
                                              _ptr(gain), _ptr(key), _ptr(qw), _stream_ptr(stream)),
                    "andes_gain_estimate")
        return gain, key, qw

    # -- andes_schedule
    def alloc_decision(self, n, B_cap, pin=False, packed=False):
        """packed: every output a view of ONE device buffer (.packed, uint8), laid out as scalars,
        V, admit, kstar, preempt, serve_mask, so that the decision's head (up to the first pmax
        preempt slots: packed_head(pmax) bytes) leaves the device in one copy."""
        torch = _torch()
        if packed:
            n1 = max(n, 1)
            sizes = [32, 8 * B_cap, 4 * B_cap, 4 * B_cap, 4 * n1, n1]
            offs = [0]
            for z in sizes[:-1]:
                offs.append(offs[-1] + (z + 15) // 16 * 16)
            buf = torch.zeros(offs[-1] + sizes[-1], dtype=torch.uint8, device=self.device)

            def view(k, dt, cnt):
                return buf[offs[k]:offs[k] + sizes[k]].view(dt)[:cnt]
            d = Decision(scalars=view(0, torch.int32, 8), V=view(1, torch.int64, B_cap),
                         admit=view(2, torch.int32, B_cap), kstar=view(3, torch.int32, B_cap),
                         preempt=view(4, torch.int32, n1), serve_mask=view(5, torch.uint8, n1))
            d.packed = buf
            d.packed_offsets = offs
            return d
        kw = dict(pin_memory=True) if pin else dict(device=self.device)
        return Decision(serve_mask=torch.empty(max(n, 1), dtype=torch.uint8, **kw),
                        admit=torch.empty(B_cap, dtype=torch.int32, **kw),
                        preempt=torch.empty(max(n, 1), dtype=torch.int32, **kw),
                        scalars=torch.empty(8, dtype=torch.int32, **kw),
                        V=torch.empty(B_cap, dtype=torch.int64, **kw),
                        kstar=torch.empty(B_cap, dtype=torch.int32, **kw))

    def schedule(self, req: dict, n: int, now_us: int, horizon_us: int, tau, kv_capacity: int,
                 preempt_cap=UINT32_MAX, cur_latency_us=0, flags=ANDES_FORCE, out: Decision | None = None,
                 stream=None, prefill_tok_s=5000, swap_tok_s=0, now_dev=None, export_host=None,
                 export_preempt=0, export_served=0) -> Decision:
        """now_dev: optional int64 [1] in device or pinned host memory; when given the decision time
        is read from it when the call runs (now_us is only the reference the kernels' time arguments
        are shifted from), so a captured graph of the call can be replayed at new times.
        export_host: optional pinned host uint8 tensor (decision_export_bytes(B_cap, export_preempt,
        export_served) bytes) that the call fills zero-copy with scalars, V, admit, the first
        export_preempt preempt entries and the next batch (decision_export_views splits it)."""
        B_cap = int(tau.numel())
        out = out or self.alloc_decision(n, B_cap)
        p = SchedParams(int(now_us), int(horizon_us), B_cap, _ptr(tau), int(kv_capacity), int(preempt_cap),
                        int(cur_latency_us), int(flags), int(prefill_tok_s), int(swap_tok_s), _ptr(now_dev))
        d = DecisionPtrs(_ptr(out.serve_mask), _ptr(out.admit), _ptr(out.preempt), _ptr(out.scalars),
                         _ptr(out.V), _ptr(out.kstar), _ptr(export_host), int(export_preempt), int(export_served))
        self._check(lib().andes_schedule(self._h, C.byref(_req_struct(req, n)), C.byref(p), C.byref(d),
                                         _stream_ptr(stream)), "andes_schedule")
        return out

    # -- andes_schedule_host (host buffers; copies inside the call; synchronous)
    def schedule_host(self, req_host: dict, n: int, now_us: int, horizon_us: int, tau_host, kv_capacity: int,
                      preempt_cap=UINT32_MAX, cur_latency_us=0, flags=ANDES_FORCE, out: Decision | None = None,
                      stream=None):
        B_cap = int(tau_host.numel())
        out = out or self.alloc_decision(n, B_cap, pin=True)
        p = SchedParams(int(now_us), int(horizon_us), B_cap, _ptr(tau_host), int(kv_capacity), int(preempt_cap),
                        int(cur_latency_us), int(flags), 5000, 0)
        d = DecisionPtrs(_ptr(out.serve_mask), _ptr(out.admit), _ptr(out.preempt), _ptr(out.scalars),
                         _ptr(out.V), _ptr(out.kstar))
        rc = self._check(lib().andes_schedule_host(self._h, C.byref(_req_struct(req_host, n)), C.byref(p),
                                                   C.byref(d), _stream_ptr(stream)), "andes_schedule_host")
        return out, rc

    # -- andes_tracker_append (device-resident Request Tracker update between decisions)
    def tracker_append(self, req: dict, n: int, idx, t_abs, serve_mask=None, stream=None):
        """req: the device request tensors (updated in place: tl_pool, n_deliv, ctx_len, running);
        idx: device int32 [count] request index of each delivered token (a request's tokens
        consecutive, in time order); t_abs: device int64 [count] absolute delivery times;
        serve_mask: device uint8 [n] (optional) -> the new running set."""
        t = Tracker(int(n), _ptr(req["arrival_us"]), _ptr(req["tl_base"]), _ptr(req["tl_pool"]),
                    int(req["tl_pool"].numel()), _ptr(req["n_deliv"]), _ptr(req["ctx_len"]), _ptr(req["running"]))
        count = int(idx.numel()) if idx is not None else 0
        self._check(lib().andes_tracker_append(self._h, C.byref(t), _ptr(idx), _ptr(t_abs), count, _ptr(serve_mask),
                                               _stream_ptr(stream)), "andes_tracker_append")

    def tracker_append_dev(self, req: dict, n: int, idx, t_abs, count_dev, serve_mask=None, stream=None):
        """As tracker_append with the token count read on the device: count_dev is a device
        int32 [1] (<= idx.numel(), the slots idx / t_abs hold), so the call is graph-capturable."""
        t = Tracker(int(n), _ptr(req["arrival_us"]), _ptr(req["tl_base"]), _ptr(req["tl_pool"]),
                    int(req["tl_pool"].numel()), _ptr(req["n_deliv"]), _ptr(req["ctx_len"]), _ptr(req["running"]))
        self._check(lib().andes_tracker_append_dev(self._h, C.byref(t), _ptr(idx), _ptr(t_abs), _ptr(count_dev),
                                                   int(idx.numel()), _ptr(serve_mask), _stream_ptr(stream)),
                    "andes_tracker_append_dev")

    # -- andes_simulate (NEXT-3: the serving loop on the device, the decision in the loop)
    def simulate(self, trace: dict, tau, kv_capacity: int, horizon_us=2_000_000, preempt_cap=UINT32_MAX, flags=0,
                 max_iters=0, stream=None):
        """trace: dict with n and numpy arrays arrival_us, ttft_us, period_us, prompt_len, output_len,
        tl_base, and tl_len (workloads.sim_trace).  Returns (n_deliv i32[n], tl_pool i32[tl_len],
        trace tensors dict, stats dict); everything stays on the device."""
        torch = _torch()
        import numpy as np
        dev = self.device
        n = int(trace["n"])
        t = {k: torch.from_numpy(np.ascontiguousarray(trace[k]).view(
            {8: np.int64, 4: np.int32}[np.asarray(trace[k]).dtype.itemsize])).to(dev)
             for k in ("arrival_us", "ttft_us", "period_us", "prompt_len", "output_len", "tl_base")}
        tl_len = int(trace["tl_len"])
        pool = torch.zeros(max(tl_len, 4), dtype=torch.int32, device=dev)
        g = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        served = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
        ws = torch.empty(int(lib().andes_sim_workspace(n)) + 16, dtype=torch.uint8, device=dev)
        sim = Sim(n, _ptr(t["arrival_us"]), _ptr(t["ttft_us"]), _ptr(t["period_us"]), _ptr(t["prompt_len"]),
                  _ptr(t["output_len"]), _ptr(t["tl_base"]), _ptr(pool), tl_len, _ptr(g), _ptr(served), _ptr(ws))
        p = SimParams(_ptr(tau), int(tau.numel()), int(kv_capacity), int(horizon_us), int(preempt_cap), int(flags),
                      int(max_iters))
        st = SimStats()
        self._check(lib().andes_simulate(self._h, C.byref(sim), C.byref(p), C.byref(st), _stream_ptr(stream)),
                    "andes_simulate")
        t["tl_pool"] = pool
        t["n_deliv"] = g
        return g[:n], pool, t, {"iterations": int(st.iterations), "start_us": int(st.start_us),
                                 "end_us": int(st.end_us), "finished": int(st.finished)}

    # -- multi-GPU decision (andes_shard_init / andes_schedule_shard)
    def shard_init(self, world: int, rank: int, B_cap: int) -> Shard:
        sh = Shard()
        self._check(lib().andes_shard_init(self._h, int(world), int(rank), int(B_cap), C.byref(sh)),
                    "andes_shard_init")
        return sh

    def alloc_shard_buffers(self, sh: Shard):
        """Device send blocks (one per round) and recv buffers (world blocks each)."""
        torch = _torch()
        send = [torch.empty(int(sh.xbytes[k]), dtype=torch.uint8, device=self.device) for k in range(SHARD_ROUNDS)]
        recv = [torch.empty(int(sh.world) * int(sh.xbytes[k]), dtype=torch.uint8, device=self.device)
                for k in range(SHARD_ROUNDS)]
        return send, recv

    def schedule_shard(self, sh: Shard, step: int, req: dict, n: int, now_us: int, horizon_us: int, tau,
                       kv_capacity: int, out: Decision, recv=None, send=None, preempt_cap=UINT32_MAX,
                       cur_latency_us=0, flags=ANDES_FORCE, stream=None):
        p = SchedParams(int(now_us), int(horizon_us), int(tau.numel()), _ptr(tau), int(kv_capacity),
                        int(preempt_cap), int(cur_latency_us), int(flags), 5000, 0)
        d = DecisionPtrs(_ptr(out.serve_mask), _ptr(out.admit), _ptr(out.preempt), _ptr(out.scalars),
                         _ptr(out.V), _ptr(out.kstar))
        self._check(lib().andes_schedule_shard(self._h, C.byref(sh), int(step), C.byref(_req_struct(req, n)),
                                               C.byref(p), C.byref(d), _ptr(recv), _ptr(send),
                                               _stream_ptr(stream)), "andes_schedule_shard")

    def alloc_shard_decision(self, n, B_cap):
        """Decision buffers of a sharded call: preempt_idx holds the global victim list."""
        torch = _torch()
        d = self.alloc_decision(n, B_cap)
        d.preempt = torch.empty(4096, dtype=torch.int32, device=self.device)
        return d


def torch_allgather(group=None):
    """allgather(send, recv) over torch.distributed: every rank's send block, in rank order, into
    recv (NCCL on GPUs; also works with gloo on CPU tensors)."""
    import torch.distributed as dist

    def ag(send, recv):
        try:
            dist.all_gather_into_tensor(recv, send, group=group)
        except (RuntimeError, NotImplementedError, AttributeError):
            dist.all_gather(list(recv.chunk(dist.get_world_size(group))), send, group=group)
    return ag


def run_shard_steps(step_fn, allgather, send, recv, steps=SHARD_STEPS):
    """Host orchestration of a sharded decision: step s runs on this rank (step_fn(s, recv_prev,
    send_s)); after every step but the last, this rank's send block is all-gathered in rank order
    into recv[s] (allgather(send_s, recv_s), e.g. torch.distributed.all_gather_into_tensor).
    Argument marshalling only: every step's arithmetic runs in the library's kernels."""
    prev = None
    for s in range(steps):
        cur = send[s] if s < len(send) else None
        step_fn(s, prev, cur)
        if cur is not None:
            allgather(cur, recv[s])
            prev = recv[s]
    return prev


class Comm:
    """The peer-memory all-gather (andes_comm_*): create on every rank, exchange .handle over any
    host channel, connect(handles in rank order); allgather(send, recv) is a device collective."""

    def __init__(self, world: int, rank: int, max_block: int, device: int = 0):
        self._h = C.c_void_p()
        h = (C.c_char * 64)()
        rc = lib().andes_comm_create(C.byref(self._h), int(device), int(world), int(rank), int(max_block), h)
        if rc < 0:
            raise AndesError(f"andes_comm_create failed rc={rc}", rc)
        self.handle = bytes(h)
        self.world = world

    def connect(self, handles):
        buf = C.create_string_buffer(b"".join(handles), 64 * self.world)
        rc = lib().andes_comm_connect(self._h, buf)
        if rc < 0:
            raise AndesError(f"andes_comm_connect failed rc={rc}", rc)

    def allgather(self, send, recv, stream=None):
        rc = lib().andes_comm_allgather(self._h, _ptr(send), _ptr(recv), int(send.numel() * send.element_size()),
                                        _stream_ptr(stream))
        if rc < 0:
            raise AndesError(f"andes_comm_allgather failed rc={rc}", rc)

    def close(self):
        if self._h:
            lib().andes_comm_destroy(self._h)
            self._h = C.c_void_p()


def schedule_sharded(ctx: Context, sh: Shard, req: dict, n: int, now_us: int, horizon_us: int, tau,
                     kv_capacity: int, allgather, out: Decision | None = None, bufs=None, preempt_cap=UINT32_MAX,
                     cur_latency_us=0, flags=ANDES_FORCE, stream=None) -> Decision:
    """One sharded decision on this rank.  allgather(send, recv) must gather every rank's send
    block in rank order into recv on `stream` (torch.distributed.all_gather_into_tensor)."""
    out = out or ctx.alloc_shard_decision(n, int(tau.numel()))
    send, recv = bufs or ctx.alloc_shard_buffers(sh)

    def step(s, prev, cur):
        ctx.schedule_shard(sh, s, req, n, now_us, horizon_us, tau, kv_capacity, out, recv=prev, send=cur,
                           preempt_cap=preempt_cap, cur_latency_us=cur_latency_us, flags=flags, stream=stream)

    run_shard_steps(step, allgather, send, recv)
    return out
