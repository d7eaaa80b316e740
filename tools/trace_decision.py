"""Internal timeline of one config-3 decision from %globaltimer stamps (andes_debug_trace).
Tile / first-tile stamps need a -DANDES_SCAN_PHASES build (ANDES_LIB_PATH).
FLUSH=1: a 256 MB write before every replay (the bench's L2-flushed timing).
Slots: 7000+2b prep CTA b start/end; 5000+2b scan CTA b start/end; 2300 bounds end (scan CTA 0);
3000+2b state CTA b; 2200/2201 state last block; 0+2b select CTA b; 2100.. finalize phases."""
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
for it in range(int(os.environ.get("ITERS", "4"))):
    if it == int(os.environ.get("ITERS", "4")) - 1:
        L.andes_debug_trace(ctx._h, 0)
        L.andes_debug_trace(ctx._h, 1)
    d = ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16)
torch.cuda.synchronize()
if os.environ.get("GRAPH", "1") == "1":
    # as the bench times it: the decision captured in a CUDA graph, replayed (stamps of the last replay)
    s = torch.cuda.Stream()
    out = ctx.alloc_decision(snap.n, 256)
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ctx.schedule(req, snap.n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=16, out=out,
                         stream=s)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            if os.environ.get("FLUSH") == "1":  # L2 flushed before each replay, as the bench times it
                flush.zero_()
            g.replay()
    s.synchronize()
tr = np.zeros(1 << 16, np.uint64)
print("read rc", L.andes_debug_read(ctx._h, 7, tr.ctypes.data, tr.nbytes))
tr = tr.astype(np.int64)


def span(lo, hi):
    x = tr[lo:hi].reshape(-1, 2)
    x = x[x[:, 0] > 0]
    return x


pr = span(7000, 8024)
t0 = pr[:, 0].min()
us = lambda v: round((int(v) - t0) / 1e3, 2)  # noqa: E731
print("prep CTAs", len(pr), "start", us(pr[:, 0].min()), "end max", us(pr[:, 1].max()))
sc = span(5000, 7000)
print("scan CTAs", len(sc), "start min/max", us(sc[:, 0].min()), us(sc[:, 0].max()), "bounds end", us(tr[2300]),
      "end min/med/max", us(sc[:, 1].min()), us(np.median(sc[:, 1])), us(sc[:, 1].max()))
st = span(3000, 4024)
if len(st):
    print("state CTAs", len(st), "start", us(st[:, 0].min()), us(st[:, 0].max()), "end min/max", us(st[:, 1].min()),
          us(st[:, 1].max()), "(fused) cut leader start / release", us(tr[2200]), us(tr[2201]))
cp = span(8100, 9124)
if len(cp):
    print("compact CTAs", len(cp), "start", us(cp[:, 0].min()), us(cp[:, 0].max()), "theta(CTA0) / (fused) barrier B",
          us(tr[2210]), "end max", us(cp[:, 1].max()))
print("select CTA255 phases", [us(tr[s]) for s in range(2400, 2409) if tr[s]], "(2400 keys, 2401 rank, 2402-3 l loads, 2406 walk, 2407 V loop, 2408 block sum, 2404 V out, 2405 cap)")
sel = span(0, 512)
print("select CTAs", len(sel), "start", us(sel[:, 0].min()), us(sel[:, 0].max()), "end min/med/max",
      us(sel[:, 1].min()), us(np.median(sel[:, 1])), us(sel[:, 1].max()))
ent = tr[9200:9456]
print("select entry min/med/max", us(ent.min()), us(np.median(ent)), us(ent.max()), "n_surv", int(tr[2410]),
      "late entries (B)", (np.argsort(-ent)[:8] + 1).tolist())
print("finalize phases", [us(tr[s]) for s in range(2100, 2106) if tr[s]])

tl = tr[16384:16384 + 2 * 16384].reshape(-1, 2)
ok = tl[:, 0] > 0
if not ok.any():  # tile stamps only in a -DANDES_SCAN_PHASES build (tools/build_variant.py)
    sys.exit(0)
ids = np.where(ok)[0]
dur = (tl[ok, 1] - tl[ok, 0]) / 1e3
print("tiles traced", ok.sum(), "body us median/p90/p99/max", np.percentile(dur, [50, 90, 99, 100]).round(2))
order = np.argsort(-dur)[:12]
base = snap.tl_base.astype(np.int64)
starts = np.bincount(base // 1024, minlength=len(tl))
for k in order:
    t = ids[k]
    print("  tile", t, "dur", round(dur[k], 2), "start", us(tl[t, 0]), "end", us(tl[t, 1]), "req starts", starts[t])
ends = np.sort(tl[ok, 1])
print("tile end percentiles us", [us(np.percentile(ends, p)) for p in (50, 90, 99, 99.9, 100)])
last = ids[np.argsort(-tl[ok, 1])[:8]]
print("last tiles to finish", [(int(t), us(tl[t, 0]), us(tl[t, 1])) for t in last])
st0 = np.sort(tl[ok, 0])
print("tile start percentiles us", [us(np.percentile(st0, p)) for p in (0, 1, 10, 50, 90, 99, 100)])
grid = np.arange(int(us(st0[0])), int(us(ends[-1])) + 2, 2.0)
live = [int(((tl[ok, 0] - t0) / 1e3 <= g).sum() - ((tl[ok, 1] - t0) / 1e3 <= g).sum()) for g in grid]
print("tiles in flight every 2 us from", grid[0], ":", live)
ph = tr[49152:65536].reshape(-1, 4)
okp = ph[:, 0] > 0
if okp.any():
    ph = ph[okp]
    for k, name in enumerate(["loop entry", "meta in", "carry done", "data in"]):
        print(f"first tile {name:10s} us p0/p10/p50/p90/max", [us(np.percentile(ph[:, k], q)) for q in (0, 10, 50, 90, 100)])
