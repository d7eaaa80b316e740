import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2404_16283_b200 as A, workloads as W
n = 3500
tl = [(np.arange(6, dtype=np.uint32) * 250_000 + 1_400_000) for _ in range(n)]
g, base, pool = W._pack(tl)
rng = np.random.default_rng(11)
snap = W.Snapshot(arrival_us=np.zeros(n, np.int64), ttft_us=np.full(n, 1_000_000, np.uint32),
                  period_us=np.full(n, 208_333, np.uint32), ctx_len=np.full(n, 100, np.uint32),
                  n_deliv=g, max_total=np.full(n, W.UINT32_MAX, np.uint32), start_off_us=np.zeros(n, np.uint32),
                  rank=rng.permutation(n).astype(np.uint32), running=(rng.random(n) < 0.02).astype(np.uint8),
                  tl_base=base, tl_pool=pool, now_us=3_000_000, horizon_us=2_000_000,
                  tau_us=W.tau_table(48), kv_capacity=4000)
ctx = A.Context(max_requests=1 << 17, max_B=256, max_tokens=1 << 24, max_running=4096)
tau = torch.from_numpy(snap.tau_us.view(np.int32)).cuda()
L = A.lib(); L.andes_debug_read.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]
for fl in (1, 1 | 32, 1 | 64):
    d = ctx.schedule(A.requests_to(snap), n, snap.now_us, snap.horizon_us, tau, snap.kv_capacity, preempt_cap=5, flags=fl)
    torch.cuda.synchronize()
    gl = np.zeros(32, np.uint32); L.andes_debug_read(ctx._h, 5, gl.ctypes.data, gl.nbytes)
    # Globals: run_l(0,1) pool_end(2,3) ntiles4 inv_minP5 n_run6 done7 B_lo8 B_hi9 trig10 err11 slow12 tile13 prep14 state15 tlo16 thi17 theta18 n_surv19 ovf20
    print(fl, 'sc', d.scalars.cpu().numpy().view(np.uint32)[:8], 'theta', hex(gl[18]), 'ns', gl[19], 'ovf', gl[20], 'slow', gl[12], 'maxrank', gl[31])
