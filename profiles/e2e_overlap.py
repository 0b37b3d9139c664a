"""Where the chained e2e step's time goes: the TP-MLP compute (AG-GEMM -> GEMM-RS
at n = 1, S = 16384) alone, the 512 MiB H2D / D2H copies alone and together,
and compute with both copies running beside it."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2511_13940_b200 as pk

S = 16384
comm = pk.local_group(1)[0]
x = comm.empty((S, S)); x.copy_(torch.randn(S, S, device="cuda").bfloat16())
w1 = torch.randn(S, S, device="cuda").bfloat16(); w2 = torch.randn(S, S, device="cuda").bfloat16()
mid = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
y = comm.empty((S, S))
hx = torch.empty(S, S, dtype=torch.bfloat16, pin_memory=True)
hy = torch.empty(S, S, dtype=torch.bfloat16, pin_memory=True)
dx = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
dy = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
cur = torch.cuda.current_stream()


def t(fn, k=6):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def compute():
    pk.all_gather_gemm(comm, x, w1, out=mid)
    pk.gemm_reduce_scatter(comm, mid, w2, out=y)


def h2d():
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    cur.wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    cur.wait_stream(s2)


def both():
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


def all3():
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    compute()
    cur.wait_stream(s1); cur.wait_stream(s2)


r = dict(compute_ms=t(compute), h2d_ms=t(h2d), d2h_ms=t(d2h), h2d_d2h_ms=t(both), all3_ms=t(all3), bytes_each=S * S * 2)
dx, dy = comm.empty((S, S)), comm.empty((S, S))     # the same copies into / out of symmetric (VMM) memory
r.update(vmm_h2d_ms=t(h2d), vmm_d2h_ms=t(d2h), vmm_h2d_d2h_ms=t(both), vmm_all3_ms=t(all3))
print(json.dumps(r))



# the bench's double-buffered pipeline (bench.py e2e_measure), chained
def pipeline(k, x_sets, y_sets, hx, hys):
    done_c, done_o = [None, None], [None, None]
    for i in range(k):
        xs, ys = x_sets[i % 2], y_sets[i % 2]
        with torch.cuda.stream(s1):
            if done_c[i % 2] is not None:
                s1.wait_event(done_c[i % 2])
            xs.copy_(hx, non_blocking=True)
            ev_in = torch.cuda.Event(); ev_in.record(s1)
        cur.wait_event(ev_in)
        if done_o[i % 2] is not None:
            cur.wait_event(done_o[i % 2])
        pk.all_gather_gemm(comm, xs, w1, out=mid)
        pk.gemm_reduce_scatter(comm, mid, w2, out=ys)
        ev_c = torch.cuda.Event(); ev_c.record(cur)
        done_c[i % 2] = ev_c
        with torch.cuda.stream(s2):
            s2.wait_event(ev_c)
            hys[i % 2].copy_(ys, non_blocking=True)
            ev_o = torch.cuda.Event(); ev_o.record(s2)
            done_o[i % 2] = ev_o
    cur.wait_stream(s1); cur.wait_stream(s2)


import time
comm2 = comm
xs2 = [x, comm.empty((S, S))]
ys2 = [y, comm.empty((S, S))]
hys = [hy, torch.empty(S, S, dtype=torch.bfloat16, pin_memory=True)]
pipeline(2, xs2, ys2, hx, hys); torch.cuda.synchronize()
for k in (4, 8, 16):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(); pipeline(k, xs2, ys2, hx, hys); e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(json.dumps(dict(pipeline_k=k, ms_per_step=e0.elapsed_time(e1) / k, host_issue_ms=(t1 - t0) * 1e3 / k)))
comm.destroy()
