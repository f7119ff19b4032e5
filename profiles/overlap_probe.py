import time, torch
n = 411041792 // 4
h_in = [torch.empty(n).pin_memory() for _ in range(2)]
h_out = [torch.empty(n).pin_memory() for _ in range(2)]
d_in = [torch.empty(n, device="cuda") for _ in range(2)]
d_out = [torch.empty(n, device="cuda") for _ in range(2)]
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
big_a = torch.empty(2 * 1024**3 // 4, device="cuda")
big_b = torch.empty_like(big_a)
s_h2d, s_d2h, s_main = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
import sys
MODE = sys.argv[1] if len(sys.argv) > 1 else "matmul"
def compute():
    if MODE == "matmul":
        for _ in range(3): a.mul_(1.0).matmul(a)
    else:  # HBM-bound: ~4 ms of 8 GB/s... device copies
        for _ in range(3): big_b.copy_(big_a)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s_main): compute()
    torch.cuda.synchronize(); print(MODE, "compute alone ms", (time.perf_counter()-t0)*1e3)
ev = {}
def step(i):
    k = i & 1
    with torch.cuda.stream(s_h2d):
        if ("in_free", k) in ev: s_h2d.wait_event(ev[("in_free", k)])
        d_in[k].copy_(h_in[k], non_blocking=True)
        e = torch.cuda.Event(); e.record(s_h2d); ev[("h2d", k)] = e
    with torch.cuda.stream(s_main):
        s_main.wait_event(ev[("h2d", k)])
        d_out[k].copy_(d_in[k])
        e = torch.cuda.Event(); e.record(s_main); ev[("in_free", k)] = e
        compute()
        e = torch.cuda.Event(); e.record(s_main); ev[("out", k)] = e
    with torch.cuda.stream(s_d2h):
        s_d2h.wait_event(ev[("out", k)])
        h_out[k].copy_(d_out[k], non_blocking=True)
for i in range(2): step(i)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(8): step(i)
torch.cuda.synchronize()
print("pipelined period ms", (time.perf_counter()-t0)/8*1e3)
