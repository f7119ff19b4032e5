"""Host↔device copy bandwidth of this box: H2D alone, D2H alone, both at once
(separate streams, pinned host memory), for the e2e roofline."""
import time

import torch

n = 411041792 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


run(True, True, 1)
for name, a, b in (("H2D", True, False), ("D2H", False, True), ("both", True, True)):
    t = run(a, b)
    print(f"{name:5s}: {t * 1e3:7.2f} ms per 411 MB each way -> {411.04 / t / 1e3:6.1f} GB/s per direction")
