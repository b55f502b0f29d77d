import time, torch, numpy as np
n = 23_000_000
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
d = torch.rand(n, device="cuda", dtype=torch.float64)
def alloc_copy():
    out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out.copy_(d, non_blocking=True); torch.cuda.synchronize()
    return out.numpy()
print("alloc+copy, result dropped", t(alloc_copy))
keep = []
def alloc_keep():
    global keep
    r = alloc_copy()
    keep = [r]
print("alloc+copy, result kept until next", t(alloc_keep))
def alloc_keep2():
    global keep
    keep = []
    r = alloc_copy()
    keep = [r]
print("alloc+copy, dropped before next", t(alloc_keep2))
