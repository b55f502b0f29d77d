import time, numpy as np, torch, mmap
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
n = 23_000_000
src = torch.rand(n, dtype=torch.float32).pin_memory()
def t(f, reps=3):
    f()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    return (time.perf_counter() - t0) / reps * 1e3
pre = np.empty(n); pre.fill(1)
print("copy into touched fp64", t(lambda: torch.from_numpy(pre).copy_(src)))
print("copy into fresh np.empty", t(lambda: torch.from_numpy(np.empty(n)).copy_(src)))
print("fresh np.empty + fill", t(lambda: np.empty(n).fill(0)))
def mm():
    m = mmap.mmap(-1, n * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | mmap.MAP_POPULATE)
    a = np.frombuffer(m, dtype=np.float64)
    torch.from_numpy(a).copy_(src)
print("mmap populate + copy", t(mm))
def mm2():
    m = mmap.mmap(-1, n * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.float64)
    torch.from_numpy(a).copy_(src)
print("mmap hugepage + copy", t(mm2))
print("torch.empty f64 + copy", t(lambda: torch.empty(n, dtype=torch.float64).copy_(src)))
