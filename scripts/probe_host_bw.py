import os, time, numpy as np, threading
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "OMP", os.environ.get("OMP_NUM_THREADS"))
a = np.ones(64 << 20, np.float32); b = np.empty_like(a)   # 256 MB
for _ in range(2):
    t = time.perf_counter(); np.copyto(b, a); dt = time.perf_counter() - t
    print("1 thread copy GB/s", a.nbytes / dt / 1e9)
def part(i, n):
    s = slice(i * len(a) // n, (i + 1) * len(a) // n); np.copyto(b[s], a[s])
for n in (4, 8, 16):
    th = [threading.Thread(target=part, args=(i, n)) for i in range(n)]
    t = time.perf_counter(); [x.start() for x in th]; [x.join() for x in th]; dt = time.perf_counter() - t
    print(n, "threads copy GB/s", a.nbytes / dt / 1e9)
import torch
x = torch.from_numpy(a)
for pin in (False, True):
    src = x.pin_memory() if pin else x
    torch.cuda.synchronize()
    for _ in range(2):
        t = time.perf_counter(); y = src.to("cuda", non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
        print("h2d pinned" if pin else "h2d pageable", a.nbytes / dt / 1e9, "GB/s")
t = time.perf_counter(); r = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0); dt = time.perf_counter() - t
print("cudaHostRegister 256MB", r, dt * 1e3, "ms")
