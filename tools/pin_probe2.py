"""Follow-up to pin_probe.py: is the slow H2D (~13 GB/s) of some pinned
buffers caused by HOW the CPU wrote them (torch multi-threaded copy / fill vs a
single-threaded numpy write) and does it persist?  4 MiB H2D, CUDA events."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 1 << 20
NB = 4 * n
d = torch.empty(n, dtype=torch.float32, device=dev)
rnd = np.random.default_rng(0).standard_normal(n).astype(np.float32)


def rate(h):
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return f"{NB / min(ts) / 1e9:5.1f}/{NB / float(np.median(ts)) / 1e9:5.1f}"


print("torch threads", torch.get_num_threads())
src = torch.from_numpy(rnd)
for trial in range(2):
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.numpy()[:] = rnd
    a = rate(h)
    h.copy_(src)
    b = rate(h)
    h.fill_(1.0)
    c = rate(h)
    h.numpy()[:] = rnd
    e = rate(h)
    time.sleep(0.5)
    f = rate(h)
    h.copy_(src)
    g = rate(h)
    big = np.ones(64 << 20, np.float32)  # 256 MB of CPU writes (evicts caches)
    big += 1
    k = rate(h)
    print(f"trial {trial}: numpy-write {a} | torch copy_ {b} | torch fill_ {c} | numpy-write again {e} | "
          f"+0.5s {f} | torch copy_ {g} | after 256MB CPU writes {k}")
    del big
p = torch.from_numpy(rnd).pin_memory()
print("from_numpy().pin_memory():", rate(p))
torch.set_num_threads(1)
p1 = torch.from_numpy(rnd).pin_memory()
print("from_numpy().pin_memory() with 1 torch thread:", rate(p1))
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.copy_(src)
print("torch copy_ with 1 thread:", rate(h))
torch.set_num_threads(16)
d2 = torch.empty(n, dtype=torch.float32, device=dev)
h.copy_(d2)
torch.cuda.synchronize()
print("after a D2H into it:", rate(h))
