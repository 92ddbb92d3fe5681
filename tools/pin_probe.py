"""Why do some pinned buffers copy H2D at ~13 GB/s and others at ~51 GB/s on
the same box?  Times 4 MiB H2D copies (CUDA events, best/median of 20) from:
  * torch pinned buffers with different contents (random / ones / zeros), the
    same buffer re-filled, to separate content from allocation;
  * mmap'd anonymous memory with MADV_HUGEPAGE (THP) vs MADV_NOHUGEPAGE,
    page-locked by cudaHostRegister;
  * one large cudaHostAlloc arena (64 MiB) carved into 4 MiB views.
Prints the THP settings and AnonHugePages of this process."""
import ctypes as C
import mmap
import os

import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 1 << 20
NB = 4 * n
d = torch.empty(n, dtype=torch.float32, device=dev)
libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
try:
    cudart = C.CDLL("libcudart.so")
except OSError:
    pass
MADV_HUGEPAGE, MADV_NOHUGEPAGE = 14, 15


def show(path):
    try:
        return open(path).read().strip()
    except OSError as e:
        return f"? {e}"


print("thp enabled:", show("/sys/kernel/mm/transparent_hugepage/enabled"))
print("thp defrag:", show("/sys/kernel/mm/transparent_hugepage/defrag"))
print("hugepages:", show("/proc/sys/vm/nr_hugepages"))


def rate(h):
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return f"{NB / min(ts) / 1e9:6.1f}/{NB / float(np.median(ts)) / 1e9:6.1f}"


rnd = np.random.default_rng(0).standard_normal(n).astype(np.float32)
for i in range(3):
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    out = []
    for name, fill in (("random", lambda a: a.__setitem__(slice(None), rnd)),
                       ("ones", lambda a: a.fill(1.0)),
                       ("zeros", lambda a: a.fill(0.0)),
                       ("random", lambda a: a.__setitem__(slice(None), rnd))):
        fill(h.numpy())
        out.append(f"{name} {rate(h)}")
    print(f"torch pinned #{i}: " + " | ".join(out))


def mmap_buf(advice):
    p = libc.mmap(None, NB + (2 << 20), 3, 0x22, -1, 0)  # RW, PRIVATE|ANON
    a = (p + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    if advice is not None:
        libc.madvise(C.c_void_p(a), NB, advice)
    arr = np.ctypeslib.as_array((C.c_float * n).from_address(a))
    arr[:] = rnd
    st = torch.cuda.cudart().cudaHostRegister(a, NB, 0)
    return a, arr, st


for name, adv in (("mmap THP", MADV_HUGEPAGE), ("mmap noTHP", MADV_NOHUGEPAGE), ("mmap default", None)):
    a, arr, st = mmap_buf(adv)
    h = torch.from_numpy(arr)
    r1 = rate(h)
    arr.fill(1.0)
    r2 = rate(h)
    print(f"{name}: register={st} random {r1} | ones {r2}")

arena = torch.empty(16 * n, dtype=torch.float32, pin_memory=True)
arena.numpy()[:] = np.tile(rnd, 16)
print("arena 64 MiB views:", " ".join(rate(arena[i * n:(i + 1) * n]) for i in range(16)))
for line in open("/proc/self/smaps_rollup"):
    if "AnonHuge" in line or "Rss" in line:
        print(line.strip())
