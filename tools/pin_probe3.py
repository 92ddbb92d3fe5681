"""Third pinned-memory probe: reproduce tools/pcie_probe.py's allocation order
(the run where buffers 3 and 4 copied H2D at ~13 GB/s), measure each buffer
twice in both orders, and for each report how physically contiguous its pages
are (/proc/self/pagemap, root only): number of physically contiguous runs and
whether they are 2 MiB runs.  Then a THP-backed (madvise) buffer registered
with cudaHostRegister for comparison."""
import ctypes as C
import os
import struct

import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 1 << 20
NB = 4 * n
d = torch.empty(n, dtype=torch.float32, device=dev)


def rate(h):
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return NB / float(np.median(ts)) / 1e9


def phys_runs(addr, nbytes):
    """(#physically contiguous runs, #4K pages, pfn of first page) via pagemap."""
    try:
        f = open("/proc/self/pagemap", "rb")
    except OSError as e:
        return f"pagemap: {e}"
    pages = nbytes // 4096
    runs, prev, first = 0, None, None
    for i in range(pages):
        f.seek(((addr // 4096) + i) * 8)
        v = struct.unpack("<Q", f.read(8))[0]
        if not (v >> 63) & 1:
            return "page not present"
        pfn = v & ((1 << 55) - 1)
        if first is None:
            first = pfn
        if pfn == 0:
            return "pfn hidden"
        if prev is None or pfn != prev + 1:
            runs += 1
        prev = pfn
    return f"{runs} runs over {pages} pages (pfn0 % 512 = {first % 512})"


bufs = {
    "pin_memory(from_numpy)": torch.from_numpy(np.random.default_rng(0).standard_normal(n).astype(np.float32)).pin_memory(),
    "empty(pin_memory=True)": torch.empty(n, dtype=torch.float32, pin_memory=True),
    "empty(pin_memory=True) filled": torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0),
    "pin_memory(from_numpy) 2": torch.from_numpy(np.ones(n, np.float32)).pin_memory(),
}
# a few more, like bench.py's (idx int64, off int64, grad f32, out f32)
for i in range(6):
    bufs[f"bench-like #{i}"] = torch.from_numpy(np.random.default_rng(i).standard_normal(n).astype(np.float32)).pin_memory()
res = {k: [rate(h)] for k, h in bufs.items()}
for k, h in reversed(list(bufs.items())):
    res[k].append(rate(h))
for k, h in bufs.items():
    print(f"{k:32s} h2d {res[k][0]:5.1f} / {res[k][1]:5.1f} GB/s  {phys_runs(h.data_ptr(), NB)}")

libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
for adv, name in ((14, "mmap+MADV_HUGEPAGE"), (15, "mmap+MADV_NOHUGEPAGE")):
    for rep in range(3):
        p = libc.mmap(None, NB + (2 << 20), 3, 0x22, -1, 0)
        a = (p + (2 << 20) - 1) // (2 << 20) * (2 << 20)
        libc.madvise(C.c_void_p(a), NB, adv)
        arr = np.ctypeslib.as_array((C.c_float * n).from_address(a))
        arr[:] = 1.0
        st = torch.cuda.cudart().cudaHostRegister(a, NB, 0)
        print(f"{name} #{rep}: register={int(st)} h2d {rate(torch.from_numpy(arr)):5.1f} GB/s  {phys_runs(a, NB)}")
