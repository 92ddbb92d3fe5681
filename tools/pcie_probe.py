"""Pinned-buffer PCIe rates on this box: H2D / D2H of 4 MiB from several
pinned host buffers (torch pin_memory, fresh pinned empty, cudaHostAlloc via
torch), CUDA events, best and median of 20."""
import numpy as np
import torch

dev = torch.device("cuda", 0)
n = 1 << 20
d = torch.empty(n, dtype=torch.float32, device=dev)
bufs = {
    "pin_memory(from_numpy)": torch.from_numpy(np.random.default_rng(0).standard_normal(n).astype(np.float32)).pin_memory(),
    "empty(pin_memory=True)": torch.empty(n, dtype=torch.float32, pin_memory=True),
    "empty(pin_memory=True) filled": torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1.0),
    "pin_memory(from_numpy) 2": torch.from_numpy(np.ones(n, np.float32)).pin_memory(),
}


def rate(fn):
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return 4 * n / min(ts) / 1e9, 4 * n / float(np.median(ts)) / 1e9


for name, h in bufs.items():
    h2d = rate(lambda: d.copy_(h, non_blocking=True))
    d2h = rate(lambda: h.copy_(d, non_blocking=True))
    print(f"{name:32s} h2d best/med {h2d[0]:6.1f}/{h2d[1]:6.1f} GB/s   d2h {d2h[0]:6.1f}/{d2h[1]:6.1f} GB/s  ptr%2M={h.data_ptr() % (2 << 20)}")
