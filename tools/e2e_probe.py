"""Where does the host-buffer (e2e) step time go?  cfg2, pinned buffers."""
import ctypes as C
import sys
import time

import numpy as np
import torch

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_11714_b200 as tt
from paper_2101_11714_b200._lib import lib
import bench

cfg = bench.CONFIGS["cfg2"]
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
plan = tt.plan_shapes(cfg["rows"], cfg["emb"], 3, cfg["rank"], cfg["rf"], cfg["cf"])
table = tt.TtTable(plan, "p", np.float32, device=0, stream=stream.cuda_stream)
table.init_sampled_gaussian(1)
idx, off, grad = bench.make_inputs(cfg, 7, tt)
L, B, N = len(idx), cfg["bags"], 16
h_idx = torch.from_numpy(idx).pin_memory()
h_off = torch.from_numpy(off).pin_memory()
h_grad = torch.from_numpy(grad).pin_memory()
h_out = torch.empty((B, N), dtype=torch.float32).pin_memory()
d_idx = torch.empty_like(h_idx, device=dev)
d_out = torch.empty_like(h_out, device=dev)
d_grad = torch.empty_like(h_grad, device=dev)


def timeit(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t0) / n * 1e6:9.1f} us", flush=True)


with torch.cuda.stream(stream):
    timeit("H2D idx 512KB", lambda: d_idx.copy_(h_idx, non_blocking=True))
    timeit("H2D grad 4MB", lambda: d_grad.copy_(h_grad, non_blocking=True))
    timeit("D2H out 4MB", lambda: h_out.copy_(d_out, non_blocking=True))
ctx = tt.ForwardContext(table)
hi, ho, hg, hout = (h_idx.numpy(), h_off.numpy(), h_grad.numpy(), h_out.numpy())


def fwd():
    st = lib().ttgpu_forward(table.handle, hi.ctypes.data_as(C.c_void_p), L,
                             ho.ctypes.data_as(C.c_void_p), B, None, 0, 2048, 1,
                             hout.ctypes.data_as(C.c_void_p), ctx.handle)
    assert st == 0


def bwd():
    st = lib().ttgpu_backward_sgd(table.handle, ctx.handle, L, B, hg.ctypes.data_as(C.c_void_p),
                                  B * N, C.c_double(0.01))
    assert st == 0


timeit("ttgpu_forward (host)", fwd)
timeit("ttgpu_forward + backward_sgd (host)", lambda: (fwd(), bwd()))
batch = tt.IndexBatch(hi, ho)
timeit("py forward_bags+backward_sgd", lambda: (tt.forward_bags(table, batch, save_intermediates=True), None))
# unpinned
ui, uo, ug = idx.copy(), off.copy(), grad.copy()
uout = np.empty((B, N), np.float32)


def fwd_u():
    st = lib().ttgpu_forward(table.handle, ui.ctypes.data_as(C.c_void_p), L,
                             uo.ctypes.data_as(C.c_void_p), B, None, 0, 2048, 1,
                             uout.ctypes.data_as(C.c_void_p), ctx.handle)
    assert st == 0


timeit("ttgpu_forward (pageable host)", fwd_u)
import os
os.environ["TTGPU_TRACE"] = "1"
for _ in range(3):
    fwd()
    bwd()
    print("---", flush=True)
