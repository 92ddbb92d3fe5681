"""Pinned-buffer H2D / D2H rates as a function of where the host pages live and
which cores drive the copy: for every NUMA node, pin this process to the node's
CPUs, first-touch a fresh pinned buffer there, and time 4 MiB copies with CUDA
events (best / median of 20).  Prints the GPU's own NUMA node from sysfs."""
import glob
import os

import numpy as np
import torch

dev = torch.device("cuda", 0)
torch.cuda.init()
bus = torch.cuda.get_device_properties(dev)
pci = "%04x:%02x:%02x.0" % (bus.pci_domain_id, bus.pci_bus_id, bus.pci_device_id)
gpu_node = open(f"/sys/bus/pci/devices/{pci}/numa_node").read().strip() if os.path.exists(
    f"/sys/bus/pci/devices/{pci}/numa_node") else "?"
local = open(f"/sys/bus/pci/devices/{pci}/local_cpulist").read().strip() if os.path.exists(
    f"/sys/bus/pci/devices/{pci}/local_cpulist") else "?"
print(f"gpu {pci} numa_node={gpu_node} local_cpulist={local} allowed={len(os.sched_getaffinity(0))} cpus")


def parse(lst):
    out = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


nodes = {}
for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    nodes[int(p.rsplit("node", 1)[1])] = parse(open(p + "/cpulist").read().strip())
print("nodes", {k: (min(v), max(v), len(v)) for k, v in nodes.items() if v})

n = 1 << 20
d = torch.empty(n, dtype=torch.float32, device=dev)
allowed = os.sched_getaffinity(0)


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


for node, cpus in nodes.items():
    cpus = cpus & allowed
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.numpy()[:] = np.random.default_rng(node).standard_normal(n).astype(np.float32)
    h2d = rate(lambda: d.copy_(h, non_blocking=True))
    d2h = rate(lambda: h.copy_(d, non_blocking=True))
    print(f"node {node}: h2d best/med {h2d[0]:6.1f}/{h2d[1]:6.1f} GB/s  d2h {d2h[0]:6.1f}/{d2h[1]:6.1f} GB/s")
    # the same buffer, copied while pinned to every other node
    for other, oc in nodes.items():
        oc = oc & allowed
        if other == node or not oc:
            continue
        os.sched_setaffinity(0, oc)
        h2d = rate(lambda: d.copy_(h, non_blocking=True))
        print(f"   pages on {node}, thread on {other}: h2d best/med {h2d[0]:6.1f}/{h2d[1]:6.1f} GB/s")
os.sched_setaffinity(0, allowed)
