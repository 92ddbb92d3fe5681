"""TT-EmbeddingBag fwd+bwd+SGD throughput (BASELINE.json metric) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config cfg2]

One step = forward_bags(save) + backward_bags + sgd_step over one batch of
the configuration's synthetic index stream (cfg2 = BASELINE configs[1]:
10,131,227 x 16, R=32, 65,536 bags x 1 index, Zipf(1.05)).  Per GPU the batch
is fixed (weak scaling); N>1 runs one process per GPU (torchrun) and sums the
dense core gradients with an NCCL allreduce before the identical SGD.

Timing: W untimed warm-up steps, then K steps, each replayed from a CUDA graph
of the whole step and bracketed by CUDA events on the table's stream; L2 is
flushed (256 MiB write) before every timed step and the flush is outside the
events.  Multi-GPU: barrier + synchronize around the timed region and the max
over ranks.  `e2e` repeats the step through the reference-facing host C-ABI
calls (host buffers, H2D of indices/offsets/grad_out and D2H of the pooled
output inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TT-EmbeddingBag fwd+bwd indices/sec (11M×16, rank 32, batch 64K) at 1/2/4/8 GPU"

CONFIGS = {
    # name: rows, emb, row_factors, col_factors, rank, bags, pooling_factor, zipf exponent
    "cfg1": dict(rows=1000000, emb=16, rf=[100, 100, 100], cf=[2, 2, 4], rank=16, bags=4096,
                 pf=1, zipf=0.0,
                 desc="1M rows (100x100x100), dim 16 (2x2x4), R=16, 4096 bags x 1, uniform"),
    "cfg2": dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32, bags=65536,
                 pf=1, zipf=1.05,
                 desc="10,131,227 rows (200x220x250), dim 16 (2x2x4), R=32, 65,536 bags x 1, "
                      "Zipf(1.05), fwd+bwd+SGD"),
    "cfg2u": dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32, bags=65536,
                  pf=1, zipf=0.0, desc="cfg2 shape with uniform indices"),
    "cfg4": dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32, bags=65536,
                 pf=1, zipf=1.2, cache=True,
                 desc="cfg2 shape with the LFU hot-row cache (0.01% = 1,013 rows), Zipf(1.2), "
                      "fwd+bwd+SGD; the cache is warmed on W other Zipf(1.2) batches (not the "
                      "timed one), then admits the top 1,013 rows"),
    "cfg2z12": dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32, bags=65536,
                    pf=1, zipf=1.2,
                    desc="cfg4 without the cache: cfg2 shape, Zipf(1.2), fwd+bwd+SGD "
                         "(the like-for-like uncached step beside cfg4)"),
    "cfg3": dict(rows=40000000, emb=64, rf=[200, 200, 1000], cf=[4, 4, 4], rank=64, bags=65536,
                 pf=32, zipf=0.0,
                 desc="40M rows (200x200x1000), dim 64 (4x4x4), R=64, 65,536 bags x 32, uniform"),
}
CONFIGS["cfg5"] = dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32,
                      bags=65536, pf=1, zipf=1.05, collection=True,
                      desc="DLRM cfg5 embeddings: 26 Criteo-Kaggle sparse features, the 7 "
                           "largest TT-compressed at R=32 (paper Table 2) + 19 uncompressed, "
                           "65,536 bags x 1 per feature, Zipf(1.05) (device sampler), "
                           "fwd+bwd+SGD in one multi-stream CUDA graph per step")
CONFIGS["cfg5m"] = dict(rows=10131227, emb=16, rf=[200, 220, 250], cf=[2, 2, 4], rank=32,
                       bags=65536, pf=1, zipf=1.05, model=True,
                       desc="DLRM cfg5 full training step (DlrmModel, model.hpp:355-538): 13 dense "
                            "features, bottom MLP 512-256-64-16, 26 Criteo-Kaggle sparse features "
                            "(7 TT at R=32 + 19 uncompressed), Dot interaction, top MLP 512-256-1, "
                            "BCE, SGD; 65,536 samples per step")
LR = 0.01


def flops_per_lookup(rf, cf, ranks):
    """F_fwd = 2*sum_{k>=1} prefix[k-1]*R_k*n_k*R_{k+1}; F_bwd = 2*F_fwd."""
    d = len(rf)
    pre = [int(np.prod(cf[: k + 1])) for k in range(d)]
    f = sum(2 * pre[k - 1] * ranks[k] * cf[k] * ranks[k + 1] for k in range(1, d))
    return 3 * f


def kernel_work(name, rf, cf, ranks, L, B, N, params):
    """Algorithmic work of one launch of a fast-path kernel (SURVEY §8(d) per-lookup
    figures, reference chain, no dedup): (flops, hbm_bytes).  3-core chain:
    fwd  H = G0[i0]·G1[i1] (2·n0·R1·n1R2), y = H·G2[i2] (2·n0n1·R2·n2)
    bwd1 D1 = D2·G2ᵀ (2·n0n1·n2·R2), dG1 += G0ᵀ·D1 and D0 = D1·G1ᵀ (2·n0·R1·n1R2 each)
    bwd2 dG2 += Hᵀ·D2 (2·n0n1·R2·n2)."""
    n0, n1, n2 = cf
    R1, R2 = ranks[1], ranks[2]
    head = 2 * n0 * R1 * n1 * R2
    tail = 2 * n0 * n1 * R2 * n2
    idx_b = 8 * L
    table = {
        "f3_fwd": (L * (head + tail), idx_b + 4 * L * N),
        "f3_bwd1": (L * (tail + 2 * head), idx_b + 4 * B * N),
        "f3_bwd2": (L * tail, idx_b + 4 * B * N),
        "f3_combine": (2 * params, 3 * 4 * params),
        "pool": (2 * L * N, 4 * L * N + 8 * (B + 1) + 4 * B * N),
        # cfg3's wide-row phases (wide3.cuh; per-lookup tail work, no dedup):
        # bwd_S = k_w3_bwd_pairs: D1 (S) and the dG2 contribution per lookup;
        # bytes: grad row in, contribution row out, indices
        "bwd_S": (L * 2 * tail, idx_b + 4 * L * N + 4 * L * R2 * n2),
        # tail_pool = k_w3_fwd + pooling: y per lookup, y rows out and back, pooled rows
        "tail_pool": (L * tail + 2 * L * N, idx_b + 2 * 4 * L * N + 4 * B * N),
    }
    return table.get(name)


def bytes_per_step(L, B, N, params):
    """Algorithmic HBM bytes per step: indices + offsets read twice (fwd, bwd),
    pooled output written, grad_out read, cores read + written once."""
    return 2 * 8 * L + 2 * 8 * (B + 1) + 4 * B * N + 4 * B * N + 2 * 4 * params


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def gpu_local_cpus(dev_index):
    """The host CPUs of the GPU's own NUMA node (sysfs local_cpulist) that this
    process may run on, or None.  The e2e section runs there, so its pinned
    buffers are allocated (first-touched) in the GPU's node: H2D DMA reads from
    a remote node's pages measured 11-18 GB/s on some boxes against ~50 GB/s
    local (tools/numa_probe.py)."""
    import torch

    if os.environ.get("TTGPU_BENCH_NUMA", "1") == "0":
        return None
    try:
        p = torch.cuda.get_device_properties(dev_index)
        pci = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        text = open(f"/sys/bus/pci/devices/{pci}/local_cpulist").read().strip()
    except Exception:  # noqa: BLE001 - no sysfs entry: leave the affinity alone
        return None
    cpus = set()
    for part in text.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    cpus &= os.sched_getaffinity(0)
    return cpus or None


def cta_timeline(path, run, flush, stream):
    """Diagnostic (outside every timed region): one graph replay with the
    per-CTA entry / exit timers of the five fast-path kernels enabled
    (ttgpu_debug_cta_times), saved raw to `path` and summarised on stderr."""
    import ctypes as C

    import torch

    from paper_2101_11714_b200._lib import lib

    names = ["f3_gsort", "f3_fwd", "f3_srows_bwd2", "f3_bwd1", "f3_combine"]
    bufs = [torch.zeros(8 * 8192, dtype=torch.int64, device="cuda") for _ in names]
    for k, b in enumerate(bufs):
        assert lib().ttgpu_debug_cta_times(k, C.c_void_p(b.data_ptr())) == 0
    with torch.cuda.stream(stream):
        flush.fill_(3)
        run()
    stream.synchronize()
    for k in range(len(names)):
        lib().ttgpu_debug_cta_times(k, None)
    out = {}
    t0 = None
    for name, b in zip(names, bufs):
        a = b.view(-1, 8).cpu().numpy()
        a = a[a[:, 0] > 0]
        out[name] = a
        if len(a) and (t0 is None or a[:, 0].min() < t0):
            t0 = a[:, 0].min()
    np.savez(path, **out)
    for name in names:
        a = out[name]
        if not len(a):
            continue
        st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        d = en - st
        print(f"[cta] {name:14s} ctas {len(a):5d} span {st.min():7.2f}..{en.max():7.2f} us  "
              f"dur mean {d.mean():6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d, 90):6.2f} "
              f"max {d.max():6.2f}  last-start {st.max():7.2f}  end p50 {np.median(en):7.2f}",
              file=sys.stderr)


def make_inputs(cfg, seed, tt):
    if cfg["zipf"] > 0:
        b = tt.generate_zipfian_batch(cfg["rows"], cfg["zipf"], seed, cfg["bags"], cfg["pf"])
        idx, off = b.indices, b.offsets
    else:
        idx = tt.uniform_indices(cfg["rows"], seed, cfg["bags"] * cfg["pf"])
        off = np.arange(0, cfg["bags"] * cfg["pf"] + 1, cfg["pf"], dtype=np.int64)
    g = np.random.default_rng(seed + 1000).standard_normal((cfg["bags"], cfg["emb"]))
    return idx, off, g.astype(np.float32)


def make_inputs_reference(cfg, seed):
    """The same bytes as make_inputs, drawn by the REFERENCE's own generators
    (oracle/_ref: ZipfianSampler + generate_zipfian_batch, Rng::uniform_int;
    data.cpp:8-47, rng.hpp:47-51) -- the reference arm never loads this repo's
    package or its libraries."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    ref = pyoracle.RefImpl()
    if cfg["zipf"] > 0:
        idx, off = ref.zipf_batch(cfg["rows"], cfg["zipf"], seed, cfg["bags"], cfg["pf"])
    else:
        idx = ref.uniform_int(seed, 0, cfg["rows"], cfg["bags"] * cfg["pf"])
        off = np.arange(0, cfg["bags"] * cfg["pf"] + 1, cfg["pf"], dtype=np.int64)
    g = np.random.default_rng(seed + 1000).standard_normal((cfg["bags"], cfg["emb"]))
    return idx, off, g.astype(np.float32)


def workload_config(cfg, world):
    """The `config` object both arms print (identical for the same flags): the
    workload only; how each arm executes it goes under `execution`."""
    L = cfg["bags"] * cfg["pf"]
    return {"workload": cfg["desc"], "global_batch": cfg["bags"] * world,
            "lookups_per_step": L * world,
            "parallelism": f"dp{world}" if world > 1 else "single-gpu",
            "l2": "GPU arm: flushed (256 MiB write) before every timed step, outside the events"}


def cpu_reference_time(cfg, idx, off, grad, budget_s=10.0, steps=None, warmup=0):
    """The reference's own OpenMP CPU step (oracle/_ref, compiled from the
    reference sources) on this host's cores; falls back to the C restatement.
    steps=None: as many steps as fit budget_s (3..50); else exactly `steps`
    timed steps after `warmup` untimed ones."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    threads = os.cpu_count() or 1
    plan = pyoracle.Plan(cfg["rows"], cfg["emb"], cfg["rf"], cfg["cf"],
                         [1] + [cfg["rank"]] * (len(cfg["rf"]) - 1) + [1])
    L = len(idx)
    if pyoracle.ref_available():
        ref = pyoracle.RefImpl()
        t = ref.table(plan, np.float32, "cpu")
        t.init_sampled_gaussian(1)
        if steps is None:
            first = t.time_step(idx, off, grad, LR, reps=1, threads=threads)
            reps = int(max(3, min(50, budget_s / max(first, 1e-6))))
        else:
            if warmup > 0:
                t.time_step(idx, off, grad, LR, reps=warmup, threads=threads)
            reps = max(1, int(steps))
        sec = t.time_step(idx, off, grad, LR, reps=reps, threads=threads)
        kind = "reference"
        # BASELINE.md §3.2 also asks for 1 thread and the serial ref:: pair
        # (bounded: 1 warm-up + 3 steps each, skipped when one step > 20 s)
        extra = {}
        if sec * threads < 20.0:
            s1 = t.time_step(idx, off, grad, LR, reps=3, threads=1)
            ss = t.time_step_serial(idx, off, grad, LR, reps=3)
            t.time_step(idx, off, grad, LR, reps=0, threads=threads)  # restore the thread count
            extra = {"threads_1": {"value": L / s1, "ms_per_step": s1 * 1e3},
                     "serial_ref": {"value": L / ss, "ms_per_step": ss * 1e3,
                                    "what": "ref::forward_bags + ref::backward_bags (serial "
                                            "oracle, embedding_ops.hpp:378-492) + sgd_step"}}
    else:
        orc = pyoracle.Oracle()
        rng = np.random.default_rng(0)
        cores = [rng.standard_normal(plan.core_size(k)).astype(np.float32) * 0.3
                 for k in range(plan.tt_dim)]
        reps = 3 if steps is None else max(1, int(steps))
        for _ in range(warmup if steps is not None else 0):
            orc.time_step(plan, cores, idx, off, grad, LR, threads)
        ts = [orc.time_step(plan, cores, idx, off, grad, LR, threads) for _ in range(reps)]
        sec, kind = float(np.median(ts)), "port"
        extra = {}
    return {"value": L / sec, "unit": "indices/s", "cores": threads, "kind": kind, **extra,
            "sample": f"{L} lookups ({cfg['bags']} bags x {cfg['pf']}), median of {reps} steps "
                      f"(fwd save + bwd + sgd, fp32, OMP threads={threads})",
            "ms_per_step": sec * 1e3}


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    idx, off, grad = make_inputs_reference(cfg, 7)
    # W untimed + K timed full-batch steps on all host threads (each step is one
    # reference fwd(save) + bwd + sgd over the whole batch)
    base = cpu_reference_time(cfg, idx, off, grad, steps=args.steps, warmup=args.warmup)
    v = base["value"]
    line = {"metric": METRIC, "value": v, "unit": "indices/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": base["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference Zipf/uniform streams, sampled-Gaussian cores)",
            "impl": "reference",
            "config": workload_config(cfg, world),
            "execution": {"device": "host CPU", "path": "oracle/_ref (reference sources, "
                          "OpenMP): forward_bags(save) + backward_bags + sgd_step",
                          "sample": f"rank 0 only, {len(idx)} lookups per step"},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                   "threads_1", "serial_ref") if k in base},
            "e2e": {"value": v, "unit": "indices/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_collection(args, cfg, rank, world, local):
    """cfg5's TT part: 7 tables trained in one step, one CUDA graph with a
    fork/join over the table streams (paper_2101_11714_b200/collection.py).
    The same step with every table on one stream is timed beside it."""
    import torch

    if os.environ.get("BENCH_SHARE_GPU") == "1":  # test-only, see main()
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("BENCH_BACKEND", "nccl") == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(os.environ["BENCH_BACKEND"])
    import paper_2101_11714_b200 as tt
    from paper_2101_11714_b200.collection import TtEmbeddingCollection, kaggle_plans
    from paper_2101_11714_b200.streams import DeviceZipfSampler, bag_offsets_device

    from paper_2101_11714_b200.dense import KAGGLE_DENSE_ROWS

    plans = kaggle_plans(cfg["rank"], cfg["emb"])
    col = TtEmbeddingCollection(plans, [f"kaggle{i}" for i in range(len(plans))], device=local,
                                dense_rows=KAGGLE_DENSE_ROWS, dense_dim=cfg["emb"])
    B, N = cfg["bags"], cfg["emb"]
    L = B * cfg["pf"]
    inputs, keep = [], []
    for i, p in enumerate(plans):
        s = DeviceZipfSampler(p.num_rows, cfg["zipf"], device=local)
        d_idx = torch.empty(L, dtype=torch.int64, device=dev)
        d_off = torch.empty(B + 1, dtype=torch.int64, device=dev)
        s.draw_device(7 + 131 * rank, i * L, L, d_idx.data_ptr())
        bag_offsets_device(B, cfg["pf"], d_off.data_ptr())
        d_out = torch.empty((B, N), dtype=torch.float32, device=dev)
        d_g = torch.randn((B, N), dtype=torch.float32, device=dev,
                          generator=torch.Generator(device=dev).manual_seed(100 + i))
        keep += [s, d_idx, d_off, d_out, d_g]
        inputs.append((d_idx.data_ptr(), L, d_off.data_ptr(), B, d_out.data_ptr(), d_g.data_ptr()))
    # the 19 uncompressed features: one (n_dense x L) index block, shared offsets
    nd = len(KAGGLE_DENSE_ROWS)
    dd_idx = torch.empty((nd, L), dtype=torch.int64, device=dev)
    for j, rows in enumerate(KAGGLE_DENSE_ROWS):
        s = DeviceZipfSampler(rows, cfg["zipf"], device=local)
        s.draw_device(11 + 131 * rank, (100 + j) * L, L, dd_idx[j].data_ptr())
        keep.append(s)
    dd_off = torch.empty(B + 1, dtype=torch.int64, device=dev)
    bag_offsets_device(B, cfg["pf"], dd_off.data_ptr())
    dd_out = torch.empty((nd, B, N), dtype=torch.float32, device=dev)
    dd_g = torch.randn((nd, B, N), dtype=torch.float32, device=dev,
                       generator=torch.Generator(device=dev).manual_seed(99))
    keep += [dd_idx, dd_off, dd_out, dd_g]
    dense_inputs = (dd_idx.data_ptr(), L, dd_off.data_ptr(), B, dd_out.data_ptr(), dd_g.data_ptr())
    torch.cuda.synchronize(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(run):
        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        with torch.cuda.stream(col.main):
            for i in range(args.steps):
                flush.fill_(i & 0xff)
                ev[i][0].record(col.main)
                run()
                ev[i][1].record(col.main)
        torch.cuda.synchronize(dev)
        tot = float(sum(a.elapsed_time(b) for a, b in ev))
        if world > 1:
            t = torch.tensor([tot], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            tot = float(t.item())
        return tot / args.steps

    for _ in range(3):  # allocate every workspace before capture
        col.step(inputs, LR, dense_inputs)
    col.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if col.capturable:
        col.capture(inputs, LR, dense_inputs)
        run_par = col.replay
    else:  # host-side collective in the step: eager launches
        def run_par():
            col.step(inputs, LR, dense_inputs)
    ms_par = timed(run_par)
    clk = clocks.stop()
    # the same step with every table on the main stream (no overlap between tables)
    for t in col.tables:
        t.set_stream(col.main.cuda_stream)
    col.dense.set_stream(col.main.cuda_stream)
    saved = col.streams
    col.streams = [col.main] * len(saved)
    col.dense_stream = col.main
    if col.capturable:
        col.capture(inputs, LR, dense_inputs)
        run_seq = col.replay
    else:
        def run_seq():
            col.step(inputs, LR, dense_inputs)
    ms_seq = timed(run_seq)
    col.synchronize()
    total = world * (len(plans) + nd) * L
    if rank == 0:
        line = {"metric": METRIC + " [cfg5: 26-feature embedding step]", "value": total / (ms_par / 1e3),
                "unit": "indices/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_par, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic: device Zipf(1.05) streams per table (reference CDF), "
                        "sampled-Gaussian cores, N(0,1) grad_out",
                "config": {"workload": cfg["desc"], "tables": len(plans) + nd, "tt_tables": len(plans),
                           "dense_tables": nd,
                           "lookups_per_step": total, "parallelism":
                               f"dp{world}" if world > 1 else "single-gpu",
                           "l2": "flushed (256 MiB write) before every timed step"},
                "gradient_reduce": ("fused-peer-reduce+sgd" if col.reducers is not None else
                                    "nccl-coalesced-allreduce+sgd") if world > 1 else None,
                "sequential_ms_per_step": ms_seq,
                "multi_stream_speedup": ms_seq / ms_par,
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_model(args, cfg, rank, world, local):
    """cfg5m: the whole DLRM training step on one GPU (paper_2101_11714_b200/dlrm.py):
    forward + BCE + backward + SGD of both MLPs and all 26 embedding tables."""
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2101_11714_b200 as tt
    from paper_2101_11714_b200.dense import KAGGLE_CARDINALITIES
    from paper_2101_11714_b200.dlrm import DlrmModel

    tables = [(n, n >= 142572, cfg["rank"]) for n in KAGGLE_CARDINALITIES]
    m = DlrmModel(13, cfg["emb"], tables, [512, 256, 64, 16], [512, 256, 1], dot=True, device=local)
    m.init(1)
    B = cfg["bags"]
    rng = np.random.default_rng(7)
    host = {"dense": rng.standard_normal((B, 13)).astype(np.float32),
            "labels": rng.integers(0, 2, B).astype(np.float64),
            "idx": [tt.generate_zipfian_batch(n, cfg["zipf"], 100 + t, B, 1).indices
                    for t, (n, _, _) in enumerate(tables)],
            "off": [np.arange(B + 1, dtype=np.int64) for _ in tables]}
    mb = m.to_device(host)
    pinned = {"dense": torch.from_numpy(host["dense"]).pin_memory(),
              "labels": torch.from_numpy(host["labels"]).pin_memory(),
              "idx": [torch.from_numpy(i).pin_memory() for i in host["idx"]],
              "off": [torch.from_numpy(o).pin_memory() for o in host["off"]]}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        m.train_step(mb, LR)
    for t in m.tables:
        t.check()
    st = m.stream
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    with torch.cuda.stream(st):
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            starts[i].record(st)
            m.train_step(mb, LR)
            ends[i].record(st)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    ms = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))
    # e2e: host minibatch copied in (pinned), loss read back, every step
    h2d = host["dense"].nbytes + host["labels"].nbytes + sum(i.nbytes for i in host["idx"]) + \
        sum(o.nbytes for o in host["off"])
    e2e = []
    for i in range(args.steps):
        flush.fill_(3)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        with torch.cuda.stream(st):
            mb["dense"].copy_(pinned["dense"], non_blocking=True)
            mb["labels"].copy_(pinned["labels"], non_blocking=True)
            for d, h in zip(mb["idx"], pinned["idx"]):
                d.copy_(h, non_blocking=True)
            for d, h in zip(mb["off"], pinned["off"]):
                d.copy_(h, non_blocking=True)
        _, loss = m.train_step(mb, LR)
        float(loss.item())
        e2e.append(time.perf_counter() - t0)
    lookups = len(tables) * B
    if rank == 0:
        e2e_med = float(np.median(e2e))
        line = {"metric": METRIC + " [cfg5m: full DLRM training step]", "value": lookups / (ms / 1e3),
                "unit": "indices/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "samples_per_s": B / (ms / 1e3),
                "data": "synthetic: host Zipf(1.05) streams per table (reference generator), N(0,1) "
                        "dense features, random labels, model init (reference distributions)",
                "config": {"workload": cfg["desc"], "tables": len(tables), "tt_tables": 7,
                           "dense_tables": len(tables) - 7, "lookups_per_step": lookups,
                           "parallelism": "single-gpu",
                           "l2": "flushed (256 MiB write) before every timed step"},
                "e2e": {"value": lookups / e2e_med, "unit": "indices/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": 8, "statistic": "median step time",
                        "path": "DlrmModel.train_step with the minibatch copied from pinned host memory "
                                "and the loss read back"},
                "clocks": clk}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--fast-forward", action="store_true",
                    help="FFMA forward instead of the bit-exact default")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ffma-backward", action="store_true",
                    help="backward head contraction on the FP32 FFMA path instead of tcgen05 3xTF32")
    ap.add_argument("--nccl", action="store_true",
                    help="N>1: NCCL allreduce + SGD kernel instead of the fused peer reduce+SGD")
    ap.add_argument("--profile", action="store_true", help="print per-phase times")
    ap.add_argument("--cta-times", default=None,
                    help="diagnostic: after the timed region, record one step's per-CTA "
                         "timeline of the fast-path kernels into this .npz (needs the "
                         "diagnostics build: make lib-diag, TTGPU_LIB=.../libttgpu_diag.so)")
    ap.add_argument("--cache-partition", action="store_true",
                    help="cfg4: the explicit partition path (eager) instead of the cache fast path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-exec this command under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if cfg.get("collection"):
        run_collection(args, cfg, rank, world, local)
        return
    if cfg.get("model"):
        run_model(args, cfg, rank, world, local)
        return

    import torch

    # test-only overrides: run an N-rank job on ONE GPU (every rank on device 0,
    # gloo for the host-side collectives) to exercise the multi-GPU path where
    # only one GPU exists; never set by the driver
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2101_11714_b200 as tt

    stream = torch.cuda.Stream(device=dev)
    plan = tt.plan_shapes(cfg["rows"], cfg["emb"], len(cfg["rf"]), cfg["rank"], cfg["rf"], cfg["cf"])
    table = tt.TtTable(plan, "bench", np.float32, device=local, stream=stream.cuda_stream)
    table.init_sampled_gaussian(1)
    table.set_exact_forward(not args.fast_forward)
    table.set_tensor_path(not args.ffma_backward)
    idx, off, grad = make_inputs(cfg, 7 + rank, tt)
    L, B, N = len(idx), cfg["bags"], cfg["emb"]
    with torch.cuda.stream(stream):
        d_idx = torch.from_numpy(idx).to(dev)
        d_off = torch.from_numpy(off).to(dev)
        d_grad = torch.from_numpy(grad).to(dev)
        d_out = torch.empty((B, N), dtype=torch.float32, device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream.synchronize()
    ctx = tt.ForwardContext(table)

    cache = None
    if cfg.get("cache"):
        # LFU cache of hot rows (lfu_cache.hpp; model.hpp:195-284): warm-up records
        # frequencies on the same stream, then warmup_finalize admits the top 0.01%
        cache = tt.LfuCache(tt.lfu_cache.default_capacity(cfg["rows"]), cfg["emb"],
                            refresh_period=1 << 30, key_space=cfg["rows"], device=local,
                            stream=stream.cuda_stream)
        cache.set_fast(not args.cache_partition)
    gbuf = None
    if world > 1:
        gptr, gn = table.grad_buffer()

        class _Arr:
            __cuda_array_interface__ = {"shape": (gn,), "typestr": "<f4", "data": (gptr, False),
                                        "version": 3, "strides": None}

        gbuf = torch.as_tensor(_Arr(), device=dev)

    from paper_2101_11714_b200._lib import lib as _L
    import ctypes as _C

    def cache_step():
        st = _L().ttgpu_cache_forward_device(cache.handle, table.handle, ctx.handle,
                                             _C.c_void_p(d_idx.data_ptr()), L,
                                             _C.c_void_p(d_off.data_ptr()), B, None, 0, 1,
                                             _C.c_void_p(d_out.data_ptr()))
        assert st == 0, _L().ttgpu_last_error()
        st = _L().ttgpu_cache_backward_step_device(cache.handle, table.handle, ctx.handle,
                                                   _C.c_void_p(d_grad.data_ptr()), _C.c_double(LR))
        assert st == 0, _L().ttgpu_last_error()

    def step():
        if cache is not None:
            cache_step()
            return
        table.forward_device(ctx, d_idx.data_ptr(), L, d_off.data_ptr(), B, d_out.data_ptr(),
                             save=True)
        if world == 1:
            table.backward_sgd_device(ctx, d_grad.data_ptr(), LR)
        elif reducer is not None:  # one fused kernel: peers' gradients over NVLink + SGD
            table.backward_device(ctx, d_grad.data_ptr())
            reducer.reduce_sgd(LR)
        else:
            table.backward_device(ctx, d_grad.data_ptr())
            with torch.cuda.stream(stream):
                dist.all_reduce(gbuf)
            table.apply_grad(LR)

    # N>1: the fused peer reduce+SGD (ttgpu_peer_reduce_sgd) unless --nccl; it falls
    # back to NCCL if P2P is unavailable, a peer wait times out, or replicas diverge
    reducer, reduce_path = None, ("nccl-allreduce+sgd" if world > 1 else None)
    if world > 1 and not args.nccl and cache is None:
        # every rank must take the same path: agree on P2P reachability first,
        # then on the attach result (PeerReducer's handle exchange is collective)
        def agree(flag):
            t = torch.tensor([1 if flag else 0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return bool(t.item())

        ok = True
        try:
            ok = share or all(torch.cuda.can_device_access_peer(local, j)
                              for j in range(torch.cuda.device_count()) if j != local)
        except Exception:  # noqa: BLE001
            ok = False
        if agree(ok):
            from paper_2101_11714_b200.sharding import PeerReducer

            try:
                reducer = PeerReducer(table)
            except Exception as e:  # noqa: BLE001
                print(f"[bench] peer attach failed ({e}); using NCCL", file=sys.stderr)
                reducer = None
            if agree(reducer is not None):
                reduce_path = "fused-peer-reduce+sgd"
            else:
                reducer = None

    # warm-up (allocates every workspace), validation, then graph capture.  The
    # cache warms on W different batches of the same stream (seeds 7 + rank +
    # 101 * (i + 1)); the timed batch is restored afterwards.
    for i in range(args.warmup):
        if cache is not None:
            widx = make_inputs(cfg, 7 + rank + 101 * (i + 1), tt)[0]
            with torch.cuda.stream(stream):
                d_idx.copy_(torch.from_numpy(widx))
        step()
    if cache is not None:
        with torch.cuda.stream(stream):
            d_idx.copy_(torch.from_numpy(idx))
    table.check()
    if reducer is not None:
        from paper_2101_11714_b200.sharding import replica_checksum

        bad = torch.tensor([1 if reducer.timed_out() else 0], device=dev)
        ck = torch.tensor(replica_checksum([table.core(k) for k in range(plan.tt_dim)]),
                          dtype=torch.int64, device=dev)
        allc = [torch.zeros_like(ck) for _ in range(world)]
        dist.all_gather(allc, ck)
        dist.all_reduce(bad)
        if int(bad.item()) or not all(torch.equal(allc[0], c) for c in allc):
            print("[bench] peer reduce failed validation; using NCCL", file=sys.stderr)
            reducer, reduce_path = None, "nccl-allreduce+sgd (fused path failed validation)"
            for _ in range(2):
                step()
            table.check()
    if cache is not None:
        cache.warmup_finalize(table)
        for _ in range(2):
            step()
        table.check()
    # the cached step is graph-captured on the cache fast path (no host sync);
    # the partition path (--cache-partition) syncs once per forward and runs eagerly
    use_graph = (cache is None or not args.cache_partition) and (world == 1 or reducer is not None)
    kernels_per_step = None
    if use_graph:
        table.graph_begin()
        step()
        kernels_per_step, _ = table.graph_end()
        run = table.graph_launch
        for _ in range(2):
            run()
    elif cache is None and world > 1 and backend == "nccl":
        # NCCL fallback: the whole step, allreduce included, in one torch-managed
        # CUDA graph on the table's stream (NCCL kernels are capturable)
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            run = g.replay
            for _ in range(2):
                run()
            use_graph = True
        except Exception as e:  # noqa: BLE001
            print(f"[bench] NCCL step capture failed ({e}); running eagerly", file=sys.stderr)
            torch.cuda.synchronize()
            run = step
    else:
        run = step
    stream.synchronize()

    if args.profile:
        table.profile(True)
        step()
        phases = table.profile_read()
        table.profile(False)
    else:
        phases = None

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            starts[i].record(stream)
            run()
            ends[i].record(stream)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * L * args.steps / (total_ms / 1e3)

    # Per-kernel times for the roofline: the same step re-captured with CUDA event
    # nodes between its kernels (external event records inside the graph), launched
    # under the same conditions as the timed region (L2 flushed before each step).
    table.profile(True)
    agg = {}
    if use_graph:
        table.graph_begin()
        step()
        table.graph_end()
        for i in range(args.steps):
            flush.fill_(i & 0xff)
            table.graph_launch()
            for name, ms in table.profile_read():
                agg.setdefault(name, []).append(ms)
    else:
        for i in range(3):
            flush.fill_(1)
            step()
            for name, ms in table.profile_read():
                agg.setdefault(name, []).append(ms)
    table.profile(False)
    phase_ms = {k: float(np.mean(v)) for k, v in agg.items()}
    if args.cta_times and rank == 0:
        cta_timeline(args.cta_times, run, flush, stream)
    dom = max(phase_ms, key=phase_ms.get)

    # e2e through the host C ABI: pinned host buffers, copies inside the region
    # page-locked host buffers; the torch tensors that own them stay referenced
    # the e2e section runs on the GPU's NUMA node, its pinned pages allocated there
    affinity0 = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    pinned = [torch.from_numpy(a).pin_memory() for a in (idx, off, grad)]
    pinned.append(torch.empty((B, N), dtype=torch.float32).pin_memory())
    h_idx, h_off, h_grad, h_out = (t.numpy() for t in pinned)
    batch = tt.IndexBatch(h_idx, h_off)
    import ctypes as C

    from paper_2101_11714_b200._lib import lib

    hctx = tt.ForwardContext(table)

    def e2e_step():
        if cache is not None:  # EmbeddingLayer forward / backward / step (model.hpp:195-284)
            st = lib().ttgpu_cache_forward(cache.handle, table.handle, hctx.handle,
                                           h_idx.ctypes.data_as(C.c_void_p), L,
                                           h_off.ctypes.data_as(C.c_void_p), B, None, 0, 1,
                                           h_out.ctypes.data_as(C.c_void_p))
            assert st == 0, lib().ttgpu_last_error()
            st = lib().ttgpu_cache_backward(cache.handle, table.handle, hctx.handle,
                                            h_grad.ctypes.data_as(C.c_void_p), B * N)
            assert st == 0, lib().ttgpu_last_error()
            st = lib().ttgpu_cache_step(cache.handle, table.handle, C.c_double(LR))
            assert st == 0, lib().ttgpu_last_error()
            return
        st = lib().ttgpu_forward(table.handle, h_idx.ctypes.data_as(C.c_void_p), L,
                                 h_off.ctypes.data_as(C.c_void_p), B, None, 0, 2048, 1,
                                 h_out.ctypes.data_as(C.c_void_p), hctx.handle)
        assert st == 0, lib().ttgpu_last_error()
        if world == 1:
            table.backward_sgd(hctx, batch, h_grad, LR)
        else:
            st = lib().ttgpu_backward(table.handle, hctx.handle, L, B,
                                      h_grad.ctypes.data_as(C.c_void_p), B * N, None)
            assert st == 0
            if reducer is not None:
                reducer.reduce_sgd(LR)
            else:
                with torch.cuda.stream(stream):
                    dist.all_reduce(gbuf)
                table.apply_grad(LR)
            table.sync()

    for _ in range(3):
        e2e_step()
    if dist:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(2)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e2e_step()
        e2e_times.append(time.perf_counter() - t0)
    # per-step median (host-side timing sees OS / PCIe jitter; one slow step
    # should not define the number), max over ranks
    e2e_med = float(np.median(e2e_times))
    e2e_mean = float(np.mean(e2e_times))
    if dist:
        t = torch.tensor([e2e_med, e2e_mean], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_med, e2e_mean = float(t[0].item()), float(t[1].item())
    e2e_value = world * L / e2e_med
    # the PCIe rates this box gives the step's own pinned buffers (grad_out
    # H2D, output D2H), CUDA events, measured right after the e2e steps: they
    # explain e2e differences between runs.  The H2D rate of one and the same
    # pinned buffer varies over time on these shared hosts (51 GB/s when
    # allocated, 11-41 GB/s a few seconds later, single-NUMA-node VMs), while
    # D2H stays at ~52 GB/s
    pcie = {}
    try:
        dbuf = torch.empty(h_out.size, dtype=torch.float32, device=dev)
        for name, cp in (("h2d", lambda: dbuf.copy_(pinned[2].view(-1), non_blocking=True)),
                         ("d2h", lambda: pinned[3].view(-1).copy_(dbuf, non_blocking=True))):
            best = 1e9
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                cp()
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e-3)
            pcie[name + "_GBs"] = h_out.nbytes / best / 1e9
        del dbuf
    except Exception:  # noqa: BLE001 - diagnostic only
        pcie = {}
    os.sched_setaffinity(0, affinity0)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(dev)
    fp32_peak_tf = props.multi_processor_count * 128 * 2 * sm_mhz * 1e6 / 1e12
    fp32_src = (f"derived: {props.multi_processor_count} SMs x 128 FFMA/clk x 2 x {sm_mhz:.0f} "
                f"MHz (no measured FP32 figure)")
    try:  # measured by tools/ffma_peak.cu on a B200 of this pool
        fp = json.load(open(os.path.join(ROOT, "profiles", "fp32_peak.json")))
        fp32_peak_tf = float(fp["fp32_tflops"])
        fp32_src = "profiles/fp32_peak.json (measured, tools/ffma_peak.cu: " + fp["how"] + ")"
    except Exception:  # noqa: BLE001
        pass
    params = plan.parameter_count()
    ranks = plan.ranks
    f_lookup = flops_per_lookup(cfg["rf"], cfg["cf"], ranks)
    step_flops = f_lookup * L + 2 * params
    step_bytes = bytes_per_step(L, B, N, params)
    step_s = ms_per_step / 1e3
    # dominant kernel: algorithmic work per launch / its event-timed duration
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernels.json")))
    except Exception:  # noqa: BLE001
        ncu = {}
    work = kernel_work(dom, cfg["rf"], cfg["cf"], ranks, L, B, N, params)
    dom_s = phase_ms[dom] / 1e3
    ncu_dom = ncu.get(args.config, {}).get(dom, {})
    traffic = ncu_dom.get("dram_bytes")
    executed = None
    if ncu_dom.get("us"):
        # ncu-executed FP32 work of the same kernel (dedup makes
        # the algorithmic rate exceed what the FMA pipe actually ran):
        # 2 flops per FFMA lane-op, 4 per FFMA2 thread instruction, over the ncu
        # (cold, serialised) duration and over this run's event duration
        ex_fl = 2.0 * ncu_dom.get("ffma_thread_inst", 0.0) + 4.0 * ncu_dom.get("ffma2_thread_inst", 0.0)
        executed = {"flops_per_launch": ex_fl,
                    "tflops_ncu_time": ex_fl / (ncu_dom["us"] * 1e-6) / 1e12,
                    "frac_ncu_time": ex_fl / (ncu_dom["us"] * 1e-6) / 1e12 / fp32_peak_tf,
                    "tflops_event_time": ex_fl / dom_s / 1e12,
                    "frac_event_time": ex_fl / dom_s / 1e12 / fp32_peak_tf,
                    "source": "profiles/ncu_kernels.json (sm__sass_thread_inst_executed_op_ffma"
                              "/ffma2 counts of one ncu --set full capture)"}
    if work:
        fl, by = work
        roofline = {"bound": "fp32", "kernel": dom, "achieved": fl / dom_s / 1e12,
                    "peak": fp32_peak_tf, "unit": "TFLOP/s", "frac": fl / dom_s / 1e12 / fp32_peak_tf,
                    "traffic": traffic, "flops_per_launch": fl, "launch_ms": phase_ms[dom],
                    "executed": executed,
                    "peak_source": fp32_src,
                    "note": "FP32 CUDA-core FFMA chain (no tensor-core path: the reference's fp32 "
                            "arithmetic order is kept); algorithmic flops, reference chain without "
                            "dedup; traffic = ncu dram read+write bytes per launch "
                            "(profiles/ncu_kernels.json)"}
        roofline_hbm = {"bound": "hbm", "kernel": dom, "achieved": by / dom_s / 1e9,
                        "peak": hbm_peak, "unit": "GB/s", "frac": by / dom_s / 1e9 / hbm_peak,
                        "traffic": traffic, "bytes_per_launch": by,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    else:
        roofline = {"bound": "fp32", "kernel": "whole step", "achieved": step_flops / step_s / 1e12,
                    "peak": fp32_peak_tf, "unit": "TFLOP/s",
                    "frac": step_flops / step_s / 1e12 / fp32_peak_tf, "traffic": None,
                    "peak_source": fp32_src,
                    "note": "algorithmic flops of the reference chain per lookup (no dedup); the "
                            "pair dedup executes fewer, so frac can exceed 1 (generic path: no "
                            "single dominant kernel)"}
        roofline_hbm = {"bound": "hbm", "kernel": "whole step", "achieved": step_bytes / step_s / 1e9,
                        "peak": hbm_peak, "unit": "GB/s",
                        "frac": step_bytes / step_s / 1e9 / hbm_peak, "traffic": None,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    line = {
        "metric": METRIC, "value": value, "unit": "indices/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference Zipf/uniform index streams (same bytes as data.cpp), "
                "sampled-Gaussian cores (initializer.hpp), N(0,1) grad_out",
        "config": workload_config(cfg, world),
        "execution": {"device": "B200", "forward": "ffma" if args.fast_forward else
                      "exact (bit-identical to reference)", "graph": use_graph,
                      "backward_head": "ffma" if args.ffma_backward else
                      "tcgen05 3xTF32 where eligible (cfg3 shape), else ffma",
                      "gradient_reduce": reduce_path},
        "gpu_launches": (kernels_per_step * args.steps) if kernels_per_step else None,
        "cache": ({"capacity": cache.capacity(), "hit_rate": cache.hit_rate(),
                   "path": ("partition (record_and_partition + forward_bags(part.tt) + combine, eager)"
                            if args.cache_partition else
                            "fast (cache probed inside f3_gsort; one CUDA graph per step)")}
                  if cache is not None else None),
        "clocks": clk,
        "roofline": roofline,
        "roofline_hbm": roofline_hbm,
        "roofline_step": {
            "bound": "fp32-ffma", "achieved": step_flops / step_s / 1e12, "peak": fp32_peak_tf,
            "unit": "TFLOP/s", "frac": step_flops / step_s / 1e12 / fp32_peak_tf,
            "flops_per_lookup": f_lookup, "hbm_GBs": step_bytes / step_s / 1e9,
            "hbm_frac": step_bytes / step_s / 1e9 / hbm_peak,
            "scope": "whole timed step (all kernels), algorithmic reference-chain flops (no dedup); "
                     "hbm bytes = 16B/lookup idx + 16B/bag offsets + 8N B/bag output+grad + "
                     "8B/param cores", "peak_source": fp32_src},
        "phases_ms": phase_ms, "dominant_phase": dom,
        "e2e": {"value": e2e_value, "unit": "indices/s",
                "h2d_bytes_per_step": int(idx.nbytes + off.nbytes + grad.nbytes),
                "d2h_bytes_per_step": int(h_out.nbytes),
                "path": "ttgpu_forward + ttgpu_backward_sgd (host C ABI, pinned buffers)",
                "statistic": "median step time over the timed steps",
                "ms_per_step_median": e2e_med * 1e3, "ms_per_step_mean": e2e_mean * 1e3,
                "pcie_best_GBs": pcie,
                "host_cpus": (f"GPU-local NUMA node ({len(local_cpus)} CPUs, sysfs local_cpulist)"
                              if local_cpus else "process default")},
    }
    if not args.no_cpu_baseline:
        cb = cpu_reference_time(cfg, idx, off, grad, budget_s=10.0)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                   "threads_1", "serial_ref") if k in cb}
    if phases:
        line["profile_single_step"] = phases
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
