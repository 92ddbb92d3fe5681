"""bench_pooling on the GPU: the reference's timing sweep
(bench.hpp:46-159, `ttrec bench`, tools/ttrec.cpp:249-275) with the same
configuration fields, the same inputs and the same CSV schema, so its trend
checks (acceptance criterion 7, acceptance.cpp:647-688) run on GPU numbers.

Inputs are the reference's exactly: plan_shapes(rows, emb_dim, tt_dim, rank),
init_tt_cores(sampled_gaussian, seed), per (rank, pooling) a batch of `bags`
bags drawn with Rng::derive(seed, rank << 20 ^ pooling).uniform_int(0, rows),
all-ones grad_output.  Timing: each rep times `inner` forward calls (no
saved state) and `inner` backward calls with CUDA events on the table's
stream, inputs resident in device memory; per-lookup / per-sample values are
the median of group means (median_of_means, bench.hpp:16-44).  The serial
columns are the reference's single-thread CPU path and are reported as 0 here
(`--no-serial` in the reference CLI).

    python -m paper_2101_11714_b200.bench_pooling --rows 50000 --ranks 4 64 \\
        --poolings 1 10 100 --bags 8 --reps 24 --out -
"""
from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass, field
from typing import List

import numpy as np

from .ttrec import ForwardContext, TtTable, derived_uniform_indices, plan_shapes

HEADER = ("pooling,rank,fwd_us_per_sample,bwd_us_per_sample,fwd_us_per_lookup,"
          "bwd_us_per_lookup,serial_fwd_us_per_lookup,serial_bwd_us_per_lookup,"
          "fwd_spread_us,bwd_spread_us")


@dataclass
class BenchConfig:
    """bench.hpp:55-67 (same defaults)."""
    rows: int = 100000
    emb_dim: int = 16
    tt_dim: int = 3
    ranks: List[int] = field(default_factory=lambda: [8, 16, 32, 64])
    poolings: List[int] = field(default_factory=lambda: [1, 10, 100])
    bags: int = 256
    reps: int = 30
    micro_batch: int = 2048
    seed: int = 0
    include_serial: bool = False
    target_lookups_per_rep: int = 8192


@dataclass
class BenchRow:
    pooling: int
    rank: int
    fwd_us_per_sample: float = 0.0
    bwd_us_per_sample: float = 0.0
    fwd_us_per_lookup: float = 0.0
    bwd_us_per_lookup: float = 0.0
    serial_fwd_us_per_lookup: float = 0.0
    serial_bwd_us_per_lookup: float = 0.0
    fwd_spread_us: float = 0.0
    bwd_spread_us: float = 0.0

    def csv(self) -> str:
        return "%d,%d,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f" % (
            self.pooling, self.rank, self.fwd_us_per_sample, self.bwd_us_per_sample,
            self.fwd_us_per_lookup, self.bwd_us_per_lookup, self.serial_fwd_us_per_lookup,
            self.serial_bwd_us_per_lookup, self.fwd_spread_us, self.bwd_spread_us)


def median_of_means(samples, groups: int = 5):
    """bench.hpp:16-44: median of per-group means and the sd of the means."""
    if not samples:
        return 0.0, 0.0
    groups = max(1, min(groups, len(samples)))
    per = len(samples) // groups
    means = []
    for g in range(groups):
        lo = g * per
        hi = len(samples) if g + 1 == groups else lo + per
        means.append(float(np.mean(samples[lo:hi])))
    means.sort()
    v = means[len(means) // 2]
    if len(means) % 2 == 0:
        v = 0.5 * (v + means[len(means) // 2 - 1])
    m = float(np.mean(means))
    return v, float(np.sqrt(np.sum((np.array(means) - m) ** 2) / len(means)))


def bench_pooling(cfg: BenchConfig, device: int = 0) -> List[BenchRow]:
    import torch

    if cfg.reps < 1 or cfg.bags < 1:
        raise ValueError("reps and bags must be positive")
    dev = torch.device("cuda", device)
    stream = torch.cuda.Stream(device=dev)
    out: List[BenchRow] = []
    for rank in cfg.ranks:
        plan = plan_shapes(cfg.rows, cfg.emb_dim, cfg.tt_dim, rank)
        table = TtTable(plan, f"bench-r{rank}", np.float32, device=device,
                        stream=stream.cuda_stream)
        table.init_sampled_gaussian(cfg.seed)
        ctx = ForwardContext(table)
        for pooling in cfg.poolings:
            L = cfg.bags * pooling
            idx = derived_uniform_indices(cfg.rows, cfg.seed, (rank << 20) ^ pooling, L)
            off = np.arange(0, L + 1, pooling, dtype=np.int64)
            with torch.cuda.stream(stream):
                d_idx = torch.from_numpy(idx).to(dev)
                d_off = torch.from_numpy(off).to(dev)
                d_grad = torch.ones((cfg.bags, cfg.emb_dim), dtype=torch.float32, device=dev)
                d_out = torch.empty((cfg.bags, cfg.emb_dim), dtype=torch.float32, device=dev)
            stream.synchronize()
            inner = max(1, cfg.target_lookups_per_rep // max(L, 1))

            def fwd(save):
                table.forward_device(ctx, d_idx.data_ptr(), L, d_off.data_ptr(), cfg.bags,
                                     d_out.data_ptr(), save=save)

            fwd(True)  # warm-up outside timing
            table.backward_device(ctx, d_grad.data_ptr())
            table.check()
            fwd_us, bwd_us = [], []
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            with torch.cuda.stream(stream):
                for _ in range(cfg.reps):
                    ev[0].record(stream)
                    for _ in range(inner):
                        fwd(False)
                    ev[1].record(stream)
                    fwd(True)
                    ev[2].record(stream)
                    for _ in range(inner):
                        table.backward_device(ctx, d_grad.data_ptr())
                    ev[3].record(stream)
                    stream.synchronize()
                    fwd_us.append(ev[0].elapsed_time(ev[1]) * 1e3 / inner)
                    bwd_us.append(ev[2].elapsed_time(ev[3]) * 1e3 / inner)
            table.check()
            f, fs = median_of_means(fwd_us)
            b, bs = median_of_means(bwd_us)
            out.append(BenchRow(pooling, rank, f / cfg.bags, b / cfg.bags, f / L, b / L, 0.0, 0.0,
                                fs / L, bs / L))
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description="Embedding kernel timing sweep (GPU)")
    c = BenchConfig()
    ap.add_argument("--rows", type=int, default=c.rows)
    ap.add_argument("--emb-dim", type=int, default=c.emb_dim)
    ap.add_argument("--tt-dim", type=int, default=c.tt_dim)
    ap.add_argument("--ranks", type=int, nargs="+", default=c.ranks)
    ap.add_argument("--poolings", "--pooling", type=int, nargs="+", default=c.poolings)
    ap.add_argument("--bags", type=int, default=c.bags)
    ap.add_argument("--reps", type=int, default=c.reps)
    ap.add_argument("--micro-batch", type=int, default=c.micro_batch)
    ap.add_argument("--seed", type=int, default=c.seed)
    ap.add_argument("--target-lookups", type=int, default=c.target_lookups_per_rep)
    ap.add_argument("--out", default="-")
    a = ap.parse_args(argv)
    cfg = BenchConfig(a.rows, a.emb_dim, a.tt_dim, a.ranks, a.poolings, a.bags, a.reps,
                      a.micro_batch, a.seed, False, a.target_lookups)
    rows = bench_pooling(cfg)
    f = sys.stdout if a.out == "-" else open(a.out, "w")
    f.write(HEADER + "\n")
    for r in rows:
        f.write(r.csv() + "\n")
    if f is not sys.stdout:
        f.close()


if __name__ == "__main__":
    main()
