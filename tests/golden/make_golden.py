"""Regenerate tests/golden/* from the REFERENCE implementation itself.

Run (only where /root/reference exists, after `make -C oracle`):
    python tests/golden/make_golden.py

Every number in the fixtures comes from oracle/_ref/libttref.so, i.e. the
unmodified reference C++ sources compiled in place: its plan_shapes,
decompose_index, Rng / ZipfianSampler / init_tt_cores streams (libstdc++
specific, hence generated once and committed), ref::forward_bags,
ref::backward_bags, sgd_step, lookup_row and LfuCache.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import RefCache, RefImpl  # noqa: E402

# tools/ttrec.cpp:29-33 kRefTables (Table 2 of the paper)
REF_TABLES = [
    (10131227, [200, 220, 250]), (8351593, [200, 200, 209]), (7046547, [200, 200, 200]),
    (5461306, [166, 175, 188]), (2202608, [125, 130, 136]), (286181, [53, 72, 75]),
    (142572, [50, 52, 55]),
]


def plans(ref):
    rows = []
    for n, rf in REF_TABLES:
        for rank in (16, 32, 64):
            p, info = ref.plan_shapes(n, 16, 3, rank, rf, [2, 2, 4])
            rows.append(dict(rows=n, rank=rank, row_factors=p.row_factors,
                             col_factors=p.col_factors, ranks=p.ranks, **info))
    auto = []
    for n, emb, d, rank in [(1000000, 16, 3, 16), (10131227, 16, 3, 32), (40000000, 64, 3, 64),
                            (500, 16, 3, 8), (40, 16, 3, 2), (300, 16, 4, 4), (64, 8, 2, 2),
                            (4096, 8, 2, 4), (20000, 8, 2, 4), (5000, 8, 3, 4), (1, 1, 2, 1)]:
        try:
            p, info = ref.plan_shapes(n, emb, d, rank)
            auto.append(dict(rows=n, emb=emb, d=d, rank=rank, row_factors=p.row_factors,
                             col_factors=p.col_factors, ranks=p.ranks, **info))
        except Exception as e:  # noqa: BLE001
            auto.append(dict(rows=n, emb=emb, d=d, rank=rank, error=str(e)))
    decode = []
    for flat in [10131226, 0, 249, 250, 55000, 10999999]:
        decode.append(dict(flat=flat, digits=[int(x) for x in
                                              ref.decompose_index(flat, [200, 220, 250])]))
    return dict(table2=rows, auto=auto, decode=decode)


def small_cases(ref):
    """Random small plans (d 2..4, ranks 1..8) x {f32, f64} x {Sum, Mean} x weights."""
    out = {}
    rng = np.random.default_rng(1234)
    n = 0
    for trial in range(16):
        d = int(rng.integers(2, 5))
        rank = int(rng.integers(1, 9))
        rows = int(rng.integers(10, 300))
        cols = [2, 2, 2, 2] if d == 4 else None
        p, _ = ref.plan_shapes(rows, 16, d, rank, None, cols)
        dt = np.float64 if trial % 4 == 3 else np.float32
        t = ref.table(p, dt, f"golden{trial}")
        t.fill_normal(500 + trial)
        cores = t.get_cores()
        idx, off, w = ref.random_batch(900 + trial, rows, int(rng.integers(1, 24)), 0, 8,
                                       trial % 2 == 1)
        pooling = 1 if trial % 3 == 0 else 0
        B = len(off) - 1
        grad = ref.normal(700 + trial, B * 16).astype(dt).reshape(B, 16)
        fwd = t.serial_forward(idx, off, w, pooling)
        grads = t.serial_backward(idx, off, grad, w, pooling)
        t.sgd(grads, 0.05)
        after = t.get_cores()
        pre = f"c{n}_"
        out[pre + "plan"] = np.array([p.num_rows, p.emb_dim, p.tt_dim, pooling,
                                      1 if dt == np.float64 else 0], np.int64)
        out[pre + "rf"] = np.array(p.row_factors, np.int64)
        out[pre + "cf"] = np.array(p.col_factors, np.int64)
        out[pre + "rk"] = np.array(p.ranks, np.int64)
        for k in range(d):
            out[pre + f"core{k}"] = cores[k]
            out[pre + f"grad{k}"] = grads[k]
            out[pre + f"after{k}"] = after[k]
        out[pre + "idx"] = idx
        out[pre + "off"] = off
        if w is not None:
            out[pre + "w"] = w
        out[pre + "grad_out"] = grad
        out[pre + "fwd"] = fwd
        n += 1
    out["count"] = np.array([n])
    return out


def cfg1(ref):
    """BASELINE configs[0]: 1M rows (100x100x100), dim 16 (2x2x4), R=16, 4096 x 1 uniform."""
    p, _ = ref.plan_shapes(1000000, 16, 3, 16, [100, 100, 100], [2, 2, 4])
    t = ref.table(p, np.float32, "cfg1")
    t.init_sampled_gaussian(1)
    cores = t.get_cores()
    idx = ref.uniform_int(3, 0, 1000000, 4096)
    off = np.arange(4097, dtype=np.int64)
    grad = ref.normal(2, 4096 * 16).astype(np.float32).reshape(4096, 16)
    out, ctx = t.forward(idx, off, save=True, keep_ctx=True)
    grads = t.backward(ctx, idx, off, grad)
    t.ctx_destroy(ctx)
    d = dict(idx=idx, off=off, grad_out=grad, fwd=out,
             rows=np.array([0, 1, 999999, 123456], np.int64))
    d["lookup"] = np.stack([t.lookup_row(r) for r in d["rows"]])
    for k in range(3):
        d[f"core{k}"] = cores[k]
        d[f"grad{k}"] = grads[k]
    return d


def cache_case(ref):
    """LfuCache admission / routing on a Zipf stream (acceptance.cpp:415-470 style)."""
    rows, cap, emb = 20000, 128, 8
    p, _ = ref.plan_shapes(rows, emb, 2, 4)
    t = ref.table(p, np.float32, "cache")
    t.init_sampled_gaussian(11)
    cache = RefCache(ref, cap, emb)
    stream_idx, stream_off = [], []
    for s in range(40):
        idx, off = ref.zipf_batch(rows, 1.05, 100 + s, 250, 2)
        cache.record_and_partition(idx, off)
        stream_idx.append(idx)
        stream_off.append(off)
    cache.warmup_finalize(t)
    hot = cache.hot_rows()
    slots = np.array([cache.slot_of(r) for r in hot], np.int64)
    values = np.stack([cache.row_values(s) for s in slots])
    idx, off, w = ref.random_batch(77, rows, 64, 0, 4, True)
    part = cache.record_and_partition(idx, off, w, 1)
    d = dict(stream_idx=np.stack(stream_idx), stream_off=np.stack(stream_off), hot=hot,
             slots=slots, values=values, probe_idx=idx, probe_off=off, probe_w=w,
             rf=np.array(p.row_factors, np.int64), cf=np.array(p.col_factors, np.int64),
             rk=np.array(p.ranks, np.int64), hit_rate=np.array([cache.hit_rate()]),
             top_k=cache.top_k(cap),
             freq_hot=np.array([cache.freq(int(r)) for r in hot], np.int64))
    for k, c in enumerate(t.get_cores()):
        d[f"core{k}"] = c
    for key, v in part.items():
        d["part_" + key] = v
    return d


CACHE_TRAIN = dict(rows=20000, cap=48, lr=0.002, steps=14, finalize_after=5, refresh_after=10,
                   bags=128, pf=3, zipf=1.2)


def cache_train_batches(ref, plan, c=CACHE_TRAIN):
    """Per-step (idx, off, weights, pooling, grad) of the cached-layer trajectory."""
    out = []
    for s in range(c["steps"]):
        idx, off = ref.zipf_batch(c["rows"], c["zipf"], 500 + s, c["bags"], c["pf"])
        w = (0.5 + 0.5 * np.abs(ref.normal(700 + s, len(idx)))) if s % 2 else None
        pooling = 1 if s % 3 == 2 else 0
        grad = ref.normal(900 + s, c["bags"] * plan.emb_dim).astype(np.float32)
        out.append((idx, off, w, pooling, grad))
    return out


def cache_train(ref, plan, c=CACHE_TRAIN):
    """EmbeddingLayer with a TT table + LFU cache (model.hpp:195-284) trained on a
    Zipf(1.2) multi-hot stream: warm-up steps, warmup_finalize, cached training
    steps, one refresh.  Records every step's output, the cache counters, the
    admitted rows/values, the drift and the final cores."""
    layer = ref.layer(plan, c["cap"], "cached")
    layer.init(5)
    d = dict(rf=np.array(plan.row_factors, np.int64), cf=np.array(plan.col_factors, np.int64),
             rk=np.array(plan.ranks, np.int64))
    for k in range(len(plan.row_factors)):
        d[f"init_core{k}"] = layer.core(k)
    outs, acc, hits = [], [], []
    for s, (idx, off, w, pooling, grad) in enumerate(cache_train_batches(ref, plan, c)):
        d[f"idx{s}"], d[f"off{s}"], d[f"grad{s}"] = idx, off, grad
        if w is not None:
            d[f"w{s}"] = w
        outs.append(layer.forward(idx, off, w, pooling))
        layer.backward(idx, off, grad, w, pooling)
        layer.step(c["lr"])
        info = layer.cache_info()
        acc.append(info["accesses"])
        hits.append(info["hits"])
        if s == c["finalize_after"]:
            layer.finalize_warmup()
            d["fin_rows"], d["fin_values"] = layer.cache_rows(c["cap"])
        if s == c["refresh_after"]:
            d["drift"] = np.array([layer.refresh()])
            d["ref_rows"], d["ref_values"] = layer.cache_rows(c["cap"])
    d["out"] = np.stack(outs)
    d["accesses"] = np.array(acc, np.int64)
    d["hits"] = np.array(hits, np.int64)
    d["end_rows"], d["end_values"] = layer.cache_rows(c["cap"])
    d["freq_end_rows"] = np.array([layer.freq(int(r)) for r in d["end_rows"]], np.int64)
    for k in range(len(plan.row_factors)):
        d[f"core{k}"] = layer.core(k)
    for key, v in d.items():
        assert np.all(np.isfinite(v)), f"cache_train: non-finite {key}"
    return d


def zipf_stream(ref):
    """First 4096 draws of the cfg2 index stream (Zipf 1.05 over 10,131,227 rows, seed 7)."""
    idx, off = ref.zipf_batch(10131227, 1.05, 7, 4096, 1)
    return dict(idx=idx, off=off)


CKPT_PLANS = {  # name -> (Plan args, dtype)
    "emb0": ((5000, 16, [10, 20, 25], [2, 2, 4], [1, 6, 5, 1]), np.float32),
    "emb1": ((300, 8, [15, 20], [2, 4], [1, 3, 1]), np.float64),
}


def checkpoint_golden(ref):
    """A TTRECV01 file written by the reference's Checkpoint::save: two tables
    (f32 3-core with init_tt_cores(sampled_gaussian, 3); f64 2-core with the
    test helpers' fill_cores(seed 5)) and one f32 array."""
    from pyoracle import Plan

    t0 = ref.table(Plan(*CKPT_PLANS["emb0"][0]), CKPT_PLANS["emb0"][1], "emb0")
    t0.init_sampled_gaussian(3)
    t1 = ref.table(Plan(*CKPT_PLANS["emb1"][0]), CKPT_PLANS["emb1"][1], "emb1")
    t1.fill_normal(5, 0.5)
    w = ref.normal(11, 37).astype(np.float32)
    ref.checkpoint_save(os.path.join(HERE, "ckpt_ref.ttrec"), [t0, t1], [("dense.w", w)])


def main():
    ref = RefImpl()
    if len(sys.argv) > 1 and sys.argv[1] == "ckpt":
        checkpoint_golden(ref)
        return
    checkpoint_golden(ref)
    with open(os.path.join(HERE, "plans.json"), "w") as f:
        json.dump(plans(ref), f, indent=1)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **small_cases(ref))
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), **cfg1(ref))
    np.savez_compressed(os.path.join(HERE, "cache_case.npz"), **cache_case(ref))
    np.savez_compressed(os.path.join(HERE, "zipf_stream.npz"), **zipf_stream(ref))
    p3, _ = ref.plan_shapes(CACHE_TRAIN["rows"], 16, 3, 16, [25, 28, 30], [2, 2, 4])
    np.savez_compressed(os.path.join(HERE, "cache_train3.npz"), **cache_train(ref, p3))
    p2, _ = ref.plan_shapes(CACHE_TRAIN["rows"], 8, 2, 4)
    np.savez_compressed(os.path.join(HERE, "cache_train2.npz"), **cache_train(ref, p2))
    for fn in sorted(os.listdir(HERE)):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))


if __name__ == "__main__":
    main()
