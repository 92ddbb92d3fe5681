"""GPU: the DLRM training step against the reference's own
DlrmModel (model.hpp:355-538) and SyntheticDataSource (data.cpp) from
oracle/_ref: the reference's initial parameters are copied onto the GPU model,
both train on the same minibatches, and logits, losses and every parameter
(MLP weights, TT cores, uncompressed tables) must agree within the fp32
tolerance after several steps -- in Dot and Concat interaction, pooling
factors 1 and 2, with the tables' SGD fused into their backward or applied
by step()."""
import numpy as np
import pytest

from helpers import scaled_max_err
from pyoracle import RefImpl, RefModel, RefSource

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _copy(rm, gm, tables, nbottom, ntop):
    for i in range(nbottom):
        gm.set_mlp("bottom", i, rm.param(0, i), rm.param(1, i))
    for i in range(ntop):
        gm.set_mlp("top", i, rm.param(2, i), rm.param(3, i))
    for t, (rows, use_tt, rank) in enumerate(tables):
        if use_tt:
            for k in range(3):
                gm.set_tt_core(t, k, rm.param(4, t, k))
        else:
            gm.set_dense_table(t, rm.param(5, t))


def _compare(rm, gm, tables, nbottom, ntop, what):
    for i in range(nbottom):
        w, b = gm.mlp_params("bottom", i)
        assert scaled_max_err(w, rm.param(0, i)) <= TOL, f"{what}: bottom.w{i}"
        assert scaled_max_err(b, rm.param(1, i)) <= TOL, f"{what}: bottom.b{i}"
    for i in range(ntop):
        w, b = gm.mlp_params("top", i)
        assert scaled_max_err(w, rm.param(2, i)) <= TOL, f"{what}: top.w{i}"
        assert scaled_max_err(b, rm.param(3, i)) <= TOL, f"{what}: top.b{i}"
    for t, (rows, use_tt, rank) in enumerate(tables):
        if use_tt:
            for k in range(3):
                assert scaled_max_err(gm.tt_core(t, k), rm.param(4, t, k)) <= TOL, f"{what}: table{t} core{k}"
        else:
            assert scaled_max_err(gm.dense_table(t).ravel(), rm.param(5, t)) <= TOL, f"{what}: table{t}"


@pytest.mark.parametrize("dot,pf", [(True, 1), (False, 2)])
def test_dlrm_steps_match_reference_model(dot, pf):
    from paper_2101_11714_b200.dlrm import DlrmModel

    ref = RefImpl()
    tables = [(20000, True, 8), (800, False, 0), (50000, True, 16), (300, False, 0), (4000, True, 4)]
    bottom, top = [32, 16], [8, 1]
    rm = RefModel(ref, 3, 16, tables, bottom, top, dot=dot)
    rm.init(5)
    gm = DlrmModel(3, 16, tables, bottom, top, dot=dot)
    _copy(rm, gm, tables, len(bottom), len(top))
    _compare(rm, gm, tables, len(bottom), len(top), "copied")
    src = RefSource(ref, 3, [t[0] for t in tables], 1.05, 256, pf, 7)
    for it in range(5):
        mb = src.next(it)
        want_logits, want_loss = rm.step(mb, 0.05)
        logits, loss = gm.train_step(gm.to_device(mb), 0.05, fused=it % 2 == 0)
        gm.stream.synchronize()
        got = logits.cpu().numpy()
        if it == 0:  # same parameters: only the MLP GEMM summation order differs
            assert scaled_max_err(got, want_logits) <= 1e-5
        assert scaled_max_err(got, want_logits) <= TOL, f"step {it} logits"
        assert abs(float(loss.item()) - want_loss) <= TOL * max(1.0, abs(want_loss)), f"step {it} loss"
    _compare(rm, gm, tables, len(bottom), len(top), "after 5 steps")


def test_dlrm_init_shapes_and_loss_decreases():
    """A fresh GPU model (its own init) learns the synthetic teacher: the BCE
    loss of the reference's SyntheticDataSource falls over 40 steps."""
    from paper_2101_11714_b200.dlrm import DlrmModel

    ref = RefImpl()
    tables = [(30000, True, 16), (500, False, 0), (90000, True, 16)]
    gm = DlrmModel(4, 16, tables, [32, 16], [16, 1])
    gm.init(3)
    src = RefSource(ref, 4, [t[0] for t in tables], 1.05, 512, 1, 11)
    losses = []
    for it in range(40):
        _, loss = gm.train_step(gm.to_device(src.next(it)), 0.1)
        losses.append(float(loss.item()))
    assert np.mean(losses[-8:]) < np.mean(losses[:8]) - 0.01, losses
