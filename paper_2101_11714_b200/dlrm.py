"""The DLRM training step on the GPU (reference
`DlrmModel`, model.hpp:355-538, and one iteration of `train()`, :566-573).

The embedding tables are this package's operators: a TT table is a `TtTable`
driven through the C ABI (forward_bags(save) + backward_bags, then sgd_step;
or the fused backward + SGD in `train_step`), an uncompressed table a
`DenseEmbeddingBags` group.  The two MLPs, the feature interaction and the
BCE loss are the model's plumbing around them and run as plain fp32 torch ops
on the same stream (TF32 disabled: the reference is fp32).  Everything stays
on the device; `train_step` reads back the loss only.

Shapes and semantics follow the reference:
  * `Mlp`: layers (out x in) with bias, ReLU between layers, none after the
    last (mlp.hpp:14-130);
  * interaction Dot: [bottom output | f_i·f_j for i < j] in (i, j)
    row-major order, or Concat of all features (model.hpp:402-436);
  * `bce_with_logits`: mean BCE, dlogits = (sigmoid(x) - y) / batch, in
    float64 (model.hpp:82-103);
  * `step(lr)`: w -= T(lr)·gw for both MLPs, gradients zeroed, then every
    table's step (model.hpp:476-482).

Parameters can be loaded from (and compared with) the reference model through
the `set_*` / getter methods; `init` draws fresh parameters with the
reference's distributions (not its RNG streams).

Data parallel (`group` with world > 1): every rank trains its
shard of the batch with replicated parameters.  dlogits are scaled by the
GLOBAL batch size, every gradient -- both MLPs, every TT table's dense core
gradient, every uncompressed table's row gradient -- goes into ONE flat buffer
and one allreduce(SUM), then the identical SGD on every replica: the update of
the full-batch step."""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .dense import DenseEmbeddingBags
from .ttrec import ForwardContext, TtTable, plan_shapes


class DlrmModel:
    def __init__(self, dense_features: int, emb_dim: int, tables: Sequence[Tuple[int, bool, int]],
                 bottom: Sequence[int], top: Sequence[int], dot: bool = True, device: int = 0,
                 group=None, data_parallel: bool = True):
        """tables: (rows, use_tt, rank) per categorical feature (TableConfig,
        model.hpp:23-31; a TT table gets plan_shapes(rows, emb_dim, 3, rank))."""
        import torch

        if not tables:
            raise ValueError("need at least one embedding table")
        if not bottom or bottom[-1] != emb_dim:
            raise ValueError("bottom MLP must end at emb_dim")
        if not top or top[-1] != 1:
            raise ValueError("top MLP must end in a single logit")
        torch.backends.cuda.matmul.allow_tf32 = False
        self.torch = torch
        import torch.distributed as dist

        self.group = group
        self.world = (dist.get_world_size(group)
                      if data_parallel and dist.is_available() and dist.is_initialized() else 1)
        self.dev = torch.device("cuda", device)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.df, self.emb, self.dot = int(dense_features), int(emb_dim), bool(dot)
        self.nt = len(tables)
        f = self.nt + 1
        self.zdim = self.emb + f * (f - 1) // 2 if self.dot else f * self.emb
        self.iu = torch.triu_indices(f, f, offset=1, device=self.dev)

        def mlp(inp, dims):
            layers, i = [], inp
            for o in dims:
                layers.append({"w": torch.zeros((o, i), device=self.dev),
                               "b": torch.zeros(o, device=self.dev),
                               "gw": torch.zeros((o, i), device=self.dev),
                               "gb": torch.zeros(o, device=self.dev)})
                i = o
            return layers

        self.bottom = mlp(self.df, list(bottom))
        self.top = mlp(self.zdim, list(top))
        self.tables: List[object] = []
        self.kinds: List[str] = []
        self.ctx: List[object] = []
        for t, (rows, use_tt, rank) in enumerate(tables):
            if use_tt:
                tab = TtTable(plan_shapes(int(rows), self.emb, 3, int(rank)), f"table{t}", np.float32,
                              device=device, stream=self.stream.cuda_stream)
                self.tables.append(tab)
                self.ctx.append(ForwardContext(tab))
                self.kinds.append("tt")
            else:
                self.tables.append(DenseEmbeddingBags([int(rows)], self.emb, np.float32, device=device,
                                                      stream=self.stream.cuda_stream))
                self.ctx.append(None)
                self.kinds.append("dense")

    # ---- parameters ---------------------------------------------------------
    def num_features(self) -> int:
        return self.nt + 1

    def init(self, seed: int):
        """Reference distributions (mlp.hpp:54-61: U(+-1/sqrt(in)), zero bias;
        sampled-Gaussian TT cores, initializer.hpp; dense U(+-1/sqrt(emb)),
        model.hpp:180-186), drawn from numpy / the TT initializer."""
        rng = np.random.default_rng(seed)
        for layers in (self.bottom, self.top):
            for layer in layers:
                o, i = layer["w"].shape
                s = 1.0 / np.sqrt(i)
                layer["w"].copy_(self.torch.from_numpy(rng.uniform(-s, s, (o, i)).astype(np.float32)))
                layer["b"].zero_()
        for t, tab in enumerate(self.tables):
            if self.kinds[t] == "tt":
                tab.init_sampled_gaussian(int(seed) + 0x7AB1E0 + t)
            else:
                s = 1.0 / np.sqrt(self.emb)
                tab.set_table(0, rng.uniform(-s, s, (tab.rows[0], self.emb)))

    def set_mlp(self, which: str, layer: int, w, b):
        L = (self.bottom if which == "bottom" else self.top)[layer]
        L["w"].copy_(self.torch.as_tensor(np.asarray(w, np.float32).reshape(L["w"].shape)))
        L["b"].copy_(self.torch.as_tensor(np.asarray(b, np.float32)))

    def mlp_params(self, which: str, layer: int):
        L = (self.bottom if which == "bottom" else self.top)[layer]
        self.stream.synchronize()
        return L["w"].cpu().numpy().ravel(), L["b"].cpu().numpy()

    def set_tt_core(self, t: int, k: int, values):
        self.tables[t].set_core(k, values)

    def tt_core(self, t: int, k: int) -> np.ndarray:
        return self.tables[t].core(k)

    def set_dense_table(self, t: int, values):
        self.tables[t].set_table(0, np.asarray(values, np.float32).reshape(-1, self.emb))

    def dense_table(self, t: int) -> np.ndarray:
        self.stream.synchronize()
        return self.tables[t].table(0)

    # ---- one step -----------------------------------------------------------
    def _mlp_forward(self, layers, x):
        saved = []
        for i, L in enumerate(layers):
            z = x @ L["w"].t() + L["b"]
            saved.append((x, z))
            x = self.torch.relu(z) if i + 1 < len(layers) else z
        return x, saved

    def _mlp_backward(self, layers, saved, dy):
        cur = dy
        for i in range(len(layers) - 1, -1, -1):
            L = layers[i]
            x, z = saved[i]
            dz = cur if i + 1 == len(layers) else cur * (z > 0)
            L["gw"] += dz.t() @ x
            L["gb"] += dz.sum(0)
            cur = dz @ L["w"]
        return cur

    def forward(self, mb) -> "object":
        """mb: dict of device tensors dense (bs x df, float32), idx / off (per
        table int64), labels (float64).  Returns the logits (bs,)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            bs = mb["dense"].shape[0]
            bout, self._bsaved = self._mlp_forward(self.bottom, mb["dense"])
            feats = [bout]
            for t, tab in enumerate(self.tables):
                out = torch.empty((bs, self.emb), dtype=torch.float32, device=self.dev)
                idx, off = mb["idx"][t], mb["off"][t]
                if self.kinds[t] == "tt":
                    tab.forward_device(self.ctx[t], idx.data_ptr(), idx.numel(), off.data_ptr(), bs,
                                       out.data_ptr(), save=True)
                else:
                    tab.forward_device(idx.data_ptr(), idx.numel(), off.data_ptr(), bs, out.data_ptr())
                feats.append(out)
            self._F = torch.stack(feats, 1)  # bs x f x emb
            if self.dot:
                Z = torch.bmm(self._F, self._F.transpose(1, 2))
                z = torch.cat([bout, Z[:, self.iu[0], self.iu[1]]], 1)
            else:
                z = self._F.reshape(bs, -1)
            logits, self._tsaved = self._mlp_forward(self.top, z)
            return logits.reshape(bs)

    @staticmethod
    def bce_with_logits(logits, labels, n=None):
        """model.hpp:82-103 in float64: (mean loss, dlogits as float32); n is the
        batch the mean is over (the global batch under data parallelism)."""
        import torch

        x = logits.double()
        y = labels
        total = torch.clamp(x, min=0) - x * y + torch.log1p(torch.exp(-x.abs()))
        sig = torch.where(x >= 0, 1.0 / (1.0 + torch.exp(-x)), torch.exp(x) / (1.0 + torch.exp(x)))
        n = x.numel() if n is None else n
        return total.sum() / n, ((sig - y) / n).float()

    def backward(self, mb, dlogits, fused_lr: float = None):
        """Gradients of every parameter for the last forward; with fused_lr the
        tables apply their SGD in the same pass (backward_bags + sgd_step fused)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            bs = dlogits.shape[0]
            dz = self._mlp_backward(self.top, self._tsaved, dlogits.reshape(bs, 1))
            f = self.num_features()
            if self.dot:
                dZ = torch.zeros((bs, f, f), dtype=torch.float32, device=self.dev)
                dZ[:, self.iu[0], self.iu[1]] = dz[:, self.emb:]
                dF = torch.bmm(dZ + dZ.transpose(1, 2), self._F)
                dF[:, 0] += dz[:, :self.emb]
            else:
                dF = dz.reshape(bs, f, self.emb)
            self._mlp_backward(self.bottom, self._bsaved, dF[:, 0].contiguous())
            self._dfeat = [dF[:, t + 1].contiguous() for t in range(self.nt)]
            for t, tab in enumerate(self.tables):
                g = self._dfeat[t]
                if self.kinds[t] == "tt":
                    if fused_lr is None:
                        tab.backward_device(self.ctx[t], g.data_ptr())
                    else:
                        tab.backward_sgd_device(self.ctx[t], g.data_ptr(), fused_lr)
                else:
                    tab.backward_device(g.data_ptr(), 0.0 if fused_lr is None else fused_lr,
                                        fused=fused_lr is not None)

    def step(self, lr: float, tables_done: bool = False):
        torch = self.torch
        with torch.cuda.stream(self.stream):
            s = torch.tensor(np.float32(lr), device=self.dev)
            for layers in (self.bottom, self.top):
                for L in layers:
                    L["w"] -= s * L["gw"]
                    L["b"] -= s * L["gb"]
                    L["gw"].zero_()
                    L["gb"].zero_()
            if not tables_done:
                for t, tab in enumerate(self.tables):
                    tab.apply_grad(lr)

    def _grad_tensors(self):
        """Every gradient buffer (device tensors / views), in a fixed order."""
        torch = self.torch
        out = []
        for layers in (self.bottom, self.top):
            for L in layers:
                out += [L["gw"], L["gb"]]
        for t, tab in enumerate(self.tables):
            ptr, n = tab.grad_buffer()

            class _Arr:
                __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                            "version": 3, "strides": None}

            out.append(torch.as_tensor(_Arr(), device=self.dev))
        return out

    def allreduce_grads(self):
        """One flat allreduce(SUM) of every gradient (data parallel)."""
        import torch.distributed as dist

        torch = self.torch
        with torch.cuda.stream(self.stream):
            gs = self._grad_tensors()
            flat = torch.cat([g.reshape(-1) for g in gs])
            dist.all_reduce(flat, group=self.group)
            o = 0
            for g in gs:
                n = g.numel()
                g.copy_(flat[o:o + n].view_as(g))
                o += n

    def train_step(self, mb, lr: float, fused: bool = True):
        """One train() iteration: forward, BCE, backward, step.  Returns the
        logits (device) and the loss (device float64 scalar; the global mean
        under data parallelism)."""
        torch = self.torch
        logits = self.forward(mb)
        n = logits.numel() * self.world
        with torch.cuda.stream(self.stream):
            loss, dlogits = self.bce_with_logits(logits, mb["labels"], n)
        if self.world > 1:
            import torch.distributed as dist

            self.backward(mb, dlogits)  # dense gradients (every table's buffer)
            self.allreduce_grads()
            self.step(lr)
            with torch.cuda.stream(self.stream):
                dist.all_reduce(loss, group=self.group)
            return logits, loss
        self.backward(mb, dlogits, fused_lr=lr if fused else None)
        self.step(lr, tables_done=fused)
        return logits, loss

    def to_device(self, mb):
        """Host minibatch (numpy, tests / the reference's SyntheticDataSource) -> device."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            return {"dense": torch.as_tensor(np.asarray(mb["dense"], np.float32), device=self.dev),
                    "labels": torch.as_tensor(np.asarray(mb["labels"], np.float64), device=self.dev),
                    "idx": [torch.as_tensor(np.asarray(i, np.int64), device=self.dev) for i in mb["idx"]],
                    "off": [torch.as_tensor(np.asarray(o, np.int64), device=self.dev) for o in mb["off"]]}
