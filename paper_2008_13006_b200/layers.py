"""Layer-chaining caller of the TW path: the reference trainer's engine
forward (trainer.py:232-250 `engine_logits`), on the GPU.

The reference runs, per layer, compact(W) -> gemm_tw -> `+ bias` -> ReLU
(not after the last layer), copying every activation back to a host
DenseMatrix.  Here every layer is one persistent TW-GEMM with the bias/ReLU
epilogue fused, and activations never leave HBM or change layout: a layer's
output C^T (N x M) is exactly the next layer's A^T (the paper's "transpose
A only in the first layer, C after the last").

Two arithmetic modes (TwMlp `precision`):
  "fp16" / "bf16": 16-bit operands, intermediate activations stored in that
      dtype (the serving path; the kernel's fused epilogue rounds once);
  "fp32" (engine_logits' default, like the reference's float32 forward):
      split-bf16 plans (TwPlan precision "fp32"), fp32 intermediates -- each
      layer writes relu(C + b) in fp32 and the next layer's [hi; lo]
      operand is cut from it on the device;
  "exact": the reference's rounding sequence per layer (CUDA cores).
The last layer always writes fp32 logits.
"""

from __future__ import annotations

import numpy as np

from .engine import DEFAULT_PRECISION, TwPlan, prep_activations
from .matrix import DenseMatrix, DimensionError, Layout
from .pattern import compact

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


class TwMlp:
    """Device-resident TW layers of an MLP: one TwPlan + fp32 bias per layer.
    `weights` K_i x N_i arrays, `biases` N_i arrays, `patterns` TilePatterns
    (the reference's MlpModel.weights / .biases and per-layer patterns)."""

    def __init__(self, weights, biases, patterns, device=None, dtype=None, precision=None):
        if not (len(weights) == len(biases) == len(patterns)):
            raise DimensionError("need one pattern per layer")  # trainer.py:239-240
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if precision is None:
            precision = {None: "fp16", torch.float16: "fp16", torch.bfloat16: "bf16"}.get(dtype, "fp16")
        if precision not in ("fp16", "bf16", "fp32", "exact"):
            raise ValueError(f"precision must be fp16, bf16, fp32 or exact, got {precision!r}")
        self.precision = precision
        # activation / plan dtype of the 16-bit path (fp32 and exact keep fp32 activations)
        self.dtype = {"fp16": torch.float16, "bf16": torch.bfloat16}.get(precision, torch.float32)
        plan_dtype = torch.float16 if precision == "fp16" else torch.bfloat16
        plan_prec = {"fp16": "bf16", "bf16": "bf16", "fp32": "fp32", "exact": "exact"}[precision]
        self.plans, self.biases = [], []
        self._acts = {}
        for w, b, p in zip(weights, biases, patterns):
            ts = compact(DenseMatrix.from_array(np.asarray(w, np.float32)), p)
            self.plans.append(TwPlan(ts, device=self.device, dtype=plan_dtype, precision=plan_prec))
            bb = np.asarray(b, np.float32).reshape(-1)
            if bb.size != ts.n:
                raise DimensionError(f"bias has {bb.size} entries, layer has {ts.n} outputs")
            self.biases.append(torch.from_numpy(bb).to(self.device))
        for a, b in zip(self.plans, self.plans[1:]):
            if a.n != b.k:
                raise DimensionError(f"layer output {a.n} does not match next layer input {b.k}")

    def _act(self, i, m):
        """Resident activation buffer of layer i for M tokens.  Its pruned
        rows hold the constant relu(bias[j]) after the first call, so later
        calls skip them (write_pruned=False): the kernel writes only the kept
        columns' rows."""
        key = (i, m)
        if key not in self._acts:
            ld = (m + 7) // 8 * 8  # next layer gathers 16-byte row chunks
            self._acts[key] = [torch.empty((self.plans[i].n, ld), dtype=self.dtype, device=self.device)[:, :m], False]
        return self._acts[key]

    def forward_t(self, at, stream=None):
        """A^T operand of layer 0 (K0 x M: plan dtype; for "fp32" the split
        operand TwPlan.prep makes; for "exact" fp32) -> logits^T (N_last x M,
        fp32), all on device."""
        last = len(self.plans) - 1
        if self.precision in ("fp32", "exact"):
            for i, (plan, b) in enumerate(zip(self.plans, self.biases)):
                if self.precision == "fp32":
                    z = plan.gemm(at, out_dtype=torch.float32, bias=b, relu=i < last, stream=stream)
                else:  # trainer.py:246-248 on the exact product: fp32 add, then max(., 0)
                    z = plan.gemm(at, stream=stream) + b[:, None]
                    if i < last:
                        z = torch.clamp_min(z, 0.0)
                if i < last:  # C^T (N x M fp32) is the next layer's COL_MAJOR A buffer
                    at = self.plans[i + 1].prep(z.contiguous(), Layout.COL_MAJOR, stream=stream)
                else:
                    at = z
            return at
        for i, (plan, b) in enumerate(zip(self.plans, self.biases)):
            m = at.shape[1]
            if i < last:
                slot = self._act(i, m)
                at = plan.gemm(at, out=slot[0], out_dtype=self.dtype, bias=b, relu=True, stream=stream,
                               write_pruned=not slot[1])
                slot[1] = True
            else:
                at = plan.gemm(at, out_dtype=torch.float32, bias=b, relu=False, stream=stream)
        return at

    def graph(self, m: int) -> "TwMlpGraph":
        """Capture the whole forward for M tokens into one CUDA graph (the
        serving path: at small M the layer chain is launch-bound).  One eager
        pass first builds the launch schedules and writes the resident
        activations' pruned rows; the captured pass then writes kept rows only
        (write_pruned=False), with bias/ReLU fused, layer to layer in HBM."""
        k0 = self.plans[0].k
        ld = (m + 7) // 8 * 8
        static_in = torch.zeros((k0, ld), dtype=self.dtype, device=self.device)[:, :m]
        self.forward_t(static_in)
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self.forward_t(static_in)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            static_out = self.forward_t(static_in)
        return TwMlpGraph(g, static_in, static_out)

    def logits(self, x) -> np.ndarray:
        """x: M x K0 (host) -> M x N_last fp32 (host), like engine_logits."""
        x = np.ascontiguousarray(np.asarray(x, np.float32))
        xt = torch.from_numpy(x).to(self.device)
        if self.precision in ("fp32", "exact"):
            at = self.plans[0].prep(xt, Layout.ROW_MAJOR)
        else:
            at = prep_activations(xt, Layout.ROW_MAJOR, self.dtype)
        return self.forward_t(at).t().contiguous().cpu().numpy()


class TwMlpGraph:
    """A captured TwMlp forward: write A^T into `.input` (K0 x M, plan dtype)
    or pass it to __call__, replay, read `.output` (N_last x M, fp32)."""

    def __init__(self, graph, static_in, static_out):
        self._g, self.input, self.output = graph, static_in, static_out

    def __call__(self, at=None):
        if at is not None:
            self.input.copy_(at)
        self._g.replay()
        return self.output


def engine_logits(model, x, patterns, workers: int = 1, *, device=None, dtype=None, precision=None) -> np.ndarray:
    """trainer.py:232-250 drop-in: float32 forward pass through the TW-GEMM
    with a bias+ReLU epilogue.  `model` is duck-typed (.weights, .biases, as
    the reference's MlpModel); `workers` is accepted for signature parity.
    Arithmetic: `precision` (default engine.DEFAULT_PRECISION, "fp32": fp32
    intermediates on split-bf16 tensor-core plans); passing a 16-bit `dtype`
    selects the 16-bit activation path instead."""
    if len(patterns) != len(model.weights):
        raise DimensionError("need one pattern per layer")
    if workers < 1:
        raise DimensionError(f"workers must be >= 1, got {workers}")
    if precision is None:
        precision = {torch.float16: "fp16", torch.bfloat16: "bf16"}.get(dtype, DEFAULT_PRECISION)
    net = TwMlp(model.weights, model.biases, patterns, device=device, precision=precision)
    return net.logits(x)
