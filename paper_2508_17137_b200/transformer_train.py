"""Training of the paper's transformer predictor (
PAPER.md:96-98) on the sm_100a kernels.

One step over a batch of whole prompts (rows in (token, layer) order,
attention inside windows of <= 512 rows of one prompt, as in inference):

  forward   the inference pipeline (K4 tcgen05 GEMMs, K5 attention), keeping
            each layer's input, qkv, attention output, pre-norm sums,
            LayerNorm outputs and FFN activations (16-bit), the head's
            pre-GELU rows and fp32 logits
  loss      BCEWithLogits against the rows' expert masks, mean over rows x
            experts (moeb_bce_logits_grad), gradient scaled by the loss scale
  backward  dX = dY W and dW = dY^T X as K4 GEMMs on transposed 16-bit
            operands (moeb_transpose16), bias / LayerNorm-affine gradients as
            column sums, LayerNorm / ReLU / GELU backward kernels, the
            windowed attention backward (moeb_attention_bwd), the layer
            embedding gradient as a per-layer row sum; the token table is
            frozen (as in the oracle, requires_grad=False)
  optimiser dynamic loss scaling (GradScaler semantics: a step whose
            gradients are not finite is skipped and the scale halved; the
            scale doubles after `growth_interval` good steps), global
            gradient-norm clipping at 1.0, AdamW (betas 0.9 / 0.98, weight
            decay 0.01) with the paper's per-group learning rates: input
            projection + layer embedding 1e-4, encoder 0.9e-4, head 0.8e-4.

fp32 master weights, 16-bit (fp16 by default) GEMM operands refreshed after
every step. Dropout (p = 0.1 in the paper) is not applied: the step equals
the eval-mode network's gradient (the parity tests compare it with the fp32
oracle's autograd).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .core import ConfigError
from .traces import PackedTraces
from .transformer import (D_FF, D_HEAD_MLP, D_LAYER, D_MODEL, D_TOK, EPI_BIAS, EPI_BIAS_RELU,
                          EPI_F32, EPI_RESID_ADD16, LN_EPS, N_LAYERS, WINDOW, TransformerWeights,
                          gemm, layernorm16, windows_of)


@dataclass
class TrainConfig:
    lr_input: float = 1e-4
    lr_encoder: float = 0.9e-4
    lr_head: float = 0.8e-4
    betas: tuple = (0.9, 0.98)
    eps: float = 1e-8
    weight_decay: float = 0.01
    clip_norm: float = 1.0
    loss_scale: float = 2.0 ** 16
    growth_interval: int = 2000
    fp16: bool = True


def _group(name: str) -> str:
    if name in ("in_w", "in_b", "layer_emb"):
        return "input"
    if name.startswith("h1_") or name.startswith("h2_"):
        return "head"
    return "encoder"


MATRICES = ("qkv_w", "o_w", "f1_w", "f2_w")


class TransformerTrainer:
    """Device training state: fp32 master weights, AdamW moments, 16-bit
    operand copies (and their transposes) for the GEMMs."""

    def __init__(self, state: dict, num_layers: int, num_experts: int,
                 config: TrainConfig | None = None, device=None):
        nat.load_library()
        self.cfg = config or TrainConfig()
        self.dev = torch.device("cuda") if device is None else torch.device(device)
        self.L, self.E = num_layers, num_experts
        if num_experts % 64:
            raise ConfigError("transformer head needs E to be a multiple of 64")
        self.dt = torch.float16 if self.cfg.fp16 else torch.bfloat16
        f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(self.dev)  # noqa: E731
        self.tok16 = f32(state["tok"]).to(self.dt).contiguous()  # frozen
        self.params = {k: f32(v) for k, v in state.items() if k != "tok"}
        self.grads = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.m = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.step_count = 0
        self.good_steps = 0
        self.scale = float(self.cfg.loss_scale)
        self._refresh16()

    # ------------------------------------------------------------------
    def _c16(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty(x.shape, dtype=self.dt, device=self.dev)
        nat.call("moeb_cast_f32_to_16", nat.ptr(x.contiguous()), x.numel(), nat.ptr(out),
                 int(self.cfg.fp16), nat.stream_ptr())
        return out

    def _t16(self, x16: torch.Tensor, rows: int | None = None) -> torch.Tensor:
        """[R][C] 16-bit -> [C][R] (R = rows of x16 used)."""
        R = x16.shape[0] if rows is None else rows
        C = x16.shape[1]
        out = torch.empty((C, R), dtype=self.dt, device=self.dev)
        nat.call("moeb_transpose16", nat.ptr(x16), R, C, x16.stride(0), nat.ptr(out), R,
                 nat.stream_ptr())
        return out

    def _refresh16(self):
        """16-bit GEMM operands of the current master weights: W [out][in] for
        the forward, W^T [in][out] for dX = dY W."""
        self.w16, self.wt16 = {}, {}
        for k, v in self.params.items():
            if v.dim() == 2 and k != "layer_emb":
                self.w16[k] = self._c16(v)
                self.wt16[k] = self._t16(self.w16[k])
        self.lay16 = self._c16(self.params["layer_emb"])
        # input projection's layer-embedding block, transposed: [512 in][512 out]
        self.win_lay_t16 = self._t16(self.w16["in_w"][:, D_TOK:].contiguous())

    def weights(self) -> TransformerWeights:
        """Inference weights of the current master state."""
        sd = {k: v.detach().cpu().numpy() for k, v in self.params.items()}
        sd["tok"] = self.tok16.float().cpu().numpy()
        return TransformerWeights(sd, self.L, self.E, fp16=self.cfg.fp16, device=self.dev)

    # ------------------------------------------------------------------
    def _rows(self, packed: PackedTraces):
        """Per-row token / layer ids (int32, padded rows: 0) and windows."""
        L = packed.shape.num_layers
        off = packed.row_off_host
        M = int(off[-1])
        Mp = (M + 63) // 64 * 64
        tok_t = packed.token_ids.cpu().numpy().astype(np.int64)
        tok = np.zeros(Mp, dtype=np.int32)
        lay = np.zeros(Mp, dtype=np.int32)
        for p in range(packed.num_prompts):
            a, b = int(off[p]), int(off[p + 1])
            r = np.arange(b - a)
            tok[a:b] = tok_t[a // L + r // L]
            lay[a:b] = r % L
        ws, wl = windows_of(off)
        d = lambda x: torch.from_numpy(x).to(self.dev)  # noqa: E731
        return M, Mp, d(tok), d(lay), d(ws), d(wl), len(ws)

    def forward_backward(self, packed: PackedTraces) -> float:
        """Loss of the batch; self.grads = d loss / d params, times the loss
        scale (fp32)."""
        cfg, dev, dt = self.cfg, self.dev, self.dt
        fp16 = int(cfg.fp16)
        if packed.token_ids is None:
            raise ConfigError("training needs per-token ids (PackedTraces.token_ids)")
        M, Mp, tok, lay, ws, wl, nw = self._rows(packed)
        E = self.E
        z16 = lambda *s: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
        P, W16, WT16 = self.params, self.w16, self.wt16
        for g in self.grads.values():
            g.zero_()
        # ---------------- forward ----------------
        F = z16(Mp, D_TOK + D_LAYER)
        nat.call("moeb_gather_inputs16", nat.ptr(self.tok16), nat.ptr(self.lay16), nat.ptr(tok),
                 nat.ptr(lay), Mp, nat.ptr(F), nat.stream_ptr())
        h = z16(Mp, D_MODEL)
        gemm(F, W16["in_w"], Mp, D_MODEL, D_TOK + D_LAYER, EPI_BIAS, bias=P["in_b"], out16=h,
             fp16=cfg.fp16)
        saved = []
        for i in range(N_LAYERS):
            pre = f"l{i}."
            qkv = z16(Mp, 3 * D_MODEL)
            gemm(h, W16[pre + "qkv_w"], Mp, 3 * D_MODEL, D_MODEL, EPI_BIAS, bias=P[pre + "qkv_b"],
                 out16=qkv, fp16=cfg.fp16)
            a = z16(Mp, D_MODEL)
            nat.call("moeb_window_attention", nat.ptr(qkv), nat.ptr(a), nat.ptr(ws), nat.ptr(wl),
                     nw, WINDOW, Mp, fp16, nat.stream_ptr())
            x1 = h.clone()
            gemm(a, W16[pre + "o_w"], Mp, D_MODEL, D_MODEL, EPI_RESID_ADD16, bias=P[pre + "o_b"],
                 out16=x1, fp16=cfg.fp16)
            h1 = x1.clone()
            layernorm16(h1, P[pre + "n1_w"], P[pre + "n1_b"], Mp, cfg.fp16)
            ff = z16(Mp, D_FF)
            gemm(h1, W16[pre + "f1_w"], Mp, D_FF, D_MODEL, EPI_BIAS_RELU, bias=P[pre + "f1_b"],
                 out16=ff, fp16=cfg.fp16)
            x2 = h1.clone()
            gemm(ff, W16[pre + "f2_w"], Mp, D_MODEL, D_FF, EPI_RESID_ADD16, bias=P[pre + "f2_b"],
                 out16=x2, fp16=cfg.fp16)
            h2 = x2.clone()
            layernorm16(h2, P[pre + "n2_w"], P[pre + "n2_b"], Mp, cfg.fp16)
            saved.append((h, qkv, a, x1, h1, ff, x2))
            h = h2
        u = z16(Mp, D_HEAD_MLP)
        gemm(h, W16["h1_w"], Mp, D_HEAD_MLP, D_MODEL, EPI_BIAS, bias=P["h1_b"], out16=u,
             fp16=cfg.fp16)
        g = z16(Mp, D_HEAD_MLP)
        nat.call("moeb_gelu_fwd16", nat.ptr(u), nat.ptr(g), u.numel(), fp16, nat.stream_ptr())
        z = torch.zeros((Mp, E), dtype=torch.float32, device=dev)
        gemm(g, W16["h2_w"], Mp, E, D_HEAD_MLP, EPI_F32, bias=P["h2_b"], out32=z, fp16=cfg.fp16)
        self.last_logits = z[:M]
        # ---------------- loss ----------------
        dz = z16(Mp, E)
        loss_sum = torch.zeros(1, dtype=torch.float64, device=dev)
        nat.call("moeb_bce_logits_grad", nat.ptr(z), nat.ptr(packed.truth), M, E, self.scale,
                 nat.ptr(dz), nat.ptr(loss_sum), fp16, nat.stream_ptr())
        # ---------------- backward ----------------
        G = self.grads

        def dW(dy16, x16, name, N, K):  # grads[name] [N][K] = dy^T x (K4 on transposes)
            gemm(self._t16(dy16), self._t16(x16), N, K, Mp, EPI_F32, out32=G[name],
                 fp16=cfg.fp16)

        def db(dy16, name):
            nat.call("moeb_colsum16", nat.ptr(dy16), Mp, dy16.shape[1], dy16.stride(0),
                     nat.ptr(G[name]), fp16, nat.stream_ptr())

        def dX(dy16, name, N, K, out16=None, resid=False):  # dy [Mp][K] . W [K][N] -> [Mp][N]
            out = out16 if out16 is not None else z16(Mp, N)
            gemm(dy16, WT16[name], Mp, N, K, EPI_RESID_ADD16 if resid else EPI_BIAS, out16=out,
                 fp16=cfg.fp16)
            return out

        dW(dz, g, "h2_w", E, D_HEAD_MLP)
        db(dz, "h2_b")
        dg = dX(dz, "h2_w", D_HEAD_MLP, E)
        nat.call("moeb_gelu_bwd16", nat.ptr(dg), nat.ptr(u), dg.numel(), fp16, nat.stream_ptr())
        dW(dg, h, "h1_w", D_HEAD_MLP, D_MODEL)
        db(dg, "h1_b")
        dh = dX(dg, "h1_w", D_MODEL, D_HEAD_MLP)
        lse2 = torch.zeros((Mp, 8), dtype=torch.float32, device=dev)
        dsum = torch.zeros((Mp, 8), dtype=torch.float32, device=dev)
        for i in reversed(range(N_LAYERS)):
            pre = f"l{i}."
            h_in, qkv, a, x1, h1, ff, x2 = saved[i]
            dx2 = z16(Mp, D_MODEL)
            nat.call("moeb_layernorm_bwd16", nat.ptr(dh), nat.ptr(x2), nat.ptr(P[pre + "n2_w"]),
                     Mp, LN_EPS, nat.ptr(dx2), nat.ptr(G[pre + "n2_w"]), nat.ptr(G[pre + "n2_b"]),
                     fp16, nat.stream_ptr())
            dff = dX(dx2, pre + "f2_w", D_FF, D_MODEL)
            dW(dx2, ff, pre + "f2_w", D_MODEL, D_FF)
            db(dx2, pre + "f2_b")
            nat.call("moeb_relu_bwd16", nat.ptr(dff), nat.ptr(ff), dff.numel(), fp16,
                     nat.stream_ptr())
            dW(dff, h1, pre + "f1_w", D_FF, D_MODEL)
            db(dff, pre + "f1_b")
            dh1 = dX(dff, pre + "f1_w", D_MODEL, D_FF, out16=dx2.clone(), resid=True)
            dx1 = z16(Mp, D_MODEL)
            nat.call("moeb_layernorm_bwd16", nat.ptr(dh1), nat.ptr(x1), nat.ptr(P[pre + "n1_w"]),
                     Mp, LN_EPS, nat.ptr(dx1), nat.ptr(G[pre + "n1_w"]), nat.ptr(G[pre + "n1_b"]),
                     fp16, nat.stream_ptr())
            da = dX(dx1, pre + "o_w", D_MODEL, D_MODEL)
            dW(dx1, a, pre + "o_w", D_MODEL, D_MODEL)
            db(dx1, pre + "o_b")
            dqkv = z16(Mp, 3 * D_MODEL)
            nat.call("moeb_attention_bwd", nat.ptr(qkv), nat.ptr(a), nat.ptr(da), nat.ptr(ws),
                     nat.ptr(wl), nw, WINDOW, nat.ptr(dqkv), nat.ptr(lse2), nat.ptr(dsum), fp16,
                     nat.stream_ptr())
            dW(dqkv, h_in, pre + "qkv_w", 3 * D_MODEL, D_MODEL)
            db(dqkv, pre + "qkv_b")
            dh = dX(dqkv, pre + "qkv_w", D_MODEL, 3 * D_MODEL, out16=dx1.clone(), resid=True)
        dW(dh, F, "in_w", D_MODEL, D_TOK + D_LAYER)
        db(dh, "in_b")
        dlay_rows = z16(Mp, D_LAYER)
        gemm(dh, self.win_lay_t16, Mp, D_LAYER, D_MODEL, EPI_BIAS, out16=dlay_rows, fp16=cfg.fp16)
        nat.call("moeb_layer_emb_grad", nat.ptr(dlay_rows), D_LAYER, M, nat.ptr(lay),
                 self.params["layer_emb"].shape[0], nat.ptr(G["layer_emb"]), fp16,
                 nat.stream_ptr())
        return float(loss_sum.item()) / (M * E)

    # ------------------------------------------------------------------
    def grad_norm(self) -> float:
        """Global L2 norm of the (unscaled) gradients."""
        acc = torch.zeros(1, dtype=torch.float64, device=self.dev)
        for g in self.grads.values():
            nat.call("moeb_sumsq_f32", nat.ptr(g), g.numel(), nat.ptr(acc), nat.stream_ptr())
        return float(acc.sqrt().item()) / self.scale

    def optimizer_step(self) -> dict:
        """GradScaler + clip_grad_norm_ + AdamW on the current gradients."""
        cfg = self.cfg
        norm = self.grad_norm()
        if not np.isfinite(norm):
            self.scale /= 2.0
            self.good_steps = 0
            return {"skipped": True, "grad_norm": norm, "scale": self.scale}
        clip = min(1.0, cfg.clip_norm / (norm + 1e-6))
        self.step_count += 1
        lrs = {"input": cfg.lr_input, "encoder": cfg.lr_encoder, "head": cfg.lr_head}
        for k, p in self.params.items():
            nat.call("moeb_adamw_f32", nat.ptr(p), nat.ptr(self.grads[k]), nat.ptr(self.m[k]),
                     nat.ptr(self.v[k]), p.numel(), lrs[_group(k)], cfg.betas[0], cfg.betas[1],
                     cfg.eps, cfg.weight_decay, self.step_count, clip / self.scale,
                     nat.stream_ptr())
        self._refresh16()
        self.good_steps += 1
        if self.good_steps >= cfg.growth_interval:
            self.scale *= 2.0
            self.good_steps = 0
        return {"skipped": False, "grad_norm": norm, "clip": clip, "scale": self.scale}

    def step(self, packed: PackedTraces) -> dict:
        loss = self.forward_backward(packed)
        info = self.optimizer_step()
        info["loss"] = loss
        return info
