"""PyTorch fp32 oracle of the MoE-Beyond transformer predictor -- TEST
INFRASTRUCTURE ONLY (the checker for the CUDA path; never imported by the
product package).

The reference repository contains no transformer code: its authors replaced
it by the linear learner. The architecture is taken
from the paper's prose with the open choices pinned once, as
SURVEY.md §8(c) lists them:

  * sequence position = trace row; rows of a prompt are cut into consecutive
    windows of 512 rows, the last one padded and key-padding-masked;
  * input x = [token embedding (2048) | layer embedding (512)] -> Linear(2560,
    512, bias); token table = torch.randn(32000, 2048), layer table
    nn.Embedding(max(L, 27), 512);
  * 4 x post-norm TransformerEncoderLayer(d=512, 8 heads, FFN 2048, ReLU,
    LayerNorm eps 1e-5, dropout = identity at inference), bidirectional
    attention within a window;
  * head Linear(512, 256) -> GELU (erf) -> Linear(256, E) = expert logits;
  * selection: top-`budget` by logit (ties to the lower id) or logit > 0.
Initialisation: torch.manual_seed(seed), then the modules in the order above
with PyTorch's default initialisers.

Parity bar (north star): CUDA logits within 1e-2 absolute of this module,
threshold decisions agreeing on >= 99.9 % of labels, masks bit-exact when the
selection head is fed this module's logits.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

VOCAB = 32000
D_TOK = 2048
D_LAYER = 512
D_MODEL = 512
N_HEAD = 8
D_FF = 2048
N_LAYERS = 4
D_HEAD_MLP = 256
WINDOW = 512
LN_EPS = 1e-5


@dataclass
class TransformerSpec:
    num_layers: int          # MoE layers L of the traced model (layer-id vocabulary)
    num_experts: int         # E (logit width)
    seed: int = 0
    window: int = WINDOW


class TransformerRef(nn.Module):
    def __init__(self, spec: TransformerSpec):
        super().__init__()
        torch.manual_seed(spec.seed)
        self.spec = spec
        self.tok = nn.Parameter(torch.randn(VOCAB, D_TOK), requires_grad=False)
        self.layer_emb = nn.Embedding(max(spec.num_layers, 27), D_LAYER)
        self.input_proj = nn.Linear(D_TOK + D_LAYER, D_MODEL)
        self.layers = nn.ModuleList([
            nn.TransformerEncoderLayer(D_MODEL, N_HEAD, D_FF, dropout=0.1, activation="relu",
                                       batch_first=True, norm_first=False, layer_norm_eps=LN_EPS)
            for _ in range(N_LAYERS)])
        self.head1 = nn.Linear(D_MODEL, D_HEAD_MLP)
        self.head2 = nn.Linear(D_HEAD_MLP, spec.num_experts)
        self.eval()

    # explicit fp32 math (same as nn.TransformerEncoderLayer post-norm, eval)
    @staticmethod
    def _encoder_layer(layer, x, pad):
        B, S, D = x.shape
        qkv = F.linear(x, layer.self_attn.in_proj_weight, layer.self_attn.in_proj_bias)
        q, k, v = qkv.split(D, dim=-1)
        q = q.view(B, S, N_HEAD, D // N_HEAD).transpose(1, 2)
        k = k.view(B, S, N_HEAD, D // N_HEAD).transpose(1, 2)
        v = v.view(B, S, N_HEAD, D // N_HEAD).transpose(1, 2)
        s = (q @ k.transpose(-1, -2)) / math.sqrt(D // N_HEAD)
        s = s.masked_fill(pad[:, None, None, :], float("-inf"))
        a = torch.softmax(s, dim=-1) @ v
        a = a.transpose(1, 2).reshape(B, S, D)
        a = F.linear(a, layer.self_attn.out_proj.weight, layer.self_attn.out_proj.bias)
        x = F.layer_norm(x + a, (D,), layer.norm1.weight, layer.norm1.bias, LN_EPS)
        f = F.linear(F.relu(F.linear(x, layer.linear1.weight, layer.linear1.bias)),
                     layer.linear2.weight, layer.linear2.bias)
        return F.layer_norm(x + f, (D,), layer.norm2.weight, layer.norm2.bias, LN_EPS)

    @torch.no_grad()
    def forward_windows(self, tok_ids, layer_ids, pad):
        """tok_ids/layer_ids [B, S] int64, pad [B, S] bool -> logits [B, S, E] fp32."""
        x = torch.cat([self.tok[tok_ids], self.layer_emb(layer_ids)], dim=-1)
        x = self.input_proj(x)
        for layer in self.layers:
            x = self._encoder_layer(layer, x, pad)
        return self.head2(F.gelu(self.head1(x)))

    @torch.no_grad()
    def logits(self, token_ids_per_row, layer_ids_per_row, row_off, device="cpu"):
        """Logits for every trace row of CSR-packed prompts (rows in (token,
        layer) order); windows never cross prompts. `device` runs the same
        fp32 math on a GPU for large checks (TF32 off)."""
        W = self.spec.window
        dev = torch.device(device)
        if dev.type == "cuda":
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
        self.to(dev)
        tok = torch.as_tensor(token_ids_per_row, dtype=torch.int64)
        lay = torch.as_tensor(layer_ids_per_row, dtype=torch.int64)
        out = torch.empty(len(tok), self.spec.num_experts)
        starts = []
        for p in range(len(row_off) - 1):
            for s in range(int(row_off[p]), int(row_off[p + 1]), W):
                starts.append((s, min(s + W, int(row_off[p + 1]))))
        for i in range(0, len(starts), 64):
            chunk = starts[i:i + 64]
            B = len(chunk)
            ti = torch.zeros(B, W, dtype=torch.int64)
            li = torch.zeros(B, W, dtype=torch.int64)
            pad = torch.ones(B, W, dtype=torch.bool)
            for b, (s, e) in enumerate(chunk):
                ti[b, :e - s] = tok[s:e]
                li[b, :e - s] = lay[s:e]
                pad[b, :e - s] = False
            y = self.forward_windows(ti.to(dev), li.to(dev), pad.to(dev)).cpu()
            for b, (s, e) in enumerate(chunk):
                out[s:e] = y[b, :e - s]
        self.to("cpu")
        return out


def row_inputs(token_ids_per_token, row_off, L):
    """Per-row token ids and layer ids from per-token ids (rows = tokens x L)."""
    tok = np.repeat(np.asarray(token_ids_per_token, dtype=np.int64), L)
    lay = np.zeros(len(tok), dtype=np.int64)
    for p in range(len(row_off) - 1):
        n = int(row_off[p + 1] - row_off[p])
        lay[int(row_off[p]):int(row_off[p + 1])] = np.arange(n) % L
    return tok, lay


def export_weights(ref: TransformerRef) -> dict:
    """Flat fp32 numpy weights (the device module packs them to bf16)."""
    sd = {"tok": ref.tok.detach().numpy(), "layer_emb": ref.layer_emb.weight.detach().numpy(),
          "in_w": ref.input_proj.weight.detach().numpy(),
          "in_b": ref.input_proj.bias.detach().numpy(),
          "h1_w": ref.head1.weight.detach().numpy(), "h1_b": ref.head1.bias.detach().numpy(),
          "h2_w": ref.head2.weight.detach().numpy(), "h2_b": ref.head2.bias.detach().numpy()}
    for i, layer in enumerate(ref.layers):
        sd[f"l{i}.qkv_w"] = layer.self_attn.in_proj_weight.detach().numpy()
        sd[f"l{i}.qkv_b"] = layer.self_attn.in_proj_bias.detach().numpy()
        sd[f"l{i}.o_w"] = layer.self_attn.out_proj.weight.detach().numpy()
        sd[f"l{i}.o_b"] = layer.self_attn.out_proj.bias.detach().numpy()
        sd[f"l{i}.f1_w"] = layer.linear1.weight.detach().numpy()
        sd[f"l{i}.f1_b"] = layer.linear1.bias.detach().numpy()
        sd[f"l{i}.f2_w"] = layer.linear2.weight.detach().numpy()
        sd[f"l{i}.f2_b"] = layer.linear2.bias.detach().numpy()
        sd[f"l{i}.n1_w"] = layer.norm1.weight.detach().numpy()
        sd[f"l{i}.n1_b"] = layer.norm1.bias.detach().numpy()
        sd[f"l{i}.n2_w"] = layer.norm2.weight.detach().numpy()
        sd[f"l{i}.n2_b"] = layer.norm2.bias.detach().numpy()
    return sd
