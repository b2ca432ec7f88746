"""The paper's transformer expert predictor on sm_100a kernels (row A10).

Architecture (pinned in SURVEY.md §8(c) and in the fp32
oracle oracle/transformer_ref.py): per trace row, x = [token embedding 2048 |
layer embedding 512] -> Linear(2560, 512) -> 4 post-norm encoder layers (d 512,
8 heads, FFN 2048 ReLU) with bidirectional attention inside windows of 512
consecutive rows of one prompt -> Linear(512, 256) -> GELU -> Linear(256, E).

Device pipeline per chunk of whole prompts (every GEMM is K4, the tcgen05
kernel, with its epilogue fused):
  embed     h = P_tok[token] + P_lay[layer]            (factorised input proj)
  per layer qkv = h Wqkv^T + b                          K4 EPI_BIAS
            a = attention(qkv, windows)                  K5
            h = LN(h + a Wo^T + bo)                      K4 EPI_RESID_LN
            f = relu(h W1^T + b1)                        K4 EPI_BIAS_RELU
            h = LN(h + f W2^T + b2)                      K4 EPI_RESID_LN
  head      y = gelu(h Wh1^T + bh1)                      K4 EPI_BIAS_GELU
            z = y Wh2^T + bh2 (fp32 logits)              K4 EPI_F32
            masks = top-k(z) / z > 0                     K2
The residual stream stays fp32; GEMM operands are 16-bit (fp16 by default,
bf16 selectable) with fp32 accumulation.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .core import ConfigError, ModelShape
from .traces import PackedTraces

VOCAB, D_TOK, D_LAYER, D_MODEL, N_HEAD, D_FF, N_LAYERS, D_HEAD_MLP = (
    32000, 2048, 512, 512, 8, 2048, 4, 256)
WINDOW = 512
LN_EPS = 1e-5
EPI_F32, EPI_BIAS, EPI_BIAS_RELU, EPI_BIAS_GELU, EPI_RESID_LN = range(5)
EPI_RESID_ADD = 6
EPI_RESID_ADD16 = 7


def init_state(num_layers: int, num_experts: int, seed: int = 0) -> dict:
    """fp32 weights of a seeded random-init predictor: torch.manual_seed(seed)
    then the modules in architecture order with PyTorch's default
    initialisers (the same recipe the fp32 oracle uses)."""
    import torch.nn as nn
    torch.manual_seed(seed)
    tok = torch.randn(VOCAB, D_TOK)
    layer_emb = nn.Embedding(max(num_layers, 27), D_LAYER)
    inp = nn.Linear(D_TOK + D_LAYER, D_MODEL)
    layers = [nn.TransformerEncoderLayer(D_MODEL, N_HEAD, D_FF, dropout=0.1, activation="relu",
                                         batch_first=True, norm_first=False,
                                         layer_norm_eps=LN_EPS) for _ in range(N_LAYERS)]
    h1, h2 = nn.Linear(D_MODEL, D_HEAD_MLP), nn.Linear(D_HEAD_MLP, num_experts)
    sd = {"tok": tok, "layer_emb": layer_emb.weight, "in_w": inp.weight, "in_b": inp.bias,
          "h1_w": h1.weight, "h1_b": h1.bias, "h2_w": h2.weight, "h2_b": h2.bias}
    for i, lay in enumerate(layers):
        sd.update({f"l{i}.qkv_w": lay.self_attn.in_proj_weight,
                   f"l{i}.qkv_b": lay.self_attn.in_proj_bias,
                   f"l{i}.o_w": lay.self_attn.out_proj.weight,
                   f"l{i}.o_b": lay.self_attn.out_proj.bias,
                   f"l{i}.f1_w": lay.linear1.weight, f"l{i}.f1_b": lay.linear1.bias,
                   f"l{i}.f2_w": lay.linear2.weight, f"l{i}.f2_b": lay.linear2.bias,
                   f"l{i}.n1_w": lay.norm1.weight, f"l{i}.n1_b": lay.norm1.bias,
                   f"l{i}.n2_w": lay.norm2.weight, f"l{i}.n2_b": lay.norm2.bias})
    return {k: v.detach().numpy().astype(np.float32) for k, v in sd.items()}


def gemm(a16, b16, M, N, K, epi, *, bias=None, out32=None, out16=None, ln=None, fp16=True,
         lda=None, ldb=None, ld16=None):
    """K4 launch; a16 [M][lda], b16 [N][ldb] 16-bit tensors (any 2-byte dtype)."""
    lw, lb = ln if ln is not None else (None, None)
    nat.call("moeb_gemm", nat.ptr(a16), lda or K, nat.ptr(b16), ldb or K, M, N, K, int(fp16),
             epi, nat.ptr(bias), nat.ptr(out32), nat.ptr(out16), ld16 or N, nat.ptr(lw),
             nat.ptr(lb), LN_EPS, nat.stream_ptr())


class TransformerWeights:
    """Device-resident predictor weights (16-bit GEMM operands, fp32 rest)."""

    def __init__(self, state: dict, num_layers: int, num_experts: int, fp16: bool = True,
                 device=None):
        nat.load_library()
        dev = torch.device("cuda") if device is None else torch.device(device)
        self.num_layers, self.num_experts, self.fp16, self.device = (num_layers, num_experts,
                                                                     fp16, dev)
        if num_experts % 64:
            raise ConfigError("transformer head needs E to be a multiple of 64")
        dt = torch.float16 if fp16 else torch.bfloat16
        f32 = lambda k: torch.from_numpy(np.ascontiguousarray(state[k])).to(dev)  # noqa: E731
        w16 = lambda k: f32(k).to(dt).contiguous()  # noqa: E731
        self.layers = []
        for i in range(N_LAYERS):
            self.layers.append({n: w16(f"l{i}.{n}_w") if n in ("qkv", "o", "f1", "f2")
                                else None for n in ("qkv", "o", "f1", "f2")})
            for n in ("qkv", "o", "f1", "f2", "n1", "n2"):
                self.layers[-1][n + "_b"] = f32(f"l{i}.{n}_b")
            self.layers[-1]["n1_w"] = f32(f"l{i}.n1_w")
            self.layers[-1]["n2_w"] = f32(f"l{i}.n2_w")
        self.h1_w, self.h1_b = w16("h1_w"), f32("h1_b")
        self.h2_w, self.h2_b = w16("h2_w"), f32("h2_b")
        # factorised input projection tables, computed once by K4 (fp32 out)
        in_w = w16("in_w")                                   # [512][2560]
        tok16 = f32("tok").to(dt).contiguous()               # [32000][2048]
        lay16 = f32("layer_emb").to(dt).contiguous()         # [Lemb][512]
        self.ptok = torch.empty((VOCAB, D_MODEL), dtype=torch.float32, device=dev)
        gemm(tok16, in_w, VOCAB, D_MODEL, D_TOK, EPI_F32, out32=self.ptok, fp16=fp16, ldb=2560)
        nl = lay16.shape[0]
        self.play = torch.empty((nl, D_MODEL), dtype=torch.float32, device=dev)
        in_w_lay = in_w[:, D_TOK:].contiguous()
        gemm(lay16, in_w_lay, nl, D_MODEL, D_LAYER, EPI_F32, bias=f32("in_b"),
             out32=self.play, fp16=fp16)
        del tok16

    @classmethod
    def random(cls, num_layers: int, num_experts: int, seed: int = 0, fp16: bool = True,
               device=None):
        return cls(init_state(num_layers, num_experts, seed), num_layers, num_experts, fp16,
                   device)


def layernorm16(x16, w, b, rows, fp16, eps=1e-5):
    """Post-norm LayerNorm of the 16-bit residual stream, in place
    (moeb_layernorm_rows16)."""
    nat.call("moeb_layernorm_rows16", nat.ptr(x16), nat.ptr(w), nat.ptr(b), rows, float(eps),
             int(bool(fp16)), nat.stream_ptr())


def layernorm(x32, x16, w, b, rows, fp16, eps=1e-5):
    """Post-norm LayerNorm of the first `rows` rows (moeb_layernorm_rows)."""
    nat.call("moeb_layernorm_rows", nat.ptr(x32), nat.ptr(x16), nat.ptr(w), nat.ptr(b), rows,
             float(eps), int(bool(fp16)), nat.stream_ptr())


def windows_of(row_off_host: np.ndarray, window: int = WINDOW):
    """(start row, length) of consecutive <= window-row windows per prompt."""
    starts, lens = [], []
    for p in range(len(row_off_host) - 1):
        a, b = int(row_off_host[p]), int(row_off_host[p + 1])
        s = np.arange(a, b, window)
        starts.append(s)
        lens.append(np.minimum(window, b - s))
    if not starts:
        return np.zeros(0, np.int64), np.zeros(0, np.int32)
    return np.concatenate(starts).astype(np.int64), np.concatenate(lens).astype(np.int32)


class TransformerPredictor:
    """Device predictor (make_predictor kind "transformer")."""

    kind = "transformer"
    unbounded_prefetch = False
    empty = False

    def __init__(self, weights: TransformerWeights, shape: ModelShape, threshold: bool = False,
                 chunk_rows: int = 1 << 20, resid16: bool | None = None):
        if shape.num_experts != weights.num_experts:
            raise ConfigError("transformer width != number of experts")
        self.weights, self.shape, self.threshold = weights, shape, threshold
        self.chunk_rows = chunk_rows
        # residual stream in the 16-bit operand format (the post-norm sum is
        # rounded once before its LayerNorm): 8 B of HBM traffic per element
        # and sublayer instead of the fp32 stream's 18. Default: with fp16
        # operands (C1: threshold agreement 99.97 %); bf16's 8-bit mantissa
        # keeps the fp32 stream
        self.resid16 = weights.fp16 if resid16 is None else bool(resid16)

    def coverage(self, packed):
        return None

    def _chunks(self, packed: PackedTraces):
        off = packed.row_off_host
        lo = 0
        while lo < packed.num_prompts:
            hi = lo + 1
            while hi < packed.num_prompts and off[hi + 1] - off[lo] <= self.chunk_rows:
                hi += 1
            yield lo, hi
            lo = hi

    def forward_logits(self, packed: PackedTraces, logits_out: torch.Tensor | None = None,
                       timing: dict | None = None):
        """fp32 logits [rows][E] for every trace row (chunked over prompts).

        With `timing` (a dict), CUDA events are recorded around every launch
        and timing[name] collects (start, end, flops) per launch."""
        W, s = self.weights, self.shape
        E, L = s.num_experts, s.num_layers
        dev = packed.device
        if packed.token_ids is None:
            raise ConfigError("transformer predictor needs per-token ids (PackedTraces.token_ids)")
        out = logits_out if logits_out is not None else torch.empty(
            (packed.rows, E), dtype=torch.float32, device=dev)
        dt = torch.float16 if W.fp16 else torch.bfloat16
        cap = min(self.chunk_rows, packed.rows) + WINDOW
        h32 = torch.empty((cap, D_MODEL), dtype=torch.float32, device=dev)
        h16 = torch.empty((cap, D_MODEL), dtype=dt, device=dev)
        qkv = torch.empty((cap, 3 * D_MODEL), dtype=dt, device=dev)
        att = torch.empty((cap, D_MODEL), dtype=dt, device=dev)
        ff = torch.empty((cap, D_FF), dtype=dt, device=dev)
        y = torch.empty((cap, D_HEAD_MLP), dtype=dt, device=dev)
        def timed(name, flops, fn, *a, **k):
            if timing is None:
                return fn(*a, **k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*a, **k)
            e1.record()
            timing.setdefault(name, []).append((e0, e1, flops))

        # every chunk's windows in one pinned upload (a pageable copy per
        # chunk would stall the launch stream)
        chunks = list(self._chunks(packed))
        roh = packed.row_off_host
        wins = [windows_of(roh[lo:hi + 1] - roh[lo]) for lo, hi in chunks]
        sizes = [len(ws) for ws, _ in wins]
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        ws_all = torch.from_numpy(np.concatenate([ws for ws, _ in wins])).pin_memory().to(
            dev, non_blocking=True)
        wl_all = torch.from_numpy(np.concatenate([wl for _, wl in wins])).pin_memory().to(
            dev, non_blocking=True)
        for ci, (lo, hi) in enumerate(chunks):
            r0, r1 = int(roh[lo]), int(roh[hi])
            M = r1 - r0
            ws, wl = wins[ci]
            ws_d = ws_all[offs[ci]:offs[ci + 1]]
            wl_d = wl_all[offs[ci]:offs[ci + 1]]
            tok = packed.token_ids[r0 // L:r1 // L]  # whole prompts: r0, r1 multiples of L
            nat.call("moeb_embed_rows", nat.ptr(W.ptok), nat.ptr(W.play), nat.ptr(tok), L, M,
                     nat.ptr(None if self.resid16 else h32), nat.ptr(h16), int(W.fp16),
                     nat.stream_ptr())
            att_flops = 4 * float(np.sum(wl.astype(np.float64) ** 2)) * D_MODEL
            for lay in W.layers:
                timed("gemm_qkv", 2.0 * M * 3 * D_MODEL * D_MODEL, gemm, h16, lay["qkv"], M,
                      3 * D_MODEL, D_MODEL, EPI_BIAS, bias=lay["qkv_b"], out16=qkv, fp16=W.fp16)
                timed("attention", att_flops, nat.call, "moeb_window_attention", nat.ptr(qkv),
                      nat.ptr(att), nat.ptr(ws_d), nat.ptr(wl_d), len(ws), WINDOW, M,
                      int(W.fp16),
                      nat.stream_ptr())
                # residual add fused into the GEMM epilogue (two TMEM
                # accumulators so epilogue and mainloop overlap), then a
                # streaming LayerNorm kernel over the rows; 16-bit residual
                # stream in place by default (see resid16)
                if self.resid16:
                    timed("gemm_out", 2.0 * M * D_MODEL * D_MODEL, gemm, att, lay["o"], M,
                          D_MODEL, D_MODEL, EPI_RESID_ADD16, bias=lay["o_b"], out16=h16,
                          fp16=W.fp16)
                    timed("layernorm", 0.0, layernorm16, h16, lay["n1_w"], lay["n1_b"], M,
                          W.fp16)
                else:
                    timed("gemm_out", 2.0 * M * D_MODEL * D_MODEL, gemm, att, lay["o"], M,
                          D_MODEL, D_MODEL, EPI_RESID_ADD, bias=lay["o_b"], out32=h32,
                          fp16=W.fp16)
                    timed("layernorm", 0.0, layernorm, h32, h16, lay["n1_w"], lay["n1_b"], M,
                          W.fp16)
                timed("gemm_ffn1", 2.0 * M * D_FF * D_MODEL, gemm, h16, lay["f1"], M, D_FF,
                      D_MODEL, EPI_BIAS_RELU, bias=lay["f1_b"], out16=ff, fp16=W.fp16)
                if self.resid16:
                    timed("gemm_ffn2", 2.0 * M * D_MODEL * D_FF, gemm, ff, lay["f2"], M, D_MODEL,
                          D_FF, EPI_RESID_ADD16, bias=lay["f2_b"], out16=h16, fp16=W.fp16)
                    timed("layernorm", 0.0, layernorm16, h16, lay["n2_w"], lay["n2_b"], M,
                          W.fp16)
                else:
                    timed("gemm_ffn2", 2.0 * M * D_MODEL * D_FF, gemm, ff, lay["f2"], M, D_MODEL,
                          D_FF, EPI_RESID_ADD, bias=lay["f2_b"], out32=h32, fp16=W.fp16)
                    timed("layernorm", 0.0, layernorm, h32, h16, lay["n2_w"], lay["n2_b"], M,
                          W.fp16)
            timed("gemm_head", 2.0 * M * (D_HEAD_MLP * D_MODEL + E * D_HEAD_MLP), self._head,
                  h16, y, out[r0:r0 + M], M)
        return out

    def _head(self, h16, y, out, M):
        W = self.weights
        gemm(h16, W.h1_w, M, D_HEAD_MLP, D_MODEL, EPI_BIAS_GELU, bias=W.h1_b, out16=y,
             fp16=W.fp16)
        gemm(y, W.h2_w, M, self.shape.num_experts, D_HEAD_MLP, EPI_F32, bias=W.h2_b, out32=out,
             fp16=W.fp16)

    def predict_masks(self, packed: PackedTraces, budget: int, warmup: int = 0, metrics=None,
                      logits=None, timing=None):
        z = self.forward_logits(packed, logits, timing)
        E = self.shape.num_experts
        masks = torch.empty((packed.rows, self.shape.mask_words), dtype=torch.int64,
                            device=packed.device)
        nat.call("moeb_mask_head", nat.ptr(z), packed.rows, E, int(budget),
                 int(bool(self.threshold)), nat.ptr(masks), nat.stream_ptr())
        if metrics is not None:
            from .metrics import mask_metrics
            mask_metrics(masks, packed.truth, packed.row_off, self.shape.num_layers, E, warmup,
                         metrics)
        return masks
