"""Transformer predictor training (paper_2508_17137_b200/transformer_train.py)
against the fp32 oracle's autograd (oracle/transformer_ref.py):
the loss, the gradient of every parameter, one AdamW step (vs
torch.optim.AdamW with the paper's groups on the same gradients), the
loss-scale overflow skip, and a short run that lowers the loss."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import paper_2508_17137_b200 as m
    from oracle import transformer_ref as R
    m.load_library()
    shape = m.ModelShape(26, 64, 6)
    packed = m.generate_packed(m.GeneratorConfig(3, 24, shape, 8, 0.9, 7))
    ref = R.TransformerRef(R.TransformerSpec(26, 64, seed=0))
    return m, R, shape, packed, ref


def _ref_loss_and_grads(R, ref, packed):
    """fp32 autograd of BCEWithLogits(mean) over every row (the oracle's
    windows, key padding), on the GPU with TF32 off."""
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda")
    ref = ref.to(dev)
    params = {n: p for n, p in ref.named_parameters() if p.requires_grad}
    for p in params.values():
        p.grad = None
    L = 26
    tok, lay = R.row_inputs(packed.token_ids.cpu().numpy(), packed.row_off_host, L)
    tok = torch.as_tensor(tok, device=dev)
    lay = torch.as_tensor(lay, device=dev)
    off = packed.row_off_host
    starts = [(s, min(s + 512, int(off[p + 1]))) for p in range(len(off) - 1)
              for s in range(int(off[p]), int(off[p + 1]), 512)]
    B = len(starts)
    ti = torch.zeros(B, 512, dtype=torch.int64, device=dev)
    li = torch.zeros(B, 512, dtype=torch.int64, device=dev)
    pad = torch.ones(B, 512, dtype=torch.bool, device=dev)
    for b, (s, e) in enumerate(starts):
        ti[b, :e - s], li[b, :e - s], pad[b, :e - s] = tok[s:e], lay[s:e], False
    x = torch.cat([ref.tok[ti], ref.layer_emb(li)], dim=-1)
    x = ref.input_proj(x)
    for layer in ref.layers:
        x = ref._encoder_layer(layer, x, pad)
    z = ref.head2(F.gelu(ref.head1(x)))
    zs = torch.cat([z[b, :e - s] for b, (s, e) in enumerate(starts)])
    truth = packed.truth.reshape(-1).cpu().numpy().view(np.uint64)
    y = torch.from_numpy(((truth[:, None] >> np.arange(64, dtype=np.uint64)) & 1)
                         .astype(np.float32)).to(dev)
    loss = F.binary_cross_entropy_with_logits(zs, y)
    loss.backward()
    names = {"input_proj.weight": "in_w", "input_proj.bias": "in_b",
             "layer_emb.weight": "layer_emb", "head1.weight": "h1_w", "head1.bias": "h1_b",
             "head2.weight": "h2_w", "head2.bias": "h2_b"}
    sub = {"self_attn.in_proj_weight": "qkv_w", "self_attn.in_proj_bias": "qkv_b",
           "self_attn.out_proj.weight": "o_w", "self_attn.out_proj.bias": "o_b",
           "linear1.weight": "f1_w", "linear1.bias": "f1_b", "linear2.weight": "f2_w",
           "linear2.bias": "f2_b", "norm1.weight": "n1_w", "norm1.bias": "n1_b",
           "norm2.weight": "n2_w", "norm2.bias": "n2_b"}
    grads = {}
    for n, p in params.items():
        if n in names:
            grads[names[n]] = p.grad.detach().clone()
        else:
            _, i, rest = n.split(".", 2)
            grads[f"l{i}.{sub[rest]}"] = p.grad.detach().clone()
    ref.to("cpu")
    return float(loss.item()), grads


def test_loss_and_gradients_match_fp32_autograd(setup):
    m, R, shape, packed, ref = setup
    from paper_2508_17137_b200 import transformer_train as TT
    tr = TT.TransformerTrainer(R.export_weights(ref), 26, 64)
    loss = tr.forward_backward(packed)
    want_loss, want = _ref_loss_and_grads(R, ref, packed)
    assert abs(loss - want_loss) < 2e-3 * abs(want_loss), (loss, want_loss)
    worst = []
    for k, g_ref in want.items():
        g = tr.grads[k] / tr.scale
        rel = float((g - g_ref).norm() / (g_ref.norm() + 1e-12))
        worst.append((rel, k, float(g_ref.norm())))
    worst.sort(reverse=True)
    print("largest relative gradient errors:", [(round(r, 4), k) for r, k, _ in worst[:6]])
    for rel, k, nrm in worst:
        assert rel < 3e-2, (k, rel, nrm)


def test_adamw_step_matches_torch(setup):
    """One optimiser step: loss-scale removal, global-norm clipping at 1.0 and
    AdamW (betas 0.9 / 0.98, decay 0.01, the paper's per-group learning
    rates) equal torch's on the same gradients."""
    m, R, shape, packed, ref = setup
    from paper_2508_17137_b200 import transformer_train as TT
    tr = TT.TransformerTrainer(R.export_weights(ref), 26, 64)
    tr.forward_backward(packed)
    before = {k: v.clone() for k, v in tr.params.items()}
    grads = {k: (g / tr.scale).clone() for k, g in tr.grads.items()}
    info = tr.optimizer_step()
    assert not info["skipped"]
    tp = {k: torch.nn.Parameter(v.clone()) for k, v in before.items()}
    for k, p in tp.items():
        p.grad = grads[k].clone()
    total = torch.nn.utils.clip_grad_norm_(list(tp.values()), 1.0)
    assert math.isclose(float(total), info["grad_norm"], rel_tol=1e-4)
    cfg = tr.cfg
    groups = {"input": cfg.lr_input, "encoder": cfg.lr_encoder, "head": cfg.lr_head}
    opt = torch.optim.AdamW([{"params": [p for k, p in tp.items() if TT._group(k) == gname],
                              "lr": lr} for gname, lr in groups.items()],
                            betas=cfg.betas, eps=cfg.eps, weight_decay=cfg.weight_decay)
    opt.step()
    for k, p in tp.items():
        torch.testing.assert_close(tr.params[k], p.detach(), atol=1e-7, rtol=1e-5)


def test_overflow_skips_step_and_halves_scale(setup):
    m, R, shape, packed, ref = setup
    from paper_2508_17137_b200 import transformer_train as TT
    tr = TT.TransformerTrainer(R.export_weights(ref), 26, 64)
    tr.forward_backward(packed)
    tr.grads["h2_b"][0] = float("inf")
    before = tr.params["h2_w"].clone()
    info = tr.optimizer_step()
    assert info["skipped"] and tr.scale == TT.TrainConfig().loss_scale / 2
    assert torch.equal(tr.params["h2_w"], before)


def test_training_lowers_loss(setup):
    m, R, shape, packed, ref = setup
    from paper_2508_17137_b200 import transformer_train as TT
    tr = TT.TransformerTrainer(R.export_weights(ref), 26, 64,
                               TT.TrainConfig(lr_input=1e-3, lr_encoder=1e-3, lr_head=1e-3))
    losses = [tr.step(packed)["loss"] for _ in range(12)]
    print("losses:", [round(x, 4) for x in losses])
    assert losses[-1] < 0.8 * losses[0]
    # the trained weights serve the inference path
    z = m.make_predictor("transformer", shape, transformer=tr.weights()).forward_logits(packed)
    assert torch.isfinite(z).all()
