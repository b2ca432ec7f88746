"""Packed decode traces in HBM and the on-device synthetic generator.

Layout: one uint64 bitmask row per (prompt, token,
layer) step, W = ceil(E/64) words per row, prompts concatenated in (token,
layer) order -- CSR over prompts with ``row_off[P+1]``. A DeepSeek-V2-Lite
trace token (26 layers) is 208 bytes; the ~66 M-row C2 workload is 528 MB.

``generate_packed`` reproduces the reference generator (traceio.py:208-283)
bit for bit: the host replays the two small leading draw blocks with numpy
itself (hot-key draws + np.argpartition ordering, token ids) and hands the
PCG64 state to ``moeb_gen_traces``, which jumps straight to each token's
slice of the large draw blocks on device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import math

import numpy as np
import torch

from . import _native as nat
from .core import ConfigError, ModelShape, PromptTrace, RangeError, TokenRecord

_TOKEN_VOCAB = 32000  # traceio.py:230


@dataclass(frozen=True)
class GeneratorConfig:
    """Synthetic trace generator settings (traceio.py:197-227), same validation."""

    num_prompts: int
    tokens_per_prompt: int
    shape: ModelShape
    hot_set_size: int
    skew: float
    seed: int
    first_prompt_id: int = 0

    def __post_init__(self):
        if self.num_prompts < 1:
            raise ConfigError(f"num_prompts must be >= 1, got {self.num_prompts}")
        if self.tokens_per_prompt < 1:
            raise ConfigError(f"tokens_per_prompt must be >= 1, got {self.tokens_per_prompt}")
        if not self.shape.top_k <= self.hot_set_size <= self.shape.num_experts:
            raise ConfigError(f"hot_set_size must be in [{self.shape.top_k}, "
                              f"{self.shape.num_experts}], got {self.hot_set_size}")
        if not 0.0 <= self.skew <= 1.0:
            raise ConfigError(f"skew must be in [0, 1], got {self.skew}")
        if self.seed < 0:
            raise ConfigError(f"seed must be non-negative, got {self.seed}")
        if self.first_prompt_id < 0:
            raise ConfigError(f"first_prompt_id must be non-negative, got {self.first_prompt_id}")


@dataclass
class PackedTraces:
    """Traces resident on one device as bitmask rows (CSR over prompts)."""

    shape: ModelShape
    truth: torch.Tensor            # int64 [rows, W] (uint64 bit patterns), device
    row_off: torch.Tensor          # int64 [P+1], device
    row_off_host: np.ndarray       # int64 [P+1]
    prompt_ids: np.ndarray         # int64 [P]
    token_ids: torch.Tensor | None = None  # int32 [rows // L] per trace token, device
    meta: dict = field(default_factory=dict)

    @property
    def num_prompts(self) -> int:
        return len(self.prompt_ids)

    @property
    def rows(self) -> int:
        return int(self.row_off_host[-1])

    @property
    def num_tokens(self) -> np.ndarray:
        return np.diff(self.row_off_host) // self.shape.num_layers

    @property
    def device(self) -> torch.device:
        return self.truth.device

    def select(self, lo: int, hi: int) -> "PackedTraces":
        """Prompts [lo, hi) as a new PackedTraces (views where possible)."""
        r0, r1 = int(self.row_off_host[lo]), int(self.row_off_host[hi])
        L = self.shape.num_layers
        off = self.row_off_host[lo:hi + 1] - r0
        meta = {k: v for k, v in self.meta.items() if k not in ("embeddings", "row_token_ids")}
        return PackedTraces(
            self.shape, self.truth[r0:r1], torch.as_tensor(off, device=self.device),
            off, self.prompt_ids[lo:hi],
            None if self.token_ids is None else self.token_ids[r0 // L:r1 // L], meta)

    def reorder(self, order) -> "PackedTraces":
        """Prompts in the given order (a gather of whole prompts on device)."""
        order = np.asarray(order, dtype=np.int64)
        L = self.shape.num_layers
        lens = np.diff(self.row_off_host)[order]
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = np.concatenate([np.arange(self.row_off_host[i], self.row_off_host[i + 1])
                              for i in order]) if len(order) else np.zeros(0, np.int64)
        idx_d = torch.from_numpy(idx).to(self.device)
        tok = None
        if self.token_ids is not None:
            tok = self.token_ids[torch.div(idx_d[::L], L, rounding_mode="floor")]
        return PackedTraces(self.shape, self.truth[idx_d].contiguous(),
                            torch.from_numpy(off).to(self.device), off, self.prompt_ids[order],
                            tok, {})

    def to(self, device) -> "PackedTraces":
        """The same prompts on another device (one copy of the mask rows)."""
        device = torch.device(device)
        if device == self.device:
            return self
        return PackedTraces(self.shape, self.truth.to(device), self.row_off.to(device),
                            self.row_off_host, self.prompt_ids,
                            None if self.token_ids is None else self.token_ids.to(device),
                            {k: v for k, v in self.meta.items()
                             if k not in ("embeddings", "row_token_ids")})

    def shard(self, rank: int, world: int) -> "PackedTraces":
        """Contiguous prompt range of this rank with ~equal row counts."""
        if world <= 1:
            return self
        targets = np.arange(1, world) * (self.rows / world)
        cuts = np.searchsorted(self.row_off_host, targets)
        bounds = [0] + [int(c) for c in cuts] + [self.num_prompts]
        return self.select(bounds[rank], bounds[rank + 1])

    # A PackedTraces is also a read-only sequence of PromptTrace (the type the
    # reference's parse_trace_csv / generate_synthetic return), materialised
    # one prompt at a time.
    def __len__(self) -> int:
        return self.num_prompts

    def __getitem__(self, i):
        if isinstance(i, slice):
            lo, hi, step = i.indices(self.num_prompts)
            if step != 1:
                return [self[k] for k in range(lo, hi, step)]
            return self.select(lo, max(lo, hi))
        if i < 0:
            i += self.num_prompts
        if not 0 <= i < self.num_prompts:
            raise IndexError(i)
        return self._prompt(i, *self._host_views())

    def __iter__(self):
        views = self._host_views()
        for i in range(self.num_prompts):
            yield self._prompt(i, *views)

    def _host_views(self):
        truth = self.truth.cpu().numpy().view(np.uint64)
        toks = None if self.token_ids is None else self.token_ids.cpu().numpy()
        rtok = self.meta.get("row_token_ids")
        rtok = None if rtok is None else rtok.cpu().numpy()
        emb = {}
        if "embeddings" in self.meta:
            from .traceio import row_embeddings
            emb = row_embeddings(self)
        return truth, toks, rtok, emb

    def _prompt(self, i, truth, toks, rtok, emb) -> PromptTrace:
        L, E = self.shape.num_layers, self.shape.num_experts
        pid = int(self.prompt_ids[i])
        tr = PromptTrace(pid)
        r0, r1 = int(self.row_off_host[i]), int(self.row_off_host[i + 1])
        for r in range(r0, r1):
            ids = []
            for w, word in enumerate(truth[r]):
                word = int(word)
                while word:
                    b = word & -word
                    ids.append(w * 64 + b.bit_length() - 1)
                    word ^= b
            t, l = (r - r0) // L, (r - r0) % L
            tid = int(rtok[r]) if rtok is not None else (0 if toks is None else int(toks[r // L]))
            tr.records.append(TokenRecord(pid, t, l, tuple(e for e in ids if e < E), tid,
                                          emb.get(r, ())))
        return tr

    def unpack(self) -> list[PromptTrace]:
        """Host PromptTrace objects (slow; for compatibility and small cases)."""
        return list(self)


def _device(device):
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def pack_traces(traces, shape: ModelShape, device=None) -> PackedTraces:
    """Pack host PromptTrace objects (validated like the reference) to device rows."""
    if isinstance(traces, PackedTraces):
        return traces
    nat.load_library()
    device = _device(device)
    L, W = shape.num_layers, shape.mask_words
    offs = [0]
    pids = []
    rows = []
    toks = []
    for tr in traces:
        if tr.records and (tr.records[0].token_index != 0 or tr.records[0].layer_id != 0):
            tr = PromptTrace(tr.prompt_id, sorted(tr.records,
                                                  key=lambda r: (r.token_index, r.layer_id)))
        n = len(tr.records)
        if n % L:
            raise RangeError(f"prompt {tr.prompt_id}: incomplete layer coverage")
        for j, rec in enumerate(tr.records):
            if rec.token_index != j // L or rec.layer_id != j % L:
                raise RangeError(f"prompt {tr.prompt_id}: records not a complete (token, layer) "
                                 f"grid at position {j}")
            # the reference's own record check (core.py:84-104): exactly top_k
            # distinct in-range ids -- a bitmask row cannot carry a duplicate
            # id, so such a record is rejected instead of silently collapsed
            rec.validate(shape)
            m = [0] * W
            for e in rec.expert_ids:
                m[e >> 6] |= 1 << (e & 63)
            rows.append(m)
            if j % L == 0:
                toks.append(rec.token_id)
        offs.append(offs[-1] + n)
        pids.append(tr.prompt_id)
    arr = np.array(rows, dtype=np.uint64).reshape(-1, W) if rows else np.zeros((0, W), np.uint64)
    off = np.array(offs, dtype=np.int64)
    return PackedTraces(
        shape, torch.from_numpy(arr.view(np.int64)).to(device), torch.from_numpy(off).to(device),
        off, np.array(pids, dtype=np.int64),
        torch.tensor(toks, dtype=torch.int32, device=device))


def _prompt_prep(cfg: GeneratorConfig, pid: int):
    """Host part of traceio._generate_prompt: the hot-key block (and the
    argpartition order of the hot set) and the token-id block."""
    shape = cfg.shape
    L, E, T, h = shape.num_layers, shape.num_experts, cfg.tokens_per_prompt, cfg.hot_set_size
    rng = np.random.default_rng(np.random.SeedSequence(cfg.seed, spawn_key=(pid,)))
    hot_keys = rng.random((L, E))
    token_ids = rng.integers(0, _TOKEN_VOCAB, size=T)
    st = rng.bit_generator.state["state"]
    hot = np.argpartition(-hot_keys, h - 1, axis=1)[:, :h]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    return (np.array([s >> 64, s & m64, inc >> 64, inc & m64], dtype=np.uint64),
            hot.astype(np.uint8), token_ids.astype(np.int32))


def generate_packed(config: GeneratorConfig, device=None) -> PackedTraces:
    """All prompts of a generator config, generated on device (bit-identical
    to traceio.generate_synthetic)."""
    nat.load_library()
    device = _device(device)
    shape = config.shape
    L, E, k = shape.num_layers, shape.num_experts, shape.top_k
    T, P, h = config.tokens_per_prompt, config.num_prompts, config.hot_set_size
    if E > 256 or k > 16:
        raise ConfigError("device generator supports E <= 256 and top_k <= 16")
    pids = np.arange(config.first_prompt_id, config.first_prompt_id + P, dtype=np.int64)
    states = np.empty((P, 4), dtype=np.uint64)
    hots = np.empty((P, L, h), dtype=np.uint8)
    toks = np.empty((P, T), dtype=np.int32)
    for i, pid in enumerate(pids):
        states[i], hots[i], toks[i] = _prompt_prep(config, int(pid))
    W = shape.mask_words
    truth = torch.empty((P * T * L, W), dtype=torch.int64, device=device)
    st_d = torch.from_numpy(states.view(np.int64)).to(device)
    hot_d = torch.from_numpy(hots).to(device)
    with torch.cuda.device(device):
        nat.call("moeb_gen_traces", nat.ptr(st_d), nat.ptr(hot_d), P, T, L, E, k, h,
                 float(config.skew), nat.ptr(truth), nat.stream_ptr())
    off = np.arange(P + 1, dtype=np.int64) * (T * L)
    return PackedTraces(shape, truth, torch.from_numpy(off).to(device), off, pids,
                        torch.from_numpy(toks.reshape(-1)).to(device),
                        {"generator": config})


def generate_synthetic(config: GeneratorConfig) -> list[PromptTrace]:
    """traceio.generate_synthetic (traceio.py:277-283), computed on device."""
    return generate_packed(config).unpack()


def masks_to_ids(truth: torch.Tensor, k: int) -> torch.Tensor:
    """One-word expert masks [rows] (or [rows][1]) -> the compact wire format:
    k expert ids per row, u8, ascending, 0xff padding (moeb_masks_to_ids)."""
    t = truth.reshape(-1).contiguous()
    ids = torch.empty((t.numel(), int(k)), dtype=torch.uint8, device=t.device)
    bad = torch.zeros(1, dtype=torch.int32, device=t.device)
    nat.call("moeb_masks_to_ids", nat.ptr(t), t.numel(), int(k), nat.ptr(ids), nat.ptr(bad),
             nat.stream_ptr())
    if int(bad.item()):
        raise RangeError(f"a row has more than {k} experts")
    return ids


def rank_bits(num_experts: int, k: int) -> int:
    """Width of a row's combinatorial rank: ceil(log2 C(E, k)) (27 for 64 / 6)."""
    return max(1, (math.comb(int(num_experts), int(k)) - 1).bit_length())


def packed_rank_words(rows: int, bits: int) -> int:
    """u32 words of a packed rank stream of `rows` rows (+1 padding word)."""
    return (rows * bits + 31) // 32 + 1


def masks_to_ranks(truth: torch.Tensor, k: int, num_experts: int,
                   packed: bool = False) -> torch.Tensor:
    """One-word expert masks -> the rank wire format: each row's rank in the
    combinatorial number system (sum_i C(c_i, i) over its ascending ids), as
    int32 holding the u32 rank (moeb_masks_to_ranks, 4 B/row) or, with
    `packed`, as a dense bit stream of rank_bits(E, k) bits per row
    (moeb_masks_to_packed_ranks, 27 bits = 3.4 B/row for 64 / 6). Every row
    must carry exactly k experts, as a validated reference trace row does."""
    if math.comb(int(num_experts), int(k)) >= 2**32 or num_experts > 64 or k > 8:
        raise ConfigError(f"rank wire format needs C(E, k) < 2^32, E <= 64, k <= 8")
    t = truth.reshape(-1).contiguous()
    bad = torch.zeros(1, dtype=torch.int32, device=t.device)
    if packed:
        bits = rank_bits(num_experts, k)
        out = torch.zeros(packed_rank_words(t.numel(), bits), dtype=torch.int32,
                          device=t.device)
        nat.call("moeb_masks_to_packed_ranks", nat.ptr(t), t.numel(), int(k),
                 int(num_experts), bits, nat.ptr(out), nat.ptr(bad), nat.stream_ptr())
    else:
        out = torch.empty(t.numel(), dtype=torch.int32, device=t.device)
        nat.call("moeb_masks_to_ranks", nat.ptr(t), t.numel(), int(k), int(num_experts),
                 nat.ptr(out), nat.ptr(bad), nat.stream_ptr())
    if int(bad.item()):
        raise RangeError(f"a row does not have exactly {k} experts")
    return out


def ranks_to_masks(ranks: torch.Tensor, k: int, num_experts: int, out: torch.Tensor,
                   bad: torch.Tensor, rows: int | None = None):
    """Device decode of rank rows into masks: `ranks` holds one u32 per row
    (moeb_ranks_to_masks) or, when `rows` is given and differs from its
    length, the packed bit stream of `rows` rows (moeb_packed_ranks_to_masks).
    bad[0] is set to 1 (asynchronously) if a rank is >= C(E, k)."""
    n = ranks.shape[0] if rows is None else int(rows)
    if n == ranks.shape[0]:
        nat.call("moeb_ranks_to_masks", nat.ptr(ranks), n, int(k), int(num_experts),
                 nat.ptr(out), nat.ptr(bad), nat.stream_ptr())
    else:
        nat.call("moeb_packed_ranks_to_masks", nat.ptr(ranks), n,
                 rank_bits(num_experts, k), int(k), int(num_experts), nat.ptr(out),
                 nat.ptr(bad), nat.stream_ptr())
    return out


def ids6_words(rows: int, k: int) -> int:
    """u32 words of a packed 6-bit id stream of `rows` rows (+2 padding words)."""
    return (rows * 6 * k + 31) // 32 + 2


def masks_to_ids6(truth: torch.Tensor, k: int) -> torch.Tensor:
    """One-word expert masks -> the packed-id wire format: each row's k
    ascending ids at 6 bits (E <= 64) in a bit stream, 4.5 B per row at k = 6
    (moeb_masks_to_ids6), as int32 words (StreamingReplay.run(wire="ids6")
    decodes them with moeb_ids6_to_masks). Every row must carry exactly k
    experts, as a validated reference trace row does."""
    if k > 8:
        raise ConfigError("the packed-id wire format takes k <= 8")
    t = truth.reshape(-1).contiguous()
    out = torch.zeros(ids6_words(t.numel(), k), dtype=torch.int32, device=t.device)
    bad = torch.zeros(1, dtype=torch.int32, device=t.device)
    nat.call("moeb_masks_to_ids6", nat.ptr(t), t.numel(), int(k), nat.ptr(out), nat.ptr(bad),
             nat.stream_ptr())
    if int(bad.item()):
        raise RangeError(f"a row does not have exactly {k} experts")
    return out


def ids6_to_masks(words: torch.Tensor, k: int, rows: int, out: torch.Tensor, bad: torch.Tensor):
    """Device decode of a packed 6-bit id stream into masks; bad[0] is set to 1
    (asynchronously) if a row does not hold k distinct experts."""
    nat.call("moeb_ids6_to_masks", nat.ptr(words), int(rows), int(k), nat.ptr(out), nat.ptr(bad),
             nat.stream_ptr())
    return out


def idpair_bits(k: int) -> int:
    """Bits per row of the packed id-pair format: 11 per sorted pair, 6 for an
    odd k's last id (33 at k = 6)."""
    return 11 * (k // 2) + 6 * (k % 2)


def idpair_words(rows: int, k: int) -> int:
    """u32 words of a packed id-pair stream of `rows` rows (+2 padding words)."""
    return (rows * idpair_bits(k) + 31) // 32 + 2


def masks_to_idpairs(truth: torch.Tensor, k: int) -> torch.Tensor:
    """One-word expert masks -> the packed id-pair wire format: each row's
    ascending ids two at a time, a sorted pair (a < b) as C(b, 2) + a in 11
    bits (4.125 B per row at k = 6; moeb_masks_to_idpairs), as int32 words
    (StreamingReplay.run(wire="idpairs") decodes them with
    moeb_idpairs_to_masks: three lookups into a 4 KB table per row). Every row
    must carry exactly k experts, as a validated reference trace row does."""
    if k > 8:
        raise ConfigError("the packed id-pair wire format takes k <= 8")
    t = truth.reshape(-1).contiguous()
    out = torch.zeros(idpair_words(t.numel(), k), dtype=torch.int32, device=t.device)
    bad = torch.zeros(1, dtype=torch.int32, device=t.device)
    nat.call("moeb_masks_to_idpairs", nat.ptr(t), t.numel(), int(k), nat.ptr(out), nat.ptr(bad),
             nat.stream_ptr())
    if int(bad.item()):
        raise RangeError(f"a row does not have exactly {k} experts")
    return out


def idpairs_to_masks(words: torch.Tensor, k: int, rows: int, out: torch.Tensor,
                     bad: torch.Tensor):
    """Device decode of a packed id-pair stream into masks; bad[0] is set to 1
    (asynchronously) if a row does not hold k distinct experts."""
    nat.call("moeb_idpairs_to_masks", nat.ptr(words), int(rows), int(k), nat.ptr(out),
             nat.ptr(bad), nat.stream_ptr())
    return out


def ids_to_masks(ids: torch.Tensor, num_experts: int, out: torch.Tensor, bad: torch.Tensor):
    """Device decode of the compact rows into masks (moeb_ids_to_masks); bad[0]
    is set to 1 (asynchronously) if an id is >= num_experts."""
    nat.call("moeb_ids_to_masks", nat.ptr(ids), ids.shape[0], ids.shape[1], int(num_experts),
             nat.ptr(out), nat.ptr(bad), nat.stream_ptr())
    return out
