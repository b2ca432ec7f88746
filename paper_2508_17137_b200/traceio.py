"""Trace and prediction file formats on device.

Mirrors moesim.traceio's file API (traceio.py:1-186 in the reference) --
``parse_trace_csv``, ``write_trace_csv``, ``parse_predictions``,
``write_predictions_jsonl``, ``ParseError``, ``TRACE_HEADER`` -- with the byte
work done by libmoeb kernels (csrc/ingest.cu): newline search, one-thread-
per-line parsing with Python's int()/float() grammar, duplicate-key and
prompt-grid checks, and the canonical writers. ``parse_trace_csv`` returns
``PackedTraces`` (a sequence of PromptTrace views over packed device masks)
instead of a list of Python records, so a 66 M-row trace never becomes 66 M
objects; ``parse_predictions`` returns a ``PredictionTable`` (a read-only
mapping over key-sorted device arrays) that ``make_predictor("external")``
joins onto traces on device.

Exactness. The device grammar covers ASCII input. A line outside it
(non-ASCII bytes, integers beyond int64, more than 32 expert ids, JSON beyond
flat integer objects) is flagged MOEB_LINE_HOST and only that line is parsed
here with the reference's own expressions (``_csv_record`` /
``_prediction_record``, restated from traceio.py:64-103 / :146-169). The
message of the first failing line or prompt is also formatted here from that
one line's text. Builder limits (documented in DESIGN.md): prompt_id,
token_index and layer_id must fit int64 and token_id int32.
"""

from __future__ import annotations

import json
import warnings
from collections.abc import Mapping

import numpy as np
import torch

from . import _native as nat
from .core import ModelShape, PromptTrace, RangeError, TokenRecord
from .traces import PackedTraces, _device

TRACE_HEADER = "prompt_id,token_index,layer_id,expert_ids,token_id,embedding"
StepKey = tuple[int, int, int]

LINE_OK, LINE_RANGE, LINE_SKIP, LINE_HOST = 0, 16, 30, 32
_LINE_PARSE_ERR = 1  # host-parsed line with a ParseError (any parse code < 16)


class ParseError(ValueError):
    """Malformed input file; carries the 1-based line number (traceio.py:32-37)."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


# ---------------------------------------------------------------------------
# Host restatement of one line (error messages, and lines outside the device
# grammar). traceio.py:40-44, :64-103.
# ---------------------------------------------------------------------------

def _parse_int(text: str, line: int, column: str) -> int:
    try:
        return int(text)
    except ValueError:
        raise ParseError(line, f"column {column}: {text!r} is not an integer") from None


def _csv_record(line_text: str, i: int, shape: ModelShape):
    """One data line -> (TokenRecord, validation error or None); raises the
    ParseError of the parse stage (traceio.py:68-91)."""
    fields = line_text.split(",")
    if len(fields) != 6:
        raise ParseError(i, f"expected 6 columns, got {len(fields)}")
    prompt_id = _parse_int(fields[0], i, "prompt_id")
    token_index = _parse_int(fields[1], i, "token_index")
    layer_id = _parse_int(fields[2], i, "layer_id")
    if not fields[3]:
        raise ParseError(i, "empty expert_ids")
    expert_ids = tuple(_parse_int(part, i, "expert_ids") for part in fields[3].split("|"))
    token_id = _parse_int(fields[4], i, "token_id")
    if fields[5]:
        try:
            embedding = tuple(float(part) for part in fields[5].split("|"))
        except ValueError:
            raise ParseError(i, f"bad embedding {fields[5]!r}") from None
    else:
        embedding = ()
    rec = TokenRecord(prompt_id, token_index, layer_id, expert_ids, token_id, embedding)
    try:
        rec.validate(shape)
        verr = None
    except RangeError as exc:
        verr = ParseError(i, str(exc))
    return rec, verr


def _prediction_record(line_text: str, i: int, shape: ModelShape):
    """One JSONL line -> (key, experts) or None for a blank line; raises the
    line's ParseError (traceio.py:146-166, without the duplicate check)."""
    if not line_text.strip():
        return None
    try:
        obj = json.loads(line_text)
    except json.JSONDecodeError as exc:
        raise ParseError(i, f"malformed JSON: {exc.msg}") from None
    if not isinstance(obj, dict):
        raise ParseError(i, "expected a JSON object")
    try:
        key = (int(obj["prompt_id"]), int(obj["token_index"]), int(obj["layer_id"]))
        experts = [int(e) for e in obj["experts"]]
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(i, f"bad prediction object: {exc}") from None
    for e in experts:
        if not 0 <= e < shape.num_experts:
            raise ParseError(i, f"expert {e} out of range [0, {shape.num_experts})")
    if not 0 <= key[2] < shape.num_layers:
        raise ParseError(i, f"layer {key[2]} out of range [0, {shape.num_layers})")
    return key, experts


def _grid_error(pid: int, toks: np.ndarray, layers: np.ndarray, L: int) -> RangeError:
    """PromptTrace.validate's message for one prompt's sorted, duplicate-free
    records (core.py:128-149)."""
    seen: dict[int, set[int]] = {}
    for t, l in zip(toks.tolist(), layers.tolist()):
        seen.setdefault(t, set()).add(l)
    tokens = sorted(seen)
    if tokens != list(range(len(tokens))):
        return RangeError(f"prompt {pid}: token indices not contiguous from 0")
    for t, layers_t in seen.items():
        if len(layers_t) != L:
            return RangeError(f"prompt {pid}: incomplete layer coverage at token {t} "
                              f"({len(layers_t)} of {L} layers)")
    return RangeError(f"prompt {pid}: invalid trace")  # unreachable for a failing prompt


# ---------------------------------------------------------------------------
# Device helpers.
# ---------------------------------------------------------------------------

def _upload(raw: bytes, dev) -> torch.Tensor:
    """File bytes in HBM, padded to 16 bytes (the kernels read whole vectors).
    One host->device copy straight from the bytes object (no host copies)."""
    n = len(raw)
    out = torch.empty(((n + 15) // 16) * 16 or 16, dtype=torch.uint8, device=dev)
    if n:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # read-only source buffer: only read here
            src = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8))
        out[:n].copy_(src)
    out[n:].zero_()
    return out


def _find_bytes(buf: torch.Tensor, n: int, value: int) -> torch.Tensor:
    """Ordered positions of `value` in buf[:n] (device int64)."""
    nb = (n + 65535) // 65536
    offs = torch.empty(nb + 1, dtype=torch.int64, device=buf.device)
    total = torch.empty(1, dtype=torch.int64, device=buf.device)
    nat.call("moeb_count_bytes", nat.ptr(buf), n, value, nat.ptr(offs), nat.ptr(total),
             nat.stream_ptr())
    cnt = int(total.item())
    pos = torch.empty(max(cnt, 1), dtype=torch.int64, device=buf.device)
    if cnt:
        nat.call("moeb_find_bytes", nat.ptr(buf), n, value, nat.ptr(offs), nat.ptr(pos),
                 nat.stream_ptr())
    return pos[:cnt]


def _segment(raw: bytes, nl_host, j: int) -> bytes:
    s = 0 if j == 0 else int(nl_host[j - 1]) + 1
    e = int(nl_host[j]) if j < len(nl_host) else len(raw)
    return raw[s:e]


def _first_status(status: torch.Tensor, skip: int = 255) -> int:
    out = torch.empty(1, dtype=torch.int64, device=status.device)
    nat.call("moeb_first_status", nat.ptr(status), status.numel(), skip, nat.ptr(out),
             nat.stream_ptr())
    return int(out.item())


def _keys_check(a, b, c, status=None, n=None):
    n = a.numel() if n is None else n
    out = torch.empty(2, dtype=torch.int64, device=a.device)
    nat.call("moeb_keys_check", nat.ptr(a), nat.ptr(b), nat.ptr(c), nat.ptr(status), LINE_SKIP,
             n, nat.ptr(out), nat.stream_ptr())
    d, first_eq = out.tolist()
    return d, first_eq


def _lexsort(a, b, c):
    """Stable permutation sorting rows by (a, b, c) (device radix sorts)."""
    order = torch.argsort(c, stable=True)
    order = order[torch.argsort(b[order], stable=True)]
    return order[torch.argsort(a[order], stable=True)]


def _first_dup_unsorted(a, b, c) -> int | None:
    """Smallest row index whose key equals an earlier row's key."""
    if a.numel() < 2:
        return None
    order = _lexsort(a, b, c)
    sa, sb, sc = a[order], b[order], c[order]
    eq = (sa[1:] == sa[:-1]) & (sb[1:] == sb[:-1]) & (sc[1:] == sc[:-1])
    if not bool(eq.any()):
        return None
    return int(order[1:][eq].min().item())


def _decode_check(raw: bytes, flags: int) -> None:
    if flags & 1:
        raw.decode("utf-8")  # raises the reference's UnicodeDecodeError


# ---------------------------------------------------------------------------
# parse_trace_csv
# ---------------------------------------------------------------------------

def parse_trace_csv(data: bytes | str, shape: ModelShape, device=None) -> PackedTraces:
    """traceio.parse_trace_csv (traceio.py:47-106) on device.

    Returns the traces as PackedTraces (prompts sorted by id, rows in (token,
    layer) order), which also behaves as a sequence of PromptTrace. Raises
    ParseError / RangeError with the reference's messages for the first
    failing line / prompt."""
    nat.load_library()
    dev = _device(device)
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    n = len(raw)
    L, E, W = shape.num_layers, shape.num_experts, shape.mask_words
    buf = _upload(raw, dev)
    nl = _find_bytes(buf, n, 10)
    n_nl = nl.numel()
    nl_host = None
    n_seg = n_nl + 1
    n_lines = n_seg - (1 if (n == 0 or raw[-1:] == b"\n") else 0)
    # header (segment 0), and the data lines 1 .. n_lines-1
    first_nl = int(nl[0].item()) if n_nl else n
    header = raw[:first_nl]
    n_data = max(n_lines - 1, 0)
    status = torch.zeros(n_data, dtype=torch.uint8, device=dev)
    pid = torch.zeros(n_data, dtype=torch.int64, device=dev)
    tok = torch.zeros(n_data, dtype=torch.int64, device=dev)
    lay = torch.zeros(n_data, dtype=torch.int32, device=dev)
    masks = torch.zeros((n_data, W), dtype=torch.int64, device=dev)
    tid = torch.zeros(n_data, dtype=torch.int64, device=dev)
    emb = torch.zeros(n_data, dtype=torch.uint8, device=dev)
    flags_d = torch.zeros(1, dtype=torch.int32, device=dev)
    if n_data:
        nat.call("moeb_parse_trace_csv", nat.ptr(buf), n, nat.ptr(nl), n_nl, 1, n_data, L, E,
                 shape.top_k, nat.ptr(status), nat.ptr(pid), nat.ptr(tok), nat.ptr(lay),
                 nat.ptr(masks), nat.ptr(tid), nat.ptr(emb), nat.ptr(flags_d), nat.stream_ptr())
    flags = int(flags_d.item())
    if any(b >= 0x80 for b in header):
        flags |= 1
    _decode_check(raw, flags)
    if n_lines == 0:
        raise ParseError(1, "empty file, expected header")
    if header != TRACE_HEADER.encode():
        raise ParseError(1, f"bad header {header.decode('utf-8')!r}, expected {TRACE_HEADER!r}")

    def line_text(d: int) -> str:
        nonlocal nl_host
        if nl_host is None:
            nl_host = nl.cpu().numpy()
        return _segment(raw, nl_host, d + 1).decode("utf-8")

    # lines outside the device grammar: the reference's expressions, here
    host_rows = torch.nonzero(status == LINE_HOST).flatten().tolist() if n_data else []
    host_info: dict[int, tuple] = {}  # line -> (exception, key or None)
    for d in host_rows:
        try:
            rec, verr = _csv_record(line_text(d), d + 2, shape)
        except ParseError as exc:
            host_info[d] = (exc, None)
            status[d] = _LINE_PARSE_ERR
            continue
        key = (rec.prompt_id, rec.token_index, rec.layer_id)
        fits = all(-2**63 <= v < 2**63 for v in key[:2]) and -2**31 <= key[2] < 2**31
        if fits:
            pid[d], tok[d], lay[d] = key
        if verr is None and not (fits and -2**63 <= rec.token_id < 2**63):
            verr = RangeError(f"line {d + 2}: prompt_id / token_index / token_id beyond "
                              "int64 (device loader limit)")
        if verr is not None:
            host_info[d] = (verr, key if fits else None)
            status[d] = LINE_RANGE
            continue
        tid[d] = rec.token_id
        emb[d] = 1 if rec.embedding else 0
        flags |= 2 if rec.embedding else 0
        m = [0] * W
        for e in rec.expert_ids:
            m[e >> 6] |= 1 << (e & 63)
        masks[d] = torch.tensor(np.array(m, dtype=np.uint64).view(np.int64))
        status[d] = LINE_OK

    # first failing line: parse/validate errors and duplicate keys (the
    # duplicate check precedes TokenRecord.validate, traceio.py:92-101)
    j = _first_status(status) if n_data else 0
    first_dup = None
    if j > 0:
        desc, first_eq = _keys_check(pid, tok, lay, None, j)
        first_dup = (first_eq if first_eq < j else None) if desc == 0 else \
            _first_dup_unsorted(pid[:j], tok[:j], lay[:j])
    if j < n_data and first_dup is None and j > 0 and int(status[j].item()) >= LINE_RANGE:
        keyed = j not in host_info or host_info[j][1] is not None
        if keyed:
            k = (pid[j], tok[j], lay[j])
            if bool(((pid[:j] == k[0]) & (tok[:j] == k[1]) & (lay[:j] == k[2])).any()):
                first_dup = j
    if first_dup is not None and first_dup <= j:
        key = (int(pid[first_dup]), int(tok[first_dup]), int(lay[first_dup]))
        raise ParseError(first_dup + 2, f"duplicate record for {key}")
    if j < n_data:
        if j in host_info:
            raise host_info[j][0]
        _, verr = _csv_record(line_text(j), j + 2, shape)  # raises the parse error
        raise verr

    # all lines valid: canonical (prompt, token, layer) order
    perm = None
    if n_data > 1:
        desc, _ = _keys_check(pid, tok, lay)
        if desc:
            perm = _lexsort(pid, tok, lay)
            pid, tok, lay, masks, tid, emb = (x[perm] for x in (pid, tok, lay, masks, tid, emb))
    return _pack_rows(shape, raw, nl, pid, tok, lay, masks, tid, emb, perm, flags, dev)


def _pack_rows(shape, raw, nl, pid, tok, lay, masks, tid, emb, perm, flags, dev) -> PackedTraces:
    L = shape.num_layers
    rows = pid.numel()
    if rows == 0:
        off = np.zeros(1, dtype=np.int64)
        return PackedTraces(shape, masks, torch.from_numpy(off).to(dev), off,
                            np.zeros(0, dtype=np.int64),
                            torch.zeros(0, dtype=torch.int32, device=dev))
    fl = torch.empty(((rows + 15) // 16) * 16, dtype=torch.uint8, device=dev)
    nat.call("moeb_prompt_flags", nat.ptr(pid), rows, nat.ptr(fl), nat.stream_ptr())
    starts = _find_bytes(fl, rows, 10)
    P = starts.numel()
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    nat.call("moeb_check_grid", nat.ptr(starts), P, rows, nat.ptr(tok), nat.ptr(lay), L,
             nat.ptr(bad), nat.stream_ptr())
    b = int(bad.item())
    st_host = starts.cpu().numpy()
    if b < P:
        r0 = int(st_host[b])
        r1 = int(st_host[b + 1]) if b + 1 < P else rows
        raise _grid_error(int(pid[r0]), tok[r0:r1].cpu().numpy(), lay[r0:r1].cpu().numpy(), L)
    off = np.append(st_host, rows).astype(np.int64)
    pids = pid[starts].cpu().numpy()
    tok2 = tid.view(-1, L)
    first = tok2[:, 0]
    if bool(((first < -2**31) | (first >= 2**31)).any()):
        raise RangeError("token_id beyond int32 (device trace layout limit)")
    meta = {"source": "trace csv"}
    if not bool((tok2 == first[:, None]).all()):
        meta["row_token_ids"] = tid  # token ids that vary across a token's layers
    if flags & 2:
        rows_with = torch.nonzero(emb).flatten()
        lines = rows_with if perm is None else perm[rows_with]
        meta["embeddings"] = (raw, nl.cpu().numpy(), rows_with.cpu().numpy(),
                              lines.cpu().numpy() + 1)
    return PackedTraces(shape, masks, torch.from_numpy(off).to(dev), off, pids,
                        first.to(torch.int32).contiguous(), meta)


def row_embeddings(packed: PackedTraces) -> dict[int, tuple[float, ...]]:
    """Embeddings of a parsed trace by row (host floats, float() of the
    original text: traceio.py:86-90)."""
    info = packed.meta.get("embeddings")
    if info is None:
        return {}
    raw, nl_host, rows, segs = info
    out = {}
    for r, s in zip(rows.tolist(), segs.tolist()):
        text = _segment(raw, nl_host, s).decode("utf-8").split(",")[5]
        out[r] = tuple(float(p) for p in text.split("|"))
    return out


# ---------------------------------------------------------------------------
# write_trace_csv
# ---------------------------------------------------------------------------

def _format_floats(values) -> str:
    return "|".join(repr(float(v)) for v in values)


def _write_records_host(traces) -> bytes:
    """traceio.write_trace_csv (traceio.py:113-128) for host PromptTrace
    lists and for packed traces carrying embeddings or per-row token ids."""
    rows = []
    for trace in sorted(traces, key=lambda t: t.prompt_id):
        rows.extend(trace.records)
    rows.sort(key=lambda r: (r.prompt_id, r.token_index, r.layer_id))
    parts = [TRACE_HEADER, "\n"]
    for r in rows:
        parts.append(f"{r.prompt_id},{r.token_index},{r.layer_id},"
                     f"{'|'.join(str(e) for e in r.expert_ids)},{r.token_id},"
                     f"{_format_floats(r.embedding)}\n")
    return "".join(parts).encode("utf-8")


def _scan(lens: torch.Tensor) -> torch.Tensor:
    n = lens.numel()
    out = torch.empty(n + 1, dtype=torch.int64, device=lens.device)
    ws = torch.empty((n + 4095) // 4096 + 1, dtype=torch.int64, device=lens.device)
    nat.call("moeb_exclusive_scan_i64", nat.ptr(lens), n, nat.ptr(out), nat.ptr(ws),
             nat.stream_ptr())
    return out


def write_trace_csv(traces) -> bytes:
    """Canonical CSV bytes (traceio.py:113-128). Packed traces are formatted
    on device (sizes -> scan -> bytes)."""
    if not isinstance(traces, PackedTraces) or "embeddings" in traces.meta \
            or "row_token_ids" in traces.meta:
        return _write_records_host(traces)
    packed = traces
    if packed.num_prompts == 0 or packed.rows == 0:
        return (TRACE_HEADER + "\n").encode()
    nat.load_library()
    pids = packed.prompt_ids
    if len(pids) > 1 and not np.all(pids[1:] > pids[:-1]):
        if len(np.unique(pids)) != len(pids):
            return _write_records_host(packed.unpack())
        packed = packed.reorder(np.argsort(pids, kind="stable"))
    dev, shape = packed.device, packed.shape
    L, E = shape.num_layers, shape.num_experts
    pid_d = torch.from_numpy(np.ascontiguousarray(packed.prompt_ids)).to(dev)
    lens = torch.empty(packed.rows, dtype=torch.int64, device=dev)
    tok = packed.token_ids.contiguous() if packed.token_ids is not None else None
    nat.call("moeb_trace_csv_lengths", nat.ptr(packed.truth), nat.ptr(pid_d),
             nat.ptr(packed.row_off), packed.num_prompts, packed.rows, L, E, nat.ptr(tok),
             nat.ptr(lens), nat.stream_ptr())
    offs = _scan(lens)
    head = (TRACE_HEADER + "\n").encode()
    total = int(offs[-1].item())
    out = torch.empty(total + len(head), dtype=torch.uint8, device=dev)
    out[:len(head)] = torch.frombuffer(bytearray(head), dtype=torch.uint8).to(dev)
    body = out[len(head):]
    nat.call("moeb_trace_csv_write", nat.ptr(packed.truth), nat.ptr(pid_d),
             nat.ptr(packed.row_off), packed.num_prompts, packed.rows, L, E, nat.ptr(tok),
             nat.ptr(offs), nat.ptr(body), nat.stream_ptr())
    return out.cpu().numpy().tobytes()


# ---------------------------------------------------------------------------
# Predictions JSONL
# ---------------------------------------------------------------------------

class PredictionTable(Mapping):
    """Read-only mapping StepKey -> frozenset[int] over key-sorted device
    arrays (the reference returns a dict, traceio.py:131-170). Host views are
    built lazily on first key lookup."""

    def __init__(self, shape: ModelShape, prompt_id, token_index, layer_id, masks):
        self.shape = shape
        self.prompt_id, self.token_index, self.layer_id, self.masks = (
            prompt_id, token_index, layer_id, masks)
        self._host = None

    @classmethod
    def from_dict(cls, table: dict, shape: ModelShape, device=None) -> "PredictionTable":
        dev = _device(device)
        W, E = shape.mask_words, shape.num_experts
        keys = sorted(table)
        n = len(keys)
        k = np.array(keys, dtype=np.int64).reshape(n, 3)
        m = np.zeros((n, W), dtype=np.uint64)
        for i, key in enumerate(keys):
            for e in table[key]:
                if not 0 <= e < E:
                    raise RangeError(f"expert {e} out of range [0, {E})")
                m[i, e >> 6] |= np.uint64(1) << np.uint64(e & 63)
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
        return cls(shape, t(k[:, 0], torch.int64), t(k[:, 1], torch.int64),
                   t(k[:, 2], torch.int32), t(m.view(np.int64), torch.int64))

    def to(self, device) -> "PredictionTable":
        """The same table on another device."""
        dev = _device(device)
        return PredictionTable(self.shape, self.prompt_id.to(dev), self.token_index.to(dev),
                               self.layer_id.to(dev), self.masks.to(dev))

    def _h(self):
        if self._host is None:
            keys = torch.stack([self.prompt_id, self.token_index,
                                self.layer_id.to(torch.int64)], 1).cpu().numpy()
            masks = self.masks.cpu().numpy().view(np.uint64)
            self._host = ({tuple(int(x) for x in k): i for i, k in enumerate(keys)}, keys, masks)
        return self._host

    def __len__(self):
        return self.prompt_id.numel()

    def __iter__(self):
        _, keys, _ = self._h()
        return (tuple(int(x) for x in k) for k in keys)

    def __getitem__(self, key):
        index, _, masks = self._h()
        i = index[tuple(key)]
        out = []
        for w, word in enumerate(masks[i]):
            word = int(word)
            while word:
                b = word & -word
                out.append(w * 64 + b.bit_length() - 1)
                word ^= b
        return frozenset(out)

    def __contains__(self, key):
        return tuple(key) in self._h()[0]


def parse_predictions(data: bytes | str, shape: ModelShape, device=None) -> PredictionTable:
    """traceio.parse_predictions (traceio.py:131-170) on device."""
    nat.load_library()
    dev = _device(device)
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    n = len(raw)
    L, E, W = shape.num_layers, shape.num_experts, shape.mask_words
    buf = _upload(raw, dev)
    nl = _find_bytes(buf, n, 10)
    n_nl = nl.numel()
    n_lines = n_nl + 1
    status = torch.zeros(n_lines, dtype=torch.uint8, device=dev)
    pid = torch.zeros(n_lines, dtype=torch.int64, device=dev)
    tok = torch.zeros(n_lines, dtype=torch.int64, device=dev)
    lay = torch.zeros(n_lines, dtype=torch.int32, device=dev)
    masks = torch.zeros((n_lines, W), dtype=torch.int64, device=dev)
    flags_d = torch.zeros(1, dtype=torch.int32, device=dev)
    nat.call("moeb_parse_predictions", nat.ptr(buf), n, nat.ptr(nl), n_nl, n_lines, L, E,
             nat.ptr(status), nat.ptr(pid), nat.ptr(tok), nat.ptr(lay), nat.ptr(masks),
             nat.ptr(flags_d), nat.stream_ptr())
    _decode_check(raw, int(flags_d.item()))
    nl_host = None

    def line_text(li: int) -> str:
        nonlocal nl_host
        if nl_host is None:
            nl_host = nl.cpu().numpy()
        return _segment(raw, nl_host, li).decode("utf-8")

    host_err: dict[int, Exception] = {}
    for li in torch.nonzero(status == LINE_HOST).flatten().tolist():
        try:
            rec = _prediction_record(line_text(li), li + 1, shape)
        except ParseError as exc:
            host_err[li] = exc
            status[li] = _LINE_PARSE_ERR
            continue
        if rec is None:
            status[li] = LINE_SKIP
            continue
        key, experts = rec
        if not all(-2**63 <= v < 2**63 for v in key):
            host_err[li] = RangeError(f"line {li + 1}: prediction key beyond int64 "
                                      "(device loader limit)")
            status[li] = LINE_RANGE
            continue
        pid[li], tok[li], lay[li] = key
        m = [0] * W
        for e in experts:
            m[e >> 6] |= 1 << (e & 63)
        masks[li] = torch.tensor(np.array(m, dtype=np.uint64).view(np.int64))
        status[li] = LINE_OK

    j = _first_status(status, LINE_SKIP)
    first_dup = None
    if j > 0:
        desc, first_eq = _keys_check(pid, tok, lay, status, j)
        if desc == 0:
            first_dup = first_eq if first_eq < j else None
        else:
            keep = torch.nonzero(status[:j] == LINE_OK).flatten()
            d = _first_dup_unsorted(pid[keep], tok[keep], lay[keep])
            first_dup = None if d is None else int(keep[d].item())
    if first_dup is not None:
        key = (int(pid[first_dup]), int(tok[first_dup]), int(lay[first_dup]))
        raise ParseError(first_dup + 1, f"duplicate prediction key {key}")
    if j < n_lines:
        if j in host_err:
            raise host_err[j]
        _prediction_record(line_text(j), j + 1, shape)  # raises the range error
        raise ParseError(j + 1, "invalid prediction line")  # unreachable

    keep = torch.nonzero(status == LINE_OK).flatten()
    pid, tok, lay, masks = pid[keep], tok[keep], lay[keep], masks[keep]
    if pid.numel() > 1:
        desc, _ = _keys_check(pid, tok, lay)
        if desc:
            order = _lexsort(pid, tok, lay)
            pid, tok, lay, masks = pid[order], tok[order], lay[order], masks[order]
    return PredictionTable(shape, pid.contiguous(), tok.contiguous(), lay.contiguous(),
                           masks.contiguous())


def _write_predictions_host(table: dict) -> bytes:
    """traceio.write_predictions_jsonl (traceio.py:172-186)."""
    out = []
    for key in sorted(table):
        prompt_id, token_index, layer_id = key
        out.append(json.dumps({"prompt_id": prompt_id, "token_index": token_index,
                               "layer_id": layer_id, "experts": sorted(table[key])},
                              separators=(",", ":")))
        out.append("\n")
    return "".join(out).encode("utf-8")


def write_predictions_jsonl(table, shape: ModelShape | None = None) -> bytes:
    """Canonical JSONL (sorted by key), formatted on device for a
    PredictionTable or a dict whose experts fit a 256-expert mask."""
    if not isinstance(table, PredictionTable):
        if not table:
            return b""
        ex = [e for s in table.values() for e in s]
        emax = max(ex) if ex else 0
        if (ex and min(ex) < 0) or emax >= 256 or any(
                not all(isinstance(v, int) and -2**63 <= v < 2**63 for v in k) for k in table):
            return _write_predictions_host(table)
        if shape is None:
            shape = ModelShape(1, max(emax + 1, 1), 1)
        nat.load_library()
        table = PredictionTable.from_dict(table, ModelShape(
            max(1, shape.num_layers), max(shape.num_experts, emax + 1), 1))
    n = len(table)
    if n == 0:
        return b""
    E = table.shape.num_experts
    dev = table.masks.device
    lens = torch.empty(n, dtype=torch.int64, device=dev)
    nat.call("moeb_predictions_jsonl_lengths", nat.ptr(table.prompt_id),
             nat.ptr(table.token_index), nat.ptr(table.layer_id), nat.ptr(table.masks), n, E,
             nat.ptr(lens), nat.stream_ptr())
    offs = _scan(lens)
    out = torch.empty(int(offs[-1].item()), dtype=torch.uint8, device=dev)
    nat.call("moeb_predictions_jsonl_write", nat.ptr(table.prompt_id),
             nat.ptr(table.token_index), nat.ptr(table.layer_id), nat.ptr(table.masks), n, E,
             nat.ptr(offs), nat.ptr(out), nat.stream_ptr())
    return out.cpu().numpy().tobytes()


def join_predictions(table: PredictionTable, packed: PackedTraces):
    """Per-row predicted masks and coverage of `packed` from a key-sorted
    table (moeb_predictions_join)."""
    dev = packed.device
    W = packed.shape.mask_words
    pred = torch.zeros((packed.rows, W), dtype=torch.int64, device=dev)
    cov = torch.zeros(packed.rows, dtype=torch.uint8, device=dev)
    if packed.rows == 0:
        return pred, cov
    pids = torch.from_numpy(np.ascontiguousarray(packed.prompt_ids)).to(dev)
    tm = table.masks
    if table.shape.mask_words != W:
        raise RangeError("prediction table and traces disagree on the expert count")
    n = len(table)
    nat.call("moeb_predictions_join", nat.ptr(table.prompt_id), nat.ptr(table.token_index),
             nat.ptr(table.layer_id), nat.ptr(tm), n, nat.ptr(pids), nat.ptr(packed.row_off),
             packed.num_prompts, packed.rows, packed.shape.num_layers,
             packed.shape.num_experts, nat.ptr(pred), nat.ptr(cov), nat.stream_ptr())
    return pred, cov
