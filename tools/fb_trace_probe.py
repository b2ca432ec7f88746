"""Timeline of the persistent attention kernel's first items on CTA 0 (needs
a library built with -DFB_TRACE, selected through MOEB_LIB)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_17137_b200 import _native as nat  # noqa: E402

nwin = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rows = nwin * 512
qkv = torch.randn(rows, 1536, device="cuda").half()
out = torch.empty(rows, 512, device="cuda", dtype=torch.half)
ws = torch.arange(nwin, device="cuda", dtype=torch.int64) * 512
wl = torch.full((nwin,), 512, device="cuda", dtype=torch.int32)
lib = nat.load_library()
buf = (ctypes.c_ulonglong * 16384)()
for rep in range(3):
    nat.call("moeb_window_attention", nat.ptr(qkv), nat.ptr(out), nat.ptr(ws), nat.ptr(wl), nwin,
             512, rows, 1, nat.stream_ptr())
    torch.cuda.synchronize()
    n = lib.moeb_debug_fb_trace(buf, 16384)
ev = np.array(buf[:n], dtype=np.uint64)
ev = ev[ev != 0]
code = (ev >> np.uint64(56)).astype(int)
chunk = ((ev >> np.uint64(48)) & np.uint64(0xff)).astype(int)
clk = (ev & np.uint64(0xffffffffffff)).astype(np.int64)
o = np.argsort(clk, kind="stable")
t0 = clk[o[0]]
names = {1: "mma:s_begin", 2: "mma:S0 issued", 3: "mma:S1 issued", 4: "mma:pv_begin",
         5: "mma:PV0 issued", 6: "mma:PV1 issued", 7: "mma:Q test (c = done + 2 t)", 8: "mma:item start", 9: "mma:Q0 ready",
         10: "mma:Q1 ready", 11: "mma:K ready", 12: "tma:q_empty wait", 13: "tma:Q issued",
         14: "tma:kv_empty wait", 15: "tma:KV issued"}
for t in (0, 1):
    for k, nm in enumerate(["wait_S", "S_ready", "ld_done", "exp_done", "pempty_ok", "P_arrived",
                            "wait_O", "O_ready"]):
        names[16 + 8 * t + k] = f"sm{t}:{nm}"
prev = t0
for i in o[:400]:
    print(f"{clk[i] - t0:8d} (+{clk[i] - prev:5d})  c={chunk[i]:2d}  {names.get(code[i], code[i])}")
    prev = clk[i]
