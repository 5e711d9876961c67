"""Phase trace of K1 (sb_draft_loop) from the in-kernel globaltimer stamps
(sb_debug_draft_trace): per barrier, CTA 0's work since the previous barrier,
the slowest CTA's arrival, and the barrier exit latency after the last arrival."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_2310_18813_b200 import _native as N  # noqa: E402

sys.argv.append("--no-run")
import draft_loop_time as T  # noqa: E402  (sets up the 68M draft, KV, workspace)

KMAXG = 160
names = ["A qkv", "B attn", "C o", "D gu", "E down"]
for b, k in ((1, 3), (8, 3)):
    d1_ids, d1_pos, d_base = T.setup(b)
    v_ids = torch.zeros(b * (k + 1), **T.i32)
    ds_ids = torch.zeros(b, **T.i32)
    ds_pos = torch.zeros(b, **T.i32)
    tr = torch.zeros(4096 + 512 * KMAXG, device=T.dev, dtype=torch.int64)
    for rep in range(3):
        tr.zero_()
        N.call("sb_debug_draft_trace", tr.data_ptr() if rep == 2 else None)
        rc = T.lib.sb_draft_loop(C.byref(T.drf.struct), C.byref(T.kv.struct), N.ptr(T.packed), b, k, N.ptr(d1_ids), N.ptr(d1_pos),
                                 N.ptr(T.slots), N.ptr(d_base), N.ptr(v_ids), N.ptr(ds_ids), N.ptr(ds_pos),
                                 N.ptr(T.ws), T.ws.numel(), N.ptr(T.sync), torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
    N.call("sb_debug_draft_trace", None)
    t = tr.cpu().numpy()
    nb = k * (5 * T.cfg.n_layers + 1)
    t0 = t[0]
    prev = t0
    print(f"b={b} k={k}: total {(t[2 * nb] - t0) / 1e3:.1f} us over {nb} barriers")
    for i in range(1, nb + 1):
        arr0, ex = t[2 * i - 1], t[2 * i]
        arrs = t[4096 + i * KMAXG: 4096 + i * KMAXG + KMAXG]
        arrs = arrs[arrs > 0]
        slow = arrs.max()
        pos = (i - 1) % (5 * T.cfg.n_layers + 1)
        name = "F lm+G" if pos == 5 * T.cfg.n_layers else f"L{pos // 5} {names[pos % 5]}"
        m1, m2 = t[2048 + 4 * i + 1], t[2048 + 4 * i + 2]
        st = f"staged +{(m1 - prev) / 1e3:5.2f}" if m1 > 0 else "staged   -  "
        td = f"tiles +{(m2 - prev) / 1e3:5.2f}" if m2 > 0 else ""
        m3 = t[2048 + 4 * i + 3]
        if m3 > 0:
            td += f" attn-compute +{(m3 - prev) / 1e3:5.2f}"
        print(f"  bar {i:3d} {name:10s} cta0 work {(arr0 - prev) / 1e3:6.2f} us ({st} {td}) | slowest arrival +{(slow - prev) / 1e3:6.2f}"
              f" | exit after last {(ex - slow) / 1e3:5.2f} us | spread {(slow - arrs.min()) / 1e3:5.2f}")
        prev = ex
