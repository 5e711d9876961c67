"""Time K1 (one-launch draft loop, sb_draft_loop) against the per-step draft
forwards it replaces: LLaMA-68M bf16, graph-replayed, per draft step (us).
Optionally flush L2 (256 MB write) before every replay (--flush) to see the
cold-weight case (the target verify between iterations streams 13 GB)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_18813_b200 import _native as N  # noqa: E402
from paper_2310_18813_b200.decoder import CONFIGS, Decoder  # noqa: E402

N.load()
N.init_device()
dev = torch.device("cuda:0")
flush = "--flush" in sys.argv
cfg = CONFIGS["llama-68m"]
drf = Decoder(cfg, dtype="bf16", device=dev, seed=1, init="device", max_pos=512)
lib = N.load()
i32 = dict(device=dev, dtype=torch.int32)
import os
P = int(os.environ.get('DL_P', '192'))
kv = drf.new_kv(8, 320)
ws = torch.zeros(max(drf.workspace_bytes(8 * P), int(lib.sb_draft_loop_workspace_bytes(C.byref(drf.struct)))),
                 device=dev, dtype=torch.uint8)
slots = torch.arange(8, **i32)
sync = torch.zeros(8, device=dev, dtype=torch.int64)
packed = torch.empty(int(lib.sb_draft_loop_packed_bytes(C.byref(drf.struct))), device=dev, dtype=torch.uint8)
N.call("sb_draft_loop_pack", C.byref(drf.struct), N.ptr(packed), packed.numel(), torch.cuda.current_stream().cuda_stream)
junk = torch.empty(256 << 20, device=dev, dtype=torch.uint8)
st = torch.cuda.Stream()


def setup(b):
    prompts = np.random.default_rng(b).integers(0, 32000, size=(b, P)).astype(np.int32)
    drf.forward(kv, torch.as_tensor(prompts[:, :P - 1].reshape(-1), **i32), slots, torch.arange(P - 1, **i32).repeat(b),
                b, P - 1, None, N.LOGITS_NONE, ws)
    d1_ids = torch.as_tensor(prompts[:, P - 2:].reshape(-1), **i32)
    d1_pos = torch.tensor([P - 2, P - 1] * b, **i32)
    d_base = torch.full((b,), P - 1, **i32)
    return d1_ids, d1_pos, d_base


def timed(fn, reps=50):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            fn()
        g.replay()
        ts = []
        for _ in range(reps):
            if flush:
                junk.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


RUN = "--no-run" not in sys.argv
for b in ((1, 2, 4, 8) if RUN else ()):
    d1_ids, d1_pos, d_base = setup(b)
    for k in (1, 3, 8):
        v_ids = torch.zeros(b * (k + 1), **i32)
        ds_ids = torch.zeros(b, **i32)
        ds_pos = torch.zeros(b, **i32)

        def loop():
            s = torch.cuda.current_stream().cuda_stream
            rc = lib.sb_draft_loop(C.byref(drf.struct), C.byref(kv.struct), N.ptr(packed), b, k, N.ptr(d1_ids), N.ptr(d1_pos),
                                   N.ptr(slots), N.ptr(d_base), N.ptr(v_ids), N.ptr(ds_ids), N.ptr(ds_pos),
                                   N.ptr(ws), ws.numel(), N.ptr(sync), s)
            assert rc == 0, rc

        def per_step():
            s = torch.cuda.current_stream().cuda_stream
            for j in range(1, k + 1):
                ids, pos, q = (d1_ids, d1_pos, 2) if j == 1 else (ds_ids, ds_pos, 1)
                sink = N.SbTokenSink(v_ids.data_ptr() + j * 4, k + 1, ds_ids.data_ptr(), ds_pos.data_ptr(),
                                     d_base.data_ptr(), j)
                drf.forward_greedy(kv, ids, slots, pos, b, q, None, N.LOGITS_LAST, ws, sink, s)

        t_loop = timed(loop)
        t_step = timed(per_step)
        print(f"b={b} k={k}: loop {t_loop * 1e3:8.1f} us ({t_loop * 1e3 / k:6.1f} us/step) | "
              f"per-step {t_step * 1e3:8.1f} us ({t_step * 1e3 / k:6.1f} us/step){' [L2 flushed]' if flush else ''}",
              flush=True)
