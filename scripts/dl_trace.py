"""Per-phase timeline of the one-launch draft loop (globaltimer at each barrier)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=2, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128,
                 max_new=128, use_graphs=False, autotune=False)
lib = N.load()
b, k = int(os.environ.get("B", "8")), int(os.environ.get("K", "3"))
_stage_context(eng, b, k, 192)
tr = torch.zeros(256, dtype=torch.int64, device=dev)
args = lambda: (C.byref(drf.struct), C.byref(eng.kv_d.struct), b, k, N.ptr(eng.d1_ids), N.ptr(eng.d1_pos),
                N.ptr(eng.slots), N.ptr(eng.d_base), N.ptr(eng.v_ids), N.ptr(eng.ds_ids), N.ptr(eng.ds_pos),
                N.ptr(eng.workspace), eng.workspace.numel(), torch.cuda.current_stream().cuda_stream)
import ctypes as C
for _ in range(3):
    lib.sb_draft_loop(*args())
lib.sb_debug_draft_loop_trace(tr.data_ptr())
lib.sb_draft_loop(*args())
torch.cuda.synchronize()
lib.sb_debug_draft_loop_trace(None)
t = tr.cpu().numpy().astype(np.float64)
n = int((t > 0).sum())
d = np.diff(t[:n]) / 1e3
names = ["qkv", "attn", "o", "gu", "down"] * drf.cfg.n_layers + ["lm", "final"]
print(f"b={b} k={k}: total {(t[n-1]-t[0])/1e3:.1f} us over {n-1} phases")
for i, x in enumerate(d):
    print(f"  step {i // len(names) + 1} {names[i % len(names)]:>6}: {x:7.2f} us")
