"""Marginal in-graph cost of each kernel class of the 68M draft step
(sb_debug_skip removes one class; outputs are garbage while skipping)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128,
                 max_new=128)
lib = N.load()
for b in (1, 8):
    base = eng.time_draft_step(b, ctx=192, reps=50) * 1e3
    row = [f"b{b} full={base:.1f}us"]
    for name, mask in [("attn", 1), ("qkv", 2), ("o", 4), ("gu", 8), ("down", 16), ("all-layer-gemms", 30), ("all-layer", 31)]:
        lib.sb_debug_skip(mask)
        t = eng.time_draft_step(b, ctx=192, reps=50) * 1e3
        lib.sb_debug_skip(0)
        row.append(f"-{name}: {t:.1f} ({(base - t) / 2:.1f} us/layer)")
    print(" | ".join(row), flush=True)
