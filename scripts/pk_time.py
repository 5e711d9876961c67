"""Verify / draft-step timing (CUDA graph replay, CUDA events): persistent
single-kernel forward vs per-layer kernels."""
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
W = tgt.cfg.streamed_bytes_per_forward(2)
for pk in (1, 0):
    lib.sb_set_persistent(pk)
    row = []
    for b, k in [(1, 3), (1, 8), (4, 3), (8, 1), (8, 3), (8, 8)]:
        ms = eng.time_verify(b, k, ctx=192, reps=20)
        T = b * (k + 1)
        byts = W + tgt.cfg.kv_bytes_per_token(2) * (b * 192 + T) + 4 * 32000 * T
        row.append(f"b{b}k{k}={ms:.3f}ms({byts / ms / 1e9:.0f}GB/s)")
    d = " ".join(f"b{b}={eng.time_draft_step(b, ctx=192, reps=50) * 1e3:.1f}us" for b in (1, 8))
    print(f"persistent={pk}: verify " + " ".join(row) + f" | draft step {d}", flush=True)
lib.sb_set_persistent(1)
