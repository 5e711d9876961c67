"""Verify timing vs flash-decoding key splits of the tensor-core attention."""
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
for sp in (1, 0, 2, 4):
    lib.sb_set_attention_splits(sp)
    r = [f"b{b}k{k}={eng.time_verify(b, k, ctx=192, reps=20):.3f}" for b, k in [(1, 3), (1, 8), (4, 3), (8, 1), (8, 3), (8, 8)]]
    d = f"draft b8 {eng.time_draft_step(8, ctx=192, reps=30) * 1e3:.1f}us"
    print(f"attn_splits={sp}: verify ms " + " ".join(r) + " | " + d, flush=True)
lib.sb_set_attention_splits(0)
