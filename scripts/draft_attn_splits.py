"""Draft step (68M) time vs the decode attention's flash-decoding key splits
(sb_set_attention_splits: 1 off, 0 auto, n forced), and the target verify for reference."""
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
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=16, max_k=8, prompt_len=128,
                 max_new=128)
lib = N.load()
for rep in range(2):
    for s in (1, 0, 2, 4):
        lib.sb_set_attention_splits(s)
        d = {b: eng.time_draft_step(b, ctx=192, reps=100) * 1e3 for b in (1, 2, 4, 8, 16)}
        v = {b: eng.time_verify(b, 7 if b <= 8 else 3, ctx=192, reps=10) for b in (1, 8)}
        print(f"splits={s}: draft step us " + " ".join(f"b={b}:{x:.1f}" for b, x in d.items()) +
              " | verify ms " + " ".join(f"b={b}:{x:.3f}" for b, x in v.items()), flush=True)
lib.sb_set_attention_splits(1)
