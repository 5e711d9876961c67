"""Draft step time (68M, per-step forwards) with the heuristic GEMM plans vs autotuned plans."""
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
bs = (1, 2, 4, 8, 16)
before = {b: min(eng.time_draft_step(b, ctx=192, reps=20) for _ in range(3)) for b in bs}
drf.autotune(set(bs) | {2 * b for b in bs})
after = {b: min(eng.time_draft_step(b, ctx=192, reps=20) for _ in range(3)) for b in bs}
for b in bs:
    print(f"b={b}: heuristic {before[b]*1e3:.1f} us, autotuned {after[b]*1e3:.1f} us", flush=True)
