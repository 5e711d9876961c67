"""Draft step time with the heuristic GEMM plans vs the measured (autotuned) ones."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128, max_new=128)
def row(tag):
    r = [f"b{b}={eng.time_draft_step(b, ctx=192, reps=30) * 1e3:.1f}us" for b in (1, 2, 4, 8)]
    print(tag, " ".join(r), flush=True)
row("heuristic")
drf.autotune(set(range(1, 17)))
row("tuned")
