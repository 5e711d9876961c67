"""OPT-6.7B (+125M draft) verify-forward time per (b, k) (graph replay), for A/B of library builds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["opt-6.7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["opt-125m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128,
                 max_new=128)
print(" | ".join(f"b={b},k={k}: {min(eng.time_verify(b, k, ctx=192, reps=20) for _ in range(3)):.3f} ms"
                 for b, k in [(1, 8), (4, 7), (8, 3), (8, 7)]), flush=True)
