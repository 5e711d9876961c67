"""Repro harness: a reduced-depth target + a draft through generate() at several (b, k)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
T, D = os.environ.get("TGT", "llama-2-70b"), os.environ.get("DRF", "llama-160m")
tgt = Decoder(replace(CONFIGS[T], n_layers=int(os.environ.get("TL", "2"))), dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS[D], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128, max_new=int(os.environ.get("NEW", "32")))
for b in (1, 2, 4, 8):
    for k in range(9):
        states = [SequenceState(request_id=i, target_len=int(os.environ.get("NEW", "32"))) for i in range(b)]
        eng.generate(states, k)
        torch.cuda.synchronize()
        print("ok", T, D, b, k, flush=True)
