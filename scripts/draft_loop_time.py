"""Speculative-iteration time (CUDA graph replay): one-launch draft loop vs
per-step draft forwards (7B target + 68M draft, injected acceptance)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context, _timed_graph
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
lib = N.load()
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128,
                 max_new=128)
for enabled in (0, 1):
    lib.sb_set_draft_loop(enabled)
    row = []
    for b, k in [(1, 3), (1, 8), (4, 3), (8, 1), (8, 3), (8, 5)]:
        _stage_context(eng, b, k, 192)
        it_ms = _timed_graph(lambda: eng._iteration(b, k), 10, eng.stream)
        v_ms = eng.time_verify(b, k, ctx=192, reps=10)
        row.append(f"b{b}k{k}: iter {it_ms:.3f} (draft+token {it_ms - v_ms:.3f})")
    print(f"draft_loop={enabled}: " + " | ".join(row), flush=True)
lib.sb_set_draft_loop(0)
