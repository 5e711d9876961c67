"""Graph-replayed iteration time (ms) of the 7B/68M engine per acceptance mode at fixed (b, k):
the cost of stochastic acceptance (materialised logits, softmax, sampling) against greedy / injected."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
for mode in ("injected", "greedy", "stochastic"):
    eng = SpecEngine(tgt, drf, mode=mode, acceptance=example_trace() if mode == "injected" else None, max_batch=8,
                     max_k=8, prompt_len=128, max_new=128)
    row = []
    for b, k in [(1, 8), (8, 3), (8, 7)]:
        _stage_context(eng, b, k, 192)
        g = eng._graph(b, k)
        with torch.cuda.stream(eng.stream):
            for _ in range(3):
                _stage_context(eng, b, k, 192)
                g.replay()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                _stage_context(eng, b, k, 192)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.replay(); e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        row.append(f"b={b},k={k}: {min(ts):.3f} ms ({eng._iter_kernels.get((b, k))} launches)")
    print(f"{mode:10s} " + " | ".join(row), flush=True)
    del eng
    torch.cuda.empty_cache()
