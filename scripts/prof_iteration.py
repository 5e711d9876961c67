"""One speculative iteration of the headline engine (Llama-2-7B + LLaMA-68M, bf16, injected
acceptance) as the bench runs it: graph-captured (b, k), replayed inside an NVTX range "iter" so
ncu can select exactly those launches:
  ncu --nvtx --nvtx-include "iter/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,... \
      python scripts/prof_iteration.py
PB / PK: batch and speculation length (default 8 / 3); PREPS: replays inside the range (default 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2310_18813_b200.decoder import CONFIGS, Decoder  # noqa: E402
from paper_2310_18813_b200.presets import example_trace  # noqa: E402
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context  # noqa: E402

b = int(os.environ.get("PB", "8"))
k = int(os.environ.get("PK", "3"))
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, seed=0, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
PMODE = os.environ.get("PMODE", "injected")  # injected | greedy | stochastic
eng = SpecEngine(tgt, drf, mode=PMODE, acceptance=example_trace() if PMODE == "injected" else None, max_batch=8,
                 max_k=8, prompt_len=128,
                 max_new=128, seed=0)
_stage_context(eng, b, k, 192)
g = eng._graph(b, k)
with torch.cuda.stream(eng.stream):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"iteration b={b} k={k}: {e0.elapsed_time(e1) / 10:.3f} ms (graph replay, {eng.kernels_per_iteration(b, k)} kernels)")
    torch.cuda.nvtx.range_push("iter")
    for _ in range(int(os.environ.get("PREPS", "1"))):
        g.replay()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
