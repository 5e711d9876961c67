"""A riding-prefill iteration (b=8 live rows at ctx 192, k=3, RIDE prompts of
127 tokens prefilled inside the verify forward) vs the plain iteration plus a
separate prefill forward: CUDA-event time of each (eager launches), for
ncu launch lists and DESIGN numbers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.serving import _prefill_rows
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=16, max_k=8, prompt_len=128,
                 max_new=128)
eng.tune_riding()
b, k, ride = 8, 3, int(os.environ.get("RIDE", "2"))
P = eng.prompt_len
rng = np.random.default_rng(0)


def stage():
    _stage_context(eng, b, k, 192)
    eng.tokens[b:b + ride, :P].copy_(torch.from_numpy(rng.integers(0, eng.V, size=(ride, P)).astype(np.int32)))
    eng.n_tok[b:b + ride].fill_(P)
    eng.produced[:b + ride].zero_()
    eng.target_len[:b + ride].fill_(128)
    torch.cuda.synchronize()


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        stage()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            e0.record()
            fn()
            e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


with torch.cuda.stream(eng.stream):
    t_ride = timed(lambda: eng._iteration(b, k, ride=ride))
    t_plain = timed(lambda: eng._iteration(b, k))
    t_sep = timed(lambda: (eng._iteration(b, k), _prefill_rows(eng, list(range(b, b + ride)))))
print(f"b={b} k={k} ride={ride}: riding iteration {t_ride:.3f} ms | plain iteration {t_plain:.3f} ms | "
      f"plain + separate prefill {t_sep:.3f} ms (eager launches)")
