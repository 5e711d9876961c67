import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from dataclasses import replace
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _stage_context
dev = torch.device("cuda:0")
tgt = Decoder(replace(CONFIGS["llama-2-7b"], n_layers=2), dtype="bf16", device=dev, seed=3, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=4, init="device", max_pos=320)
for b in (1, 4, 8):
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=64,
                     max_new=32, seed=7, use_graphs=False, autotune=False)
    _stage_context(eng, b, 2, 150)
    for mode in (N.LOGITS_LAST, N.LOGITS_ALL):
        kv = drf.new_kv(eng.max_batch, eng.ctx_max)
        rows = b if mode == N.LOGITS_LAST else 2 * b
        lg = torch.zeros(rows, drf.cfg.vocab, device=dev)
        drf.forward(kv, eng.d1_ids, eng.slots, eng.d1_pos, b, 2, lg, mode, eng.workspace)
        torch.cuda.synchronize()
        bad = torch.isnan(lg).any(1).nonzero().flatten().tolist()
        print(b, "LAST" if mode == N.LOGITS_LAST else "ALL", "nan rows", bad, "d1_pos", eng.d1_pos[:2*b].tolist(),
              "ids", eng.d1_ids[:2*b].tolist()[:6], flush=True)
