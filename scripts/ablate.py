"""Verify/draft timing ablations (graph replay, CUDA events): PDL on/off, attention impl."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=8, max_k=8, prompt_len=128, max_new=128)
lib = N.load()
for pdl in (1, 0):
    for attn in (0, 1):
        lib.sb_set_pdl(pdl); lib.sb_set_attention_impl(attn)
        row = []
        for b, k in [(1, 3), (8, 1), (8, 3), (8, 8)]:
            row.append(f"b{b}k{k}={eng.time_verify(b, k, ctx=192, reps=10):.3f}")
        print(f"pdl={pdl} attn={attn}: verify ms " + " ".join(row) + f" | draft b8 {eng.time_draft_step(8, ctx=192, reps=10):.4f}", flush=True)

# per-stage warm timings of the real launch sequence (events between kernels)
import ctypes as C
from paper_2310_18813_b200.spec_engine import _stage_context
lib.sb_set_pdl(1); lib.sb_set_attention_impl(0)
for b, k in [(8, 3), (1, 3), (8, 8)]:
    _stage_context(eng, b, k, 192)
    buf = C.create_string_buffer(4096)
    for rep in range(3):
        rc = lib.sb_profile_forward(C.byref(tgt.struct), C.byref(eng.kv_t.struct), eng.v_ids.data_ptr(), eng.slots.data_ptr(),
                                    eng.v_pos.data_ptr(), b, k + 1, eng.t_logits.data_ptr(), N.LOGITS_ALL,
                                    eng.workspace.data_ptr(), eng.workspace.numel(), torch.cuda.current_stream().cuda_stream, buf, 4096)
    parts = [p.split("=") for p in buf.value.decode().strip(";").split(";")]
    tot = sum(float(v) for _, v in parts)
    print(f"b={b} k={k} eager-with-events total {tot:.3f} ms: " + " ".join(f"{t}={float(v)*1e3/ (32 if t not in ('embed','norm_f','lm_head') else 1):.1f}us" for t, v in parts), flush=True)
