"""Verify time (b=8, k=3) with one GEMM shape's tuned plan overridden
(sb_gemm_tune_set): PLANS="N,K,cps,splits,wt,tn;..." for T = b(k+1)."""
import ctypes as C, os, sys
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
b, k = int(os.environ.get("B", "8")), int(os.environ.get("K", "3"))
T = b * (k + 1)
def cur(n, kk):
    v = [C.c_int32() for _ in range(4)]
    rc = N.load().sb_gemm_tune_get(T, n, kk, *[C.byref(x) for x in v])
    return [x.value for x in v] if rc == 0 else None
for name, (n, kk, w) in tgt.gemm_shapes().items():
    print(name, n, kk, "tuned:", cur(n, kk))
base = [eng.time_verify(b, k, ctx=192, reps=20) for _ in range(3)]
print("base", [round(x, 4) for x in base], flush=True)
for spec in os.environ.get("PLANS", "").split(";"):
    if not spec:
        continue
    n, kk, cps, sp, wt, tn = [int(x) for x in spec.split(",")]
    old = cur(n, kk)
    N.call("sb_gemm_tune_set", T, n, kk, cps, sp, wt, tn)
    t = [eng.time_verify(b, k, ctx=192, reps=20) for _ in range(3)]
    print(spec, [round(x, 4) for x in t], flush=True)
    if old:
        N.call("sb_gemm_tune_set", T, n, kk, *old)
