"""In-forward GEMM plan tuning (coordinate descent over the verify forward's projections): for each
(b, k) the plan (CTAs/SM, K splits, weight tiles) of qkv / o / gu / down / lm is chosen by timing the
WHOLE graph-replayed verify forward, against the isolated-GEMM autotune.  python scripts/fwd_tune.py b k ..."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine
args = [int(a) for a in sys.argv[1:]] or [8, 3, 16, 8, 32, 8]
cells = list(zip(args[0::2], args[1::2]))
dev = torch.device("cuda:0")
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=max(b for b, _ in cells),
                 max_k=8, prompt_len=128, max_new=128)
shapes = tgt.gemm_shapes()
def get(T, n, k):
    v = [C.c_int32() for _ in range(4)]
    N.call("sb_gemm_tune_get", T, n, k, *[C.byref(x) for x in v])
    return tuple(x.value for x in v)
def tv(b, k):
    return min(eng.time_verify(b, k, ctx=192, reps=10) for _ in range(2))
for b, k in cells:
    T = b * (k + 1)
    base = tv(b, k)
    cur = base
    out = [f"b={b} k={k} T={T}: isolated-autotune plan {base:.3f} ms"]
    for name in ("gu", "qkv", "down", "o", "lm"):
        n, kk, _ = shapes[name]
        rows = b if name == "lm" else T
        if name == "lm":
            continue  # (the verify lm_head rows = T as well; skip: one launch)
        orig = get(rows, n, kk)
        best, best_t = orig, cur
        cands = [(cps, sp, 1, orig[3]) for cps in (1, 2) for sp in (1, 2, 4, 8)]
        if rows >= 96:  # two weight tiles per CTA share the token stage (half the L2 token traffic per MAC)
            nt = -(-rows // 256)
            bal = (-(-rows // nt) + 15) // 16 * 16
            for tn in sorted({0, 128, 192, bal if nt > 1 else 0}):
                if tn == 0 or tn < min(256, (rows + 15) // 16 * 16):
                    cands += [(1, 1, 2, tn), (1, 1, 1, tn), (2, 1, 1, tn)]
        for c in dict.fromkeys(cands):
            if c == orig:
                continue
            if N.load().sb_gemm_tune_set(rows, n, kk, *c) != 0:
                continue
            t = tv(b, k)
            if t < best_t - 0.005:
                best, best_t = c, t
        N.call("sb_gemm_tune_set", rows, n, kk, *best)
        cur = best_t
        out.append(f"  {name}: {orig} -> {best}: {cur:.3f} ms")
    print("\n".join(out), flush=True)
