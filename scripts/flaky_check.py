"""Repeat spec-vs-plain equality checks (tests/test_gpu_model.py) to catch
races / nondeterminism.  DT=fp32|bf16, KS=comma list of k (first is the
reference), SEED, REPS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.decoder import tiny_pair
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.spec_engine import SpecEngine

dev = torch.device("cuda:0")
dt = os.environ.get("DT", "fp32")
ks = [int(x) for x in os.environ.get("KS", "0,4,8").split(",")]
seed = int(os.environ.get("SEED", "2"))
B = int(os.environ.get("B", "6"))
tgt, drf = tiny_pair(dt, device=dev, seed=seed, max_pos=512)
print("head_dim", tgt.cfg.hidden // tgt.cfg.n_heads, "heads", tgt.cfg.n_heads, tgt.cfg.n_kv_heads)
bad = 0
reps = int(os.environ.get("REPS", "10"))
for rep in range(reps):
    outs = []
    for k in ks:
        eng = SpecEngine(tgt, drf, mode="greedy", max_batch=int(os.environ.get("MB", "8")), max_k=int(os.environ.get("MK", "8")), prompt_len=16, max_new=24, seed=3)
        states = [SequenceState(request_id=i, target_len=24) for i in range(B)]
        eng.generate(states, k)
        outs.append([st.tokens for st in states])
    diffs = []
    for j in range(1, len(ks)):
        for s in range(B):
            if outs[0][s] != outs[j][s]:
                d = next(i for i, (a, b) in enumerate(zip(outs[0][s], outs[j][s])) if a != b)
                diffs.append((ks[j], s, d))
    if diffs:
        bad += 1
        print(f"rep {rep}: (k, seq, first diff) {diffs}")
print(f"{dt}: {bad}/{reps} reps with mismatches")
