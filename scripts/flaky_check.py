"""Repeat the fp32 batch-invariance check (tests/test_gpu_model.py) to catch races."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.engine import SequenceState
from paper_2310_18813_b200.decoder import tiny_pair

dev = torch.device("cuda:0")
dt = os.environ.get("DT", "fp32")
tgt, drf = tiny_pair(dt, device=dev, seed=2, max_pos=512)
bad = 0
reps = int(os.environ.get("REPS", "20"))
for rep in range(reps):
    outs = []
    for k, graphs in [(0, True), (4, True), (4, False), (8, True)]:
        eng = SpecEngine(tgt, drf, mode="greedy", max_batch=8, max_k=8, prompt_len=12, max_new=32, seed=1,
                         use_graphs=graphs)
        states = [SequenceState(request_id=10 + i, target_len=32) for i in range(6)]
        eng.generate(states, k)
        outs.append([st.tokens for st in states])
    ok = outs[0] == outs[1] == outs[2] == outs[3]
    if not ok:
        bad += 1
        for j in range(1, 4):
            for s in range(6):
                if outs[0][s] != outs[j][s]:
                    d = next(i for i, (a, b) in enumerate(zip(outs[0][s], outs[j][s])) if a != b)
                    print(f"rep {rep} variant {j} seq {s} first diff at {d}: {outs[0][s][d:d+4]} vs {outs[j][s][d:d+4]}")
print(f"{dt}: {bad}/{reps} mismatching reps")
