"""Config-5 trace: formed-batch adaptive serving vs continuous batching with
several admission-batching rules (wall clock, time-compressed)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.policy import AdaptivePolicy, build_lut
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.serving import serve_continuous
from paper_2310_18813_b200.simulator import ServerConfig, serve_wallclock
from paper_2310_18813_b200.spec_engine import SpecEngine
from paper_2310_18813_b200.traffic import PhaseSchedule, TrafficConfig, gen_phased
dev = torch.device("cuda:0")
scale = float(os.environ.get("TS", "0.1"))
trace = example_trace()
tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, seed=0, init="device", max_pos=320)
drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
eng = SpecEngine(tgt, drf, mode="injected", acceptance=trace, max_batch=16, max_k=8, prompt_len=128, max_new=128)
lut = build_lut(None, trace, s_grid=range(9), profiled_sizes=(1, 2, 4, 8, 16), mode="measured", sample_size=1,
                rng=np.random.default_rng(0), gen_len=128, engine=eng)
for bb in range(1, 17):
    for kk in range(1, 9):
        eng._graph(bb, kk)
NPH = int(os.environ.get("NPH", "6"))
phases = tuple((50.0, TrafficConfig(mean_interval=0.2 if i % 2 == 0 else 1.0, cv=1.0, count=1000)) for i in range(NPH))
wl = gen_phased(PhaseSchedule(phases=phases), np.random.default_rng([0, 6]), gen_len=128)
pol = AdaptivePolicy(lut)
out = {}
rep = serve_wallclock(wl, ServerConfig(policy=pol, max_batch=16), eng, time_scale=scale)
out["formed"] = rep.avg_latency / scale
print("formed", out["formed"], flush=True)
for riding in (True, False):
    rep, ex = serve_continuous(wl, eng, pol, time_scale=scale, max_batch=16, riding=riding)
    out[f"cont_riding{int(riding)}"] = (rep.avg_latency / scale, ex)
    print("riding", riding, out[f"cont_riding{int(riding)}"], flush=True)
print("SUMMARY " + json.dumps(out))
