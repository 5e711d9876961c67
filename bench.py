"""Benchmark: batched speculative decoding, Llama-2-7B target + LLaMA-68M draft,
bf16, one B200 per rank (BASELINE.json configs[2]; replicas across GPUs).

A "step" = one formed batch of b=8 requests (P=128 prompt, N=128 new tokens)
run to completion through SpecEngine.generate at the adaptive k chosen by the
b->k LUT (profiled on this GPU), incl. prefill.  value = generated tokens/s
(whole job, all ranks).  Acceptance is INJECTED from the reference's
example_trace (TraceSampler law): random weights give ~0 real acceptance, the
draft/verify/accept/commit work is real.  Inputs (13.5 GB of weights) exceed
the 126 MB L2, so no explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# workload -> (target, draft): "7b" = BASELINE configs[2] (the headline), "70b" =
# configs[3] (Llama-2-70B; tensor-parallel over the ranks when launched with
# torchrun --nproc-per-node N, whole model on one B200 at N=1)
WORKLOADS = {"7b": ("llama-2-7b", "llama-68m"), "70b": ("llama-2-70b", "llama-160m"),
             "opt": ("opt-6.7b", "opt-125m"), "trace": ("llama-2-7b", "llama-68m")}
TARGET, DRAFT = WORKLOADS["7b"]
B, P, NEW = 8, 128, 128
K_GRID = tuple(range(9))


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=B)
    ap.add_argument("--k", type=int, default=-1, help="fixed k (default: adaptive LUT)")
    ap.add_argument("--quick", action="store_true", help="skip the k sweep")
    ap.add_argument("--workload", default="7b", choices=sorted(WORKLOADS))
    ap.add_argument("--trace-scale", type=float, default=0.1,
                    help="config 5: wall seconds per trace second (0.1 = the 6 x 50 s schedule in 30 s)")
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1650.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def verify_bytes(cfg, b, k, ctx_avg):
    """Algorithmic bytes of one verify forward: weights streamed
    once + KV read (all cached keys of every sequence) + KV write for the
    b(k+1) new tokens + fp32 logits + embedding gather."""
    T = b * (k + 1)
    w = cfg.streamed_bytes_per_forward(2)
    kv_tok = cfg.kv_bytes_per_token(2)
    return w + kv_tok * b * ctx_avg + kv_tok * T + 4 * cfg.vocab * T + 2 * cfg.hidden * T


# ============================================================== reference arm (CPU)
def cpu_sample(b, k, iters=1, threads=None, layers=None):
    """The CPU oracle (oracle/model_ref.py forward_batch, fp32, all host
    threads) running the same speculative iteration -- draft k steps + verify
    b(k+1) tokens of the full 7B/68M pair, batched over the b sequences -- on a
    bounded sample (`iters` iterations after an untimed prefill).  Weights are a
    tiled random block (timing only; CPU parity is tested on the tiny pair).
    Returns (tokens/s, description, cores)."""
    import torch

    from oracle import model_ref, spec_ref
    from paper_2310_18813_b200.decoder import CONFIGS
    from paper_2310_18813_b200.presets import example_trace

    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    tc, dc = CONFIGS[TARGET], CONFIGS[DRAFT]
    L = tc.n_layers if layers is None else layers
    block = torch.empty(1 << 20).uniform_(-0.035, 0.035, generator=torch.Generator().manual_seed(0))

    def mk(*shape):
        n = int(np.prod(shape))
        reps = (n + block.numel() - 1) // block.numel()
        return block.repeat(reps)[:n].view(*shape).clone()

    def masters(cfg, n_layers):
        h, hd = cfg.hidden, cfg.head_dim
        return {"embed": mk(cfg.vocab, h), "lm_head": mk(cfg.vocab, h), "gf": 1 + mk(h),
                "layers": [{"wq": mk(cfg.n_heads * hd, h), "wk": mk(cfg.n_kv_heads * hd, h),
                            "wv": mk(cfg.n_kv_heads * hd, h), "wo": mk(h, cfg.n_heads * hd), "wg": mk(cfg.ffn, h),
                            "wu": mk(cfg.ffn, h), "wd": mk(h, cfg.ffn), "ga": 1 + mk(h), "gm": 1 + mk(h)}
                           for _ in range(n_layers)]}

    def opt_masters(cfg, n_layers):
        h, F = cfg.hidden, cfg.ffn
        lay = lambda: dict(wq=mk(h, h), wk=mk(h, h), wv=mk(h, h), bq=mk(h), bk=mk(h), bv=mk(h), wo=mk(h, h),
                           bo=mk(h), f1=mk(F, h), b1=mk(F), f2=mk(h, F), b2=mk(h), g1=1 + mk(h), c1=mk(h),
                           g2=1 + mk(h), c2=mk(h))
        return {"embed": mk(cfg.vocab, h), "pos": mk(P + NEW + 32, h), "layers": [lay() for _ in range(n_layers)],
                "gf": 1 + mk(h), "cf": mk(h)}

    def build(cfg, n_layers):
        if cfg.arch == "opt":
            return model_ref.OptRef(opt_masters(cfg, n_layers), cfg.n_heads, cfg.rms_eps, dtype=torch.float32)
        return model_ref.LlamaRef(masters(cfg, n_layers), cfg.n_heads, cfg.n_kv_heads, cfg.rms_eps,
                                  max_pos=P + NEW + 16, dtype=torch.float32)

    t_init = time.perf_counter()
    tgt = build(tc, L)
    drf = build(dc, dc.n_layers)
    rng = np.random.default_rng(0)
    prompts = [list(map(int, rng.integers(0, tc.vocab, P))) for _ in range(b)]
    tcache = [tgt.new_cache() for _ in range(b)]
    dcache = [drf.new_cache() for _ in range(b)]
    pre = [p[:P - 1] for p in prompts]
    ppos = [list(range(P - 1))] * b
    model_ref.forward_batch(tgt, pre, ppos, tcache)
    model_ref.forward_batch(drf, pre, ppos, dcache)
    t_init = time.perf_counter() - t_init
    trace = example_trace()
    toks = [list(p) for p in prompts]
    gen = 0
    t0 = time.perf_counter()
    for it in range(iters):
        l_inj = np.minimum(spec_ref.injected_lengths(0, it, b, trace.samples), k)
        ns = [len(t) for t in toks]
        drafts = [[] for _ in range(b)]
        if k > 0:
            lg = model_ref.forward_batch(drf, [t[n - 2:n] for t, n in zip(toks, ns)], [[n - 2, n - 1] for n in ns],
                                         dcache)[:, -1]
            for j in range(1, k + 1):
                if j > 1:
                    lg = model_ref.forward_batch(drf, [[d[-1]] for d in drafts], [[n - 2 + j] for n in ns],
                                                 dcache)[:, -1]
                for s in range(b):
                    drafts[s].append(int(np.argmax(lg[s])))
        tl = model_ref.forward_batch(tgt, [[t[n - 1]] + d for t, n, d in zip(toks, ns, drafts)],
                                     [list(range(n - 1, n + k)) for n in ns], tcache)
        for s in range(b):
            l = int(l_inj[s])
            new = drafts[s][:l] + [int(np.argmax(tl[s, l]))]
            toks[s].extend(new)
            gen += len(new)
    dt = time.perf_counter() - t0
    desc = (f"{iters} speculative iteration(s) (b={b}, k={k}, injected example_trace acceptance, prompt {P}) of the "
            f"fp32 CPU oracle pair {TARGET}+{DRAFT} batched over sequences ({L}/{tc.n_layers} target layers"
            f"{'' if L == tc.n_layers else ', time scaled by layer count'}); weight init + prefill {t_init:.1f}s untimed")
    if L != tc.n_layers:
        dt *= tc.n_layers / L
    return gen / dt, desc, threads


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    k = args.k if args.k >= 0 else 3
    layers = int(os.environ.get("SB_CPU_LAYERS", "8")) or None
    tps, desc, cores = cpu_sample(args.batch, k, iters=max(1, min(args.steps, 3)), layers=layers)
    v = float(tps)
    line = {"metric": "generated tokens/s (batched speculative decoding)", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "impl": "reference", "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{TARGET}+{DRAFT} b={args.batch} k={k} P={P} N={NEW}"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "vs_baseline": None}
    print(json.dumps(line), flush=True)



# ============================================================== config 5 (serving trace)
def run_trace(args):
    """BASELINE configs[4]: a time-varying Poisson trace (the reference's
    timeline schedule, harness.py:257-265: alternating intense 0.2 s / sparse
    1.0 s mean gaps, CV 1, 6 x 50 s phases, max_batch 16) replayed in WALL
    time on the GPU engine (simulator.serve_wallclock), once with the adaptive
    LUT policy and once per fixed k = 1..8.  Metric: mean request latency
    (queueing + prefill + decode), lower is better.  The schedule is time
    compressed by --trace-scale so one policy takes ~30 s."""
    import torch

    from paper_2310_18813_b200.decoder import CONFIGS, Decoder
    from paper_2310_18813_b200.policy import AdaptivePolicy, FixedPolicy, build_lut
    from paper_2310_18813_b200.presets import example_trace
    from paper_2310_18813_b200.simulator import ServerConfig, serve_wallclock
    from paper_2310_18813_b200.spec_engine import SpecEngine
    from paper_2310_18813_b200.traffic import PhaseSchedule, TrafficConfig, gen_phased

    rank, world, local = _dist()
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    trace = example_trace()
    tgt = Decoder(CONFIGS[TARGET], dtype="bf16", device=dev, seed=0, init="device", max_pos=P + NEW + 32)
    drf = Decoder(CONFIGS[DRAFT], dtype="bf16", device=dev, seed=1, init="device", max_pos=P + NEW + 32)
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=trace, max_batch=16, max_k=8, prompt_len=P,
                     max_new=NEW, seed=0)
    lut = build_lut(None, trace, s_grid=K_GRID, profiled_sizes=(1, 2, 4, 8, 16), mode="measured",
                    sample_size=1, rng=np.random.default_rng(0), gen_len=NEW, engine=eng)
    phases = tuple((50.0, TrafficConfig(mean_interval=0.2 if i % 2 == 0 else 1.0, cv=1.0, count=1000))
                   for i in range(6))
    workload = gen_phased(PhaseSchedule(phases=phases), np.random.default_rng([0, 6]), gen_len=NEW)
    policies = [AdaptivePolicy(lut)] + [FixedPolicy(k) for k in range(1, 9)]
    lat, batches = {}, {}
    t_cap = time.perf_counter()
    for bb in range(1, 17):  # capture every (b, k) iteration graph up front: no capture inside a replay
        for kk in range(1, 9):
            eng._graph(bb, kk)
    t_cap = time.perf_counter() - t_cap
    t_run = time.perf_counter()
    for pol in policies:
        rep = serve_wallclock(workload, ServerConfig(policy=pol, max_batch=16), eng, time_scale=args.trace_scale)
        lat[pol.label] = rep.avg_latency / args.trace_scale  # back to trace seconds
        sizes = [r.served_batch_size for r in rep.records]
        batches[pol.label] = round(float(np.mean(sizes)), 2)
    # continuous batching: retire / admit every iteration, k from the LUT per iteration
    from paper_2310_18813_b200.serving import serve_continuous
    cont = {}
    for pol in [AdaptivePolicy(lut), FixedPolicy(3)]:
        rep, extra = serve_continuous(workload, eng, pol, time_scale=args.trace_scale, max_batch=16)
        cont[pol.label] = {"latency_s": round(rep.avg_latency / args.trace_scale, 4),
                           "mean_live_batch": round(extra["mean_live_batch"], 2), "mean_k": round(extra["mean_k"], 2),
                           "riding_prefill_rows": extra["ridden_rows"], "separate_prefill_rows": extra["prefill_rows"]}
    t_run = time.perf_counter() - t_run
    fixed = {k: v for k, v in lat.items() if k.startswith("fixed")}
    best = min(fixed, key=fixed.get)
    ad = [k for k in lat if k not in fixed][0]
    line = {"metric": "mean request latency, phased Poisson trace (adaptive k)", "value": lat[ad], "unit": "s",
            "n_gpus": 1, "higher_is_better": False, "impl": "ours", "dtype": "bf16",
            "data": "synthetic (random-init weights, injected example_trace acceptance)",
            "config": {"workload": f"{TARGET} target + {DRAFT} draft, timeline trace 6x50s (0.2/1.0 s gaps, CV 1), "
                                   f"max_batch 16, N={NEW}, P={P}", "time_scale": args.trace_scale,
                       "requests": len(workload), "lut": {str(k): v for k, v in lut.entries.items()}},
            "latency_s_by_policy": {k: round(v, 4) for k, v in lat.items()},
            "mean_batch_by_policy": batches, "best_fixed": best,
            "adaptive_vs_best_fixed_latency": lat[ad] / fixed[best], "wall_s": round(t_run, 1),
            "continuous_batching": cont,
            "graph_capture_s": round(t_cap, 1)}
    print(json.dumps(line), flush=True)

# ============================================================== our arm (GPU)
def run_ours(args):
    import torch

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    from paper_2310_18813_b200 import _native as N
    from paper_2310_18813_b200.decoder import CONFIGS, Decoder
    from paper_2310_18813_b200.engine import SequenceState, run_batch
    from paper_2310_18813_b200.policy import build_lut, lookup
    from paper_2310_18813_b200.presets import example_trace
    from paper_2310_18813_b200.profiler import calibrate
    from paper_2310_18813_b200.replicas import max_over_ranks
    from paper_2310_18813_b200.spec_engine import SpecEngine

    b = args.batch
    trace = example_trace()
    tp = args.workload == "70b" and world > 1  # tensor-parallel target over the ranks (config 4)
    if tp:
        from paper_2310_18813_b200.tp import NcclTP, shard_config

        # each rank draws its own shard directly (random init; no full copy anywhere)
        tgt = Decoder(shard_config(CONFIGS[TARGET], world), dtype="bf16", device=dev, seed=100 + rank,
                      init="device", max_pos=P + NEW + 32)
        tgt.world, tgt.rank = world, rank
        ids = [NcclTP.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(ids, src=0)
        tp_group = NcclTP(world, rank, ids[0])
        tp_group.attach(tgt)
    else:
        tgt = Decoder(CONFIGS[TARGET], dtype="bf16", device=dev, seed=0, init="device", max_pos=P + NEW + 32)
    drf = Decoder(CONFIGS[DRAFT], dtype="bf16", device=dev, seed=1, init="device", max_pos=P + NEW + 32)
    # replicas: independent request streams per rank; TP: one engine spanning the ranks (same seed)
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=trace, max_batch=max(b, 8), max_k=8, prompt_len=P,
                     max_new=NEW, seed=0 if tp else rank)

    # ---- the paper's profiler on THIS GPU: every (b, k) cell runs the real
    # engine (build_lut mode="measured"); the analytic LUT from a measured
    # LinearStepModel calibration is reported beside it.
    cal, samples = calibrate(eng, batch_sizes=(1, 2, 4, 8), k_grid=range(1, 9), reps=5)
    lut_analytic = build_lut(cal, trace, s_grid=K_GRID, profiled_sizes=(1, 2, 4, 8))
    sizes = tuple(x for x in (1, 2, 4, 8) if x <= b) if not args.quick else (b,)
    lut = build_lut(None, trace, s_grid=K_GRID, profiled_sizes=sizes, mode="measured", sample_size=1,
                    rng=np.random.default_rng(0), gen_len=NEW, engine=eng)
    k = args.k if args.k >= 0 else lookup(lut, b).chosen_s
    cells = lut.provenance.get("ms_per_token", {})
    sweep = {int(key.split(",")[1]): 1e3 / v for key, v in cells.items() if int(key.split(",")[0]) == b}
    # the metric is "tokens/s vs batch size (adaptive k vs best fixed k)": every profiled b
    by_batch = {}
    for bb in sorted({int(key.split(",")[0]) for key in cells}):
        row = {int(key.split(",")[1]): 1e3 / v for key, v in cells.items() if int(key.split(",")[0]) == bb}
        kb_ = lookup(lut, bb).chosen_s
        bf = max(row, key=row.get)
        by_batch[str(bb)] = {"adaptive_k": kb_, "adaptive_tokens_per_s": round(row[kb_], 1), "best_fixed_k": bf,
                             "best_fixed_tokens_per_s": round(row[bf], 1),
                             "k_sweep": {str(kk): round(v, 1) for kk, v in sorted(row.items())}}

    def batch(step):
        return [SequenceState(request_id=step * 1000 + i, target_len=NEW) for i in range(b)]

    # ---- warmup + timed steps (device time, CUDA events around whole generate incl. prefill)
    for w in range(args.warmup):
        eng.generate(batch(80000 + w), k)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    step_ms, decode_ms, iters, launches = [], [], 0, 0
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        for s in range(args.steps):
            res = eng.generate(batch(s), k)
            step_ms.append(res.total_time + eng.stats.prefill_ms)
            decode_ms.append(res.total_time)
            iters += res.steps
            launches += res.steps * eng.stats.kernels_per_iteration
        e1.record(eng.stream)
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    total_ms = max_over_ranks(total_ms, device=dev)
    jobs = 1 if tp else world  # TP: the ranks share one batch
    tokens = jobs * args.steps * b * NEW
    value = tokens / (total_ms / 1e3)

    # ---- e2e through the public API (SpecEngine.generate(batch, k) -- the north_star's
    # call): each step's prompts H2D from pinned host memory inside the timed region,
    # generated tokens D2H into the caller's SequenceStates (wall clock)
    pinned = [torch.from_numpy(np.stack([eng.prompt_fn(st.request_id) for st in batch(100 + s)])).pin_memory()
              for s in range(args.steps)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(args.steps):
        sts = batch(100 + s)
        res = eng.generate(sts, k, prompts=pinned[s])
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    # the reference-facing path (run_batch, engine.py:176) gives the same streams
    chk = batch(100)
    run_batch(chk, k, None, eng, np.random.default_rng(0))
    e2e = jobs * args.steps * b * NEW / e2e_s

    # ---- config 3 names stochastic rejection sampling: the same pair in stochastic mode
    # (REAL acceptance of the random-init weights at temperature 1, canonical inverse-CDF
    # resampling, materialised fp32 logits/probabilities), device-timed
    stoch = None
    if not tp:
        eng_s = SpecEngine(tgt, drf, mode="stochastic", max_batch=max(b, 8), max_k=8, prompt_len=P, max_new=NEW,
                           seed=rank, autotune=False)
        eng_s.generate(batch(90000), k)
        ms_s, acc_s, prop_s = 0.0, 0, 0
        for s in range(2):
            r = eng_s.generate(batch(91000 + s), k)
            ms_s += r.total_time + eng_s.stats.prefill_ms
            log = eng_s.stats.accepted
            acc_s += int(log[log >= 0].sum())
            prop_s += int(k * (log >= 0).sum())
        stoch = {"tokens_per_s": 2 * b * NEW / (ms_s / 1e3), "k": k,
                 "acceptance_rate": acc_s / max(prop_s, 1), "acceptance": "real (random-init pair, T=1)"}
        del eng_s
        torch.cuda.empty_cache()

    # ---- roofline of the verify forward (the north_star's roofline object), timed live
    hbm, tf, peak_kind = _peaks()
    ctx_avg = P + NEW // 2
    vb = verify_bytes(tgt.cfg, b, k, ctx_avg)
    v_ms = eng.time_verify(b, k, ctx=ctx_avg, reps=20)
    achieved = vb / (v_ms / 1e3) / 1e9
    verify_by_batch = {}  # north_star: >= 60% of the HBM roofline for verification at b <= 8
    for bb in (1, 2, 4, 8):
        if bb > eng.max_batch:
            continue
        kb_ = lookup(lut, bb).chosen_s if str(bb) in by_batch else k
        ms_ = eng.time_verify(bb, kb_, ctx=ctx_avg, reps=10)
        verify_by_batch[str(bb)] = {"k": kb_, "verify_ms": round(ms_, 4),
                                    "frac_hbm": round(verify_bytes(tgt.cfg, bb, kb_, ctx_avg) / (ms_ / 1e3) / 1e9 / hbm, 4)}
    traffic = None
    tf_path = ROOT / "profiles" / "verify_traffic.json"
    if tf_path.exists():
        tfd = json.loads(tf_path.read_text())
        if tfd.get("b") == b and tfd.get("k") == k and str(tfd.get("workload", "")).startswith(TARGET + " "):
            traffic = tfd["dram_bytes_read_plus_write"]

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and os.environ.get("SB_SKIP_CPU", "0") != "1":
        try:
            layers = int(os.environ.get("SB_CPU_LAYERS", "8" if TARGET == "llama-2-7b" else "2")) or None
            tps, desc, cores = cpu_sample(b, k, iters=1, layers=layers)
            cpu = {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        best_fixed = max(sweep, key=sweep.get) if sweep else None  # sweep: decode tokens/s of the batch
        line = {
            "metric": "generated tokens/s (batched speculative decoding, adaptive k)", "value": value,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong" if tp else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, random prompts)",
            "config": {"workload": f"{TARGET} target + {DRAFT} draft, bf16, b={b}, P={P}, N={NEW}",
                       "k": k, "k_source": "adaptive LUT (profiled on this GPU)" if args.k < 0 else "fixed",
                       "lut": {str(kk): v for kk, v in lut.entries.items()},
                       "lut_analytic_from_measured_calibration": {str(kk): v for kk, v in lut_analytic.entries.items()},
                       "acceptance": "injected: TraceSampler(example_trace()) law on device",
                       "parallelism": f"tp{world} (NCCL all-reduce / all-gather)" if tp else f"replicas x{world}",
                       "l2": "inputs (weights >= 13.5 GB) > L2; no flush"},
            "decode_tokens_per_s": jobs * args.steps * b * NEW / (sum(decode_ms) / 1e3) if world == 1 else None,
            "k_sweep_decode_tokens_per_s": {str(kk): round(v, 1) for kk, v in sorted(sweep.items())},
            "tokens_per_s_by_batch": by_batch,
            "verify_roofline_by_batch": verify_by_batch,
            "best_fixed_k": best_fixed,
            "adaptive_vs_best_fixed": (sweep[k] / sweep[best_fixed]) if (sweep and k in sweep) else None,
            "iterations_per_step": iters / args.steps,
            "gpu_launches": launches,
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": b * P * 4 + b * 4,
                    "d2h_bytes_per_step": b * eng.cap * 4 + b * 4 * 2 + eng.log_cap * b * 4 + 4 * 8,
                    "api": "SpecEngine.generate(batch, k, prompts=pinned) (wall clock)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "kernel": f"verify forward b={b} k={k}",
                         "algorithmic_bytes": vb, "verify_ms": v_ms, "peak_kind": peak_kind,
                         "frac_of_8TBs": achieved / 8000.0},
            "cpu_baseline": cpu,
            "stochastic": stoch,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    a = _args()
    TARGET, DRAFT = WORKLOADS[a.workload]
    if a.impl == "reference":
        run_reference(a)
    elif a.workload == "trace":
        run_trace(a)
    else:
        run_ours(a)
