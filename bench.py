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
REPEATS = 3  # independent re-timings of every (b, k) cell after the LUT is built
LUT_SIZES = (1, 2, 4, 8, 16, 32, 64)  # the reference's profiled powers of two (policy.py:72-82), to config 2's b=64
# ONE metric and ONE workload string for both arms (the driver pairs the lines by them)
METRIC = "generated tokens/s of a formed batch (prefill + speculative decode to completion), adaptive k"


def workload_str(b):
    return (f"{TARGET} target + {DRAFT} draft, b={b}, P={P}, N={NEW}, injected example_trace acceptance, "
            f"k from the b->k LUT profiled on the executing hardware")


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
    ap.add_argument("--trace-seeds", type=int, default=3, help="config 5: arrival seeds (rng [seed, 6])")
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


def verify_flops(cfg, b, k, ctx_avg):
    """Algorithmic FLOPs of one verify forward: 2 x streamed
    parameters x tokens + attention (QK^T and PV over the cached context and the
    causal window)."""
    T = b * (k + 1)
    params = cfg.streamed_bytes_per_forward(2) // 2
    attn = 4 * cfg.n_layers * cfg.n_heads * cfg.head_dim * b * (k + 1) * (ctx_avg + (k + 2) / 2)
    return 2 * params * T + attn


# ============================================================== reference arm (CPU)
def _ref_pkg():
    """The reference package itself (baseline/_ref, installed by pip from
    /root/reference; travels with the repo to the GPU box) for its cost model
    and LUT builder; our golden-identical mirror when it is absent."""
    rp = ROOT / "baseline" / "_ref"
    if (rp / "specbatch").exists():
        sys.path.insert(0, str(rp))
        import specbatch  # noqa: F401

        from specbatch.cost_model import LinearStepModel
        from specbatch.policy import build_lut, lookup
        from specbatch.presets import example_trace

        return LinearStepModel, build_lut, lookup, example_trace, "reference specbatch (baseline/_ref)"
    from paper_2310_18813_b200.cost_model import LinearStepModel
    from paper_2310_18813_b200.policy import build_lut, lookup
    from paper_2310_18813_b200.presets import example_trace

    return LinearStepModel, build_lut, lookup, example_trace, "golden-identical mirror (baseline/_ref absent)"


def iterations_needed(b, k, seed=0):
    """Iterations a formed batch of b x NEW tokens takes under the injected
    acceptance law (spec_ref.injected_lengths, the same counter RNG the GPU
    engine draws from): advance = min(l + 1, remaining) (engine.py:167)."""
    from oracle import spec_ref
    from paper_2310_18813_b200.presets import example_trace

    samples = example_trace().samples
    produced = np.zeros(b, np.int64)
    it = 0
    while np.any(produced < NEW):
        l_inj = np.minimum(spec_ref.injected_lengths(seed, it, b, samples), k)
        produced = np.minimum(produced + l_inj + 1, NEW)
        it += 1
    return it


class CpuPair:
    """The CPU oracle pair (oracle/model_ref.py, fp32, all host threads) of the
    headline shapes: a `layers`-layer slice of the target (its time is scaled
    by n_layers / layers) and the whole draft.  Weights are a tiled random
    block (timing only; CPU parity runs on the tiny pair in tests/)."""

    def __init__(self, b, layers, threads):
        import torch

        from oracle import model_ref
        from paper_2310_18813_b200.decoder import CONFIGS

        torch.set_num_threads(threads)
        self.b = b
        self.tc, self.dc = CONFIGS[TARGET], CONFIGS[DRAFT]
        self.L = self.tc.n_layers if layers is None else min(layers, self.tc.n_layers)
        self.scale = self.tc.n_layers / self.L
        block = torch.empty(1 << 20).uniform_(-0.035, 0.035, generator=torch.Generator().manual_seed(0))

        def mk(*shape):
            n = int(np.prod(shape))
            reps = (n + block.numel() - 1) // block.numel()
            return block.repeat(reps)[:n].view(*shape).clone()

        def masters(cfg, n_layers):
            h, hd = cfg.hidden, cfg.head_dim
            return {"embed": mk(cfg.vocab, h), "lm_head": mk(cfg.vocab, h), "gf": 1 + mk(h),
                    "layers": [{"wq": mk(cfg.n_heads * hd, h), "wk": mk(cfg.n_kv_heads * hd, h),
                                "wv": mk(cfg.n_kv_heads * hd, h), "wo": mk(h, cfg.n_heads * hd),
                                "wg": mk(cfg.ffn, h), "wu": mk(cfg.ffn, h), "wd": mk(h, cfg.ffn), "ga": 1 + mk(h),
                                "gm": 1 + mk(h)} for _ in range(n_layers)]}

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

        self.tgt = build(self.tc, self.L)
        self.drf = build(self.dc, self.dc.n_layers)
        self.fwd = model_ref.forward_batch
        rng = np.random.default_rng(0)
        self.prompts = [list(map(int, rng.integers(0, self.tc.vocab, P))) for _ in range(b)]
        self.reset()

    def reset(self):
        self.tcache = [self.tgt.new_cache() for _ in range(self.b)]
        self.dcache = [self.drf.new_cache() for _ in range(self.b)]
        self.toks = [list(p) for p in self.prompts]
        self.it = 0

    def prefill(self):
        """Returns seconds (target part scaled to the full depth)."""
        pre = [p[:P - 1] for p in self.prompts]
        ppos = [list(range(P - 1))] * self.b
        t0 = time.perf_counter()
        self.fwd(self.tgt, pre, ppos, self.tcache)
        t1 = time.perf_counter()
        self.fwd(self.drf, pre, ppos, self.dcache)
        t2 = time.perf_counter()
        return (t1 - t0) * self.scale + (t2 - t1)

    def iteration(self, k):
        """One speculative iteration (draft k steps + verify b(k+1) tokens +
        injected acceptance).  Returns (seconds, draft seconds, verify seconds)."""
        from oracle import spec_ref
        from paper_2310_18813_b200.presets import example_trace

        b = self.b
        l_inj = np.minimum(spec_ref.injected_lengths(0, self.it, b, example_trace().samples), k)
        ns = [len(t) for t in self.toks]
        drafts = [[] for _ in range(b)]
        t0 = time.perf_counter()
        if k > 0:
            lg = self.fwd(self.drf, [t[n - 2:n] for t, n in zip(self.toks, ns)], [[n - 2, n - 1] for n in ns],
                          self.dcache)[:, -1]
            for j in range(1, k + 1):
                if j > 1:
                    lg = self.fwd(self.drf, [[d[-1]] for d in drafts], [[n - 2 + j] for n in ns], self.dcache)[:, -1]
                for s in range(b):
                    drafts[s].append(int(np.argmax(lg[s])))
        t1 = time.perf_counter()
        tl = self.fwd(self.tgt, [[t[n - 1]] + d for t, n, d in zip(self.toks, ns, drafts)],
                      [list(range(n - 1, n + k)) for n in ns], self.tcache)
        t2 = time.perf_counter()
        for s in range(b):
            l = int(l_inj[s])
            self.toks[s].extend(drafts[s][:l] + [int(np.argmax(tl[s, l]))])
        self.it += 1
        return (t1 - t0) + (t2 - t1) * self.scale, t1 - t0, (t2 - t1) * self.scale


def cpu_reference_run(b, steps, warmup, threads=None, layers=None):
    """The reference's own method on the host CPU: calibrate the reference's
    LinearStepModel on this CPU (verify at s = 1 and 8, one draft step), let
    the reference's build_lut (analytic, example_trace acceptance) choose k
    for b, then time `steps` real iterations of the CPU oracle pair at that k
    (after `warmup` untimed ones).  The batch time is the measured prefill +
    iterations_needed(b, k) x the mean measured iteration (a bounded sample:
    the full batch would take minutes on the CPU).  Returns a dict."""
    LinearStepModel, build_lut, lookup, example_trace, ref_src = _ref_pkg()
    threads = threads or os.cpu_count()
    t_init = time.perf_counter()
    pair = CpuPair(b, layers, threads)
    t_init = time.perf_counter() - t_init
    prefill_s = pair.prefill()
    # calibration cells (each from a fresh copy of the post-prefill state would cost a second prefill:
    # the iterations simply run on; context grows by <= 9 tokens per cell, negligible vs P=128)
    it1, _, v1 = pair.iteration(1)
    it8, d8, v8 = pair.iteration(8)
    ssm = d8 / 8.0
    slope = max((v8 - v1) / 7.0, 1e-6)
    beta = max(v1 - slope, 1e-6)
    cal = LinearStepModel(alpha={b: slope * 1e3}, beta=beta * 1e3, ssm_step={b: ssm * 1e3})
    lut = build_lut(cal, example_trace(), s_grid=K_GRID, profiled_sizes=(b,))
    k = lookup(lut, b).chosen_s
    for _ in range(warmup):
        pair.iteration(k)
    times = [pair.iteration(k)[0] for _ in range(steps)]
    n_it = iterations_needed(b, k)
    batch_s = prefill_s + n_it * float(np.mean(times))
    return {"value": b * NEW / batch_s, "k": k, "threads": threads, "prefill_s": prefill_s,
            "iteration_s": times, "iterations_needed": n_it, "batch_s": batch_s,
            "calibration_ms": {"alpha": slope * 1e3, "beta": beta * 1e3, "ssm_step": ssm * 1e3},
            "lut_source": ref_src, "layers": pair.L, "init_s": t_init,
            "sample": (f"fp32 CPU oracle pair {TARGET}+{DRAFT} (target {pair.L}/{pair.tc.n_layers} layers timed, "
                       f"scaled by depth), batched over b={b} sequences: measured prefill {prefill_s:.2f} s + "
                       f"{iterations_needed(b, k)} iterations x mean of {steps} measured iterations at k={k} "
                       f"(k from the reference's build_lut on a LinearStepModel calibrated on this CPU); "
                       f"weight init {t_init:.1f} s untimed")}


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    layers = int(os.environ.get("SB_CPU_LAYERS", "8" if TARGET == "llama-2-7b" else "2")) or None
    r = cpu_reference_run(args.batch, max(1, min(args.steps, 3)), min(args.warmup, 1), layers=layers)
    v = float(r["value"])
    line = {"metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "impl": "reference", "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_str(args.batch), "k": r["k"], "k_source": r["lut_source"]},
            "ms_per_step": r["batch_s"] * 1e3,
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["threads"], "kind": "port",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {k_: r[k_] for k_ in ("prefill_s", "iteration_s", "iterations_needed", "calibration_ms")},
            "vs_baseline": None}
    print(json.dumps(line), flush=True)


# ============================================================== config 5 (serving trace)
def _ref_harness():
    """The reference's experiment harness + simulator from baseline/_ref (None if absent)."""
    rp = ROOT / "baseline" / "_ref"
    if not (rp / "specbatch").exists():
        return None
    if str(rp) not in sys.path:
        sys.path.insert(0, str(rp))
    import specbatch.cost_model as rcm
    import specbatch.harness as rh
    import specbatch.policy as rpol
    import specbatch.simulator as rsim

    return rh, rsim, rpol, rcm


def run_trace(args):
    """BASELINE configs[4]: a time-varying Poisson trace (the reference's
    timeline schedule, harness.py:257-265: alternating intense 0.2 s / sparse
    1.0 s mean gaps, CV 1, 6 x 50 s phases, max_batch 16) replayed in WALL
    time on the GPU engine (simulator.serve_wallclock), with the adaptive LUT
    policy and every fixed k = 1..8, over --trace-seeds arrival seeds (seed 0 =
    the reference's own timeline workload, rng [0, 6]).  Metric: mean request
    latency (queueing + prefill + decode), lower is better.  The schedule is
    time compressed by --trace-scale so one policy takes ~30 s.

    SURVEY §8(f)1 closure: profiler.calibrate's measured B200 costs are written
    in the reference's formats (calibration JSON, step-sample CSV, trace CSV)
    and fed to the reference's UNCHANGED harness.cmd_timeline / run_simulation /
    build_lut (baseline/_ref): their virtual-time predictions are reported
    beside the wall-clock replay, with the analytic delta-root and the LUTs of
    every construction (analytic linear, simulated linear, simulated on the
    measured cost table, measured)."""
    import torch

    from paper_2310_18813_b200.acceptance import estimate_expected_correct, fit_power_law, save_trace
    from paper_2310_18813_b200.cost_model import OptimalityParams, optimal_speculation_continuous, \
        save_calibration, save_step_samples
    from paper_2310_18813_b200.decoder import CONFIGS, Decoder
    from paper_2310_18813_b200.policy import AdaptivePolicy, DensePolicy, FixedPolicy, build_lut, save_lut
    from paper_2310_18813_b200.presets import example_trace
    from paper_2310_18813_b200.profiler import calibrate, dense_tables, measure_cost_table, table_lut
    from paper_2310_18813_b200.serving import serve_continuous
    from paper_2310_18813_b200.simulator import ServerConfig, serve_wallclock
    from paper_2310_18813_b200.spec_engine import SpecEngine
    from paper_2310_18813_b200.traffic import PhaseSchedule, TrafficConfig, gen_phased

    rank, world, local = _dist()
    if rank != 0:
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    trace = example_trace()
    sizes = (1, 2, 4, 8, 16)
    tgt = Decoder(CONFIGS[TARGET], dtype="bf16", device=dev, seed=0, init="device", max_pos=P + NEW + 32)
    drf = Decoder(CONFIGS[DRAFT], dtype="bf16", device=dev, seed=1, init="device", max_pos=P + NEW + 32)
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=trace, max_batch=16, max_k=8, prompt_len=P,
                     max_new=NEW, seed=0)
    lut = build_lut(None, trace, s_grid=K_GRID, profiled_sizes=sizes, mode="measured",
                    sample_size=1, rng=np.random.default_rng(0), gen_len=NEW, engine=eng)

    # ---- (f)1: measured calibration -> reference formats -> the reference's own code
    out = ROOT / "gpurun_out" / "config5"
    out.mkdir(parents=True, exist_ok=True)
    model, samples = calibrate(eng, batch_sizes=sizes, k_grid=range(1, 9), reps=10)
    ctx = P + NEW // 2
    verify_ms = {(smp.batch_size, smp.query_len): smp.measured_time for smp in samples}
    for b in sizes:
        verify_ms[(b, 0)] = eng.time_verify(b, 0, ctx=ctx, reps=10)
    draft_ms = {b: eng.time_draft_step(b, ctx=ctx, reps=10) for b in sizes}
    pts = [(s, estimate_expected_correct(trace, s)) for s in range(1, 9)]
    fit = fit_power_law(pts)
    save_calibration(model, out / "calibration.json", fit=fit)
    save_step_samples(samples, out / "step_samples.csv")
    save_trace(trace, out / "trace.csv")
    save_lut(lut, out / "lut_measured.csv", seed=0, calibration="measured on this B200 (build_lut mode=measured)")
    lut_table, _cells = table_lut(verify_ms, draft_ms, trace, s_grid=K_GRID, profiled_sizes=sizes,
                                  sample_size=200, rng=np.random.default_rng([0, 2]), gen_len=NEW)
    # dense tables: every live size 1..16 measured (the reference rule resolves 9..15 to min(s_8, s_16))
    dense_sizes = range(1, 17)
    vms_all, dms_all = measure_cost_table(eng, dense_sizes, k_grid=K_GRID, ctx=ctx, reps=10)
    tab_formed, tab_cont, _ = dense_tables(vms_all, dms_all, trace, dense_sizes, s_grid=K_GRID, sample_size=200,
                                           rng=np.random.default_rng([0, 3]), gen_len=NEW)
    delta_root = {str(b): round(optimal_speculation_continuous(OptimalityParams.from_model(model, fit, b), 1, 8,
                                                               tol=1e-6), 3) for b in sizes}
    ref = _ref_harness()
    closure = {"calibration": {"alpha": {str(b): round(v, 5) for b, v in model.alpha.items()},
                               "beta": round(model.beta, 5),
                               "ssm_step": {str(b): round(v, 5) for b, v in model.ssm_step.items()}},
               "verify_ms": {f"{b},{s}": round(v, 4) for (b, s), v in sorted(verify_ms.items())},
               "draft_step_ms": {str(b): round(v, 4) for b, v in draft_ms.items()},
               "delta_root_s": delta_root,
               "lut_measured": {str(b): v for b, v in lut.entries.items()},
               "lut_table_simulated": {str(b): v for b, v in lut_table.entries.items()},
               "dense_formed_table": {str(b): v for b, v in tab_formed.items()},
               "dense_continuous_table": {str(b): v for b, v in tab_cont.items()},
               "verify_ms_dense": {f"{b},{s}": round(v, 4) for (b, s), v in sorted(vms_all.items())},
               "draft_step_ms_dense": {str(b): round(v, 4) for b, v in dms_all.items()}}
    if ref is not None:
        rh, rsim, rpol, rcm = ref
        rmodel, rfit = rcm.load_calibration(out / "calibration.json")
        import specbatch.acceptance as racc
        trace_r = racc.load_trace(out / "trace.csv")  # the reference's own AcceptanceTrace type
        closure["source"] = "reference specbatch (baseline/_ref), unchanged"
        closure["lut_analytic_linear"] = {str(b): v for b, v in
                                          rpol.build_lut(rmodel, trace_r, s_grid=K_GRID, profiled_sizes=sizes).entries.items()}
        closure["lut_simulated_linear"] = {str(b): v for b, v in rpol.build_lut(
            rmodel, trace_r, s_grid=K_GRID, profiled_sizes=sizes, mode="simulated", sample_size=200,
            rng=np.random.default_rng([0, 2]), gen_len=NEW).entries.items()}
        cfg = rh.ExperimentConfig(calibration=str(out / "calibration.json"), trace=str(out / "trace.csv"),
                                  sizes=sizes, out_dir=str(out / "ref_timeline"))
        summ = rh.cmd_timeline(cfg)
        rows = [ln.split(",") for ln in Path(summ).read_text().splitlines() if ln and not ln.startswith("#")]
        closure["ref_cmd_timeline_latency_s"] = {r[0]: round(float(r[1]), 4) for r in rows[1:]}
        # the same simulator on every policy of the wall replay, at the replay's load: arrivals
        # compressed by time_scale exactly as replayed, latency / time_scale (trace seconds)
        import specbatch.traffic as rtr
        rlut = rpol.build_lut(rmodel, trace_r, s_grid=K_GRID, profiled_sizes=sizes)
        pred = {}
        for seed in range(args.trace_seeds):
            wl0 = rtr.gen_phased(rh.timeline_schedule(cfg), np.random.default_rng([seed, 6]), gen_len=NEW)
            wls = [rtr.Request(id=r.id, arrival=r.arrival * args.trace_scale, gen_len=r.gen_len) for r in wl0]
            for pol in [rpol.AdaptivePolicy(rlut)] + [rpol.fixed_policy(k) for k in range(1, 9)]:
                rep = rsim.run_simulation(wls, rsim.ServerConfig(policy=pol, max_batch=16), rmodel, trace_r,
                                          np.random.default_rng([0, 7]))
                pred.setdefault(pol.label, []).append(round(rep.avg_latency / args.trace_scale, 4))
        closure["ref_run_simulation_latency_s_at_replay_load"] = pred
    else:
        closure["source"] = "baseline/_ref absent: reference harness not run"

    # ---- wall-clock replay on the GPU engine, every policy, several arrival seeds
    phases = tuple((50.0, TrafficConfig(mean_interval=0.2 if i % 2 == 0 else 1.0, cv=1.0, count=1000))
                   for i in range(6))
    policies = [AdaptivePolicy(lut), DensePolicy(tab_formed)] + [FixedPolicy(k) for k in range(1, 9)]
    t_cap = time.perf_counter()
    for bb in range(1, 17):  # capture every (b, k) iteration graph up front: no capture inside a replay
        for kk in range(0, 9):
            eng._graph(bb, kk)
    t_cap = time.perf_counter() - t_cap
    t_run = time.perf_counter()
    lat = {pol.label: [] for pol in policies}
    batches = {pol.label: [] for pol in policies}
    n_req = []
    for seed in range(args.trace_seeds):
        workload = gen_phased(PhaseSchedule(phases=phases), np.random.default_rng([seed, 6]), gen_len=NEW)
        n_req.append(len(workload))
        for pol in policies:
            rep = serve_wallclock(workload, ServerConfig(policy=pol, max_batch=16), eng, time_scale=args.trace_scale)
            lat[pol.label].append(rep.avg_latency / args.trace_scale)  # back to trace seconds
            batches[pol.label].append(float(np.mean([r.served_batch_size for r in rep.records])))
    # continuous batching: retire / admit every iteration, k re-chosen per iteration:
    # the formed-batch LUT (reference lookup rule), the dense continuous table, and every fixed k
    cont_pols = [AdaptivePolicy(lut), DensePolicy(tab_cont, "adaptive-cont")] + [FixedPolicy(kk) for kk in range(1, 9)]
    cont = {pol.label: {"latency_s_per_seed": [], "mean_live_batch": [], "mean_k": [], "riding_prefill_rows": [],
                        "separate_prefill_rows": []} for pol in cont_pols}
    for seed in range(args.trace_seeds):
        workload = gen_phased(PhaseSchedule(phases=phases), np.random.default_rng([seed, 6]), gen_len=NEW)
        for pol in cont_pols:
            rep, extra = serve_continuous(workload, eng, pol, time_scale=args.trace_scale, max_batch=16)
            c = cont[pol.label]
            c["latency_s_per_seed"].append(round(rep.avg_latency / args.trace_scale, 4))
            c["mean_live_batch"].append(round(extra["mean_live_batch"], 2))
            c["mean_k"].append(round(extra["mean_k"], 2))
            c["riding_prefill_rows"].append(extra["ridden_rows"])
            c["separate_prefill_rows"].append(extra["prefill_rows"])
    for c in cont.values():
        c["latency_s"] = round(float(np.mean(c["latency_s_per_seed"])), 4)
    cfixed = {k: v["latency_s"] for k, v in cont.items() if k.startswith("fixed")}
    cbest = min(cfixed, key=cfixed.get)
    cont_summary = {"best_fixed": cbest,
                    **{f"{a}_vs_best_fixed": round(cont[a]["latency_s"] / cfixed[cbest], 4)
                       for a in ("adaptive", "adaptive-cont")},
                    **{f"{a}_vs_best_fixed_per_seed": [round(x / y, 4) for x, y in zip(
                        cont[a]["latency_s_per_seed"], cont[cbest]["latency_s_per_seed"])]
                       for a in ("adaptive", "adaptive-cont")}}
    t_run = time.perf_counter() - t_run
    mean = {k: float(np.mean(v)) for k, v in lat.items()}
    fixed = {k: v for k, v in mean.items() if k.startswith("fixed")}
    best = min(fixed, key=fixed.get)
    ad = "adaptive"
    per_seed_ratio = [a / f for a, f in zip(lat[ad], lat[best])]
    per_seed_best = [min(fixed, key=lambda k: lat[k][i]) for i in range(args.trace_seeds)]
    per_seed_ratio_own_best = [lat[ad][i] / lat[per_seed_best[i]][i] for i in range(args.trace_seeds)]
    dn = "adaptive-dense"
    dense_ratio = [a / f for a, f in zip(lat[dn], lat[best])]
    line = {"metric": "mean request latency, phased Poisson trace (adaptive k)", "value": mean[ad], "unit": "s",
            "n_gpus": 1, "higher_is_better": False, "impl": "ours", "dtype": "bf16",
            "data": "synthetic (random-init weights, injected example_trace acceptance)",
            "config": {"workload": f"{TARGET} target + {DRAFT} draft, timeline trace 6x50s (0.2/1.0 s gaps, CV 1), "
                                   f"max_batch 16, N={NEW}, P={P}", "time_scale": args.trace_scale,
                       "seeds": args.trace_seeds, "requests_per_seed": n_req,
                       "lut": {str(k): v for k, v in lut.entries.items()}},
            "latency_s_by_policy": {k: round(v, 4) for k, v in mean.items()},
            "latency_s_by_policy_per_seed": {k: [round(x, 4) for x in v] for k, v in lat.items()},
            "mean_batch_by_policy": {k: round(float(np.mean(v)), 2) for k, v in batches.items()},
            "best_fixed": best,
            "adaptive_vs_best_fixed_latency": mean[ad] / fixed[best],
            "adaptive_vs_best_fixed_per_seed": [round(x, 4) for x in per_seed_ratio],
            "adaptive_vs_per_seed_best_fixed": [round(x, 4) for x in per_seed_ratio_own_best],
            "per_seed_best_fixed": per_seed_best,
            "adaptive_dense_vs_best_fixed_latency": mean[dn] / fixed[best],
            "adaptive_dense_vs_best_fixed_per_seed": [round(x, 4) for x in dense_ratio],
            "continuous_summary": cont_summary,
            "wall_s": round(t_run, 1), "continuous_batching": cont, "graph_capture_s": round(t_cap, 1),
            "f1_closure": closure}
    (out / "result.json").write_text(json.dumps(line, indent=1) + "\n")
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
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=trace,
                     max_batch=b if args.quick else max(b, max(LUT_SIZES)), max_k=8, prompt_len=P,
                     max_new=NEW, seed=0 if tp else rank)

    # ---- the paper's profiler on THIS GPU: every (b, k) cell runs the real
    # engine (build_lut mode="measured"); the analytic LUT from a measured
    # LinearStepModel calibration is reported beside it.
    cal, samples = calibrate(eng, batch_sizes=(1, 2, 4, 8), k_grid=range(1, 9), reps=5)
    lut_analytic = build_lut(cal, trace, s_grid=K_GRID, profiled_sizes=(1, 2, 4, 8))
    sizes = tuple(x for x in LUT_SIZES if x <= eng.max_batch) if not args.quick else (b,)
    lut = build_lut(None, trace, s_grid=K_GRID, profiled_sizes=sizes, mode="measured", sample_size=1,
                    rng=np.random.default_rng(0), gen_len=NEW, engine=eng)
    k = args.k if args.k >= 0 else lookup(lut, b).chosen_s

    # ---- "tokens/s vs batch size, adaptive k vs best fixed k": re-timed INDEPENDENTLY of the
    # LUT-building pass, every (b, k) cell REPEATS times on fresh batches (decode tokens/s,
    # prefill excluded as in the profiler / the reference cost model); median and spread
    by_batch = {}
    if not args.quick:
        for bb in sizes:
            cell = {}
            for kk in K_GRID:
                tps = []
                for r in range(REPEATS):
                    sts = [SequenceState(request_id=500000 + 1000 * r + i, target_len=NEW) for i in range(bb)]
                    res = eng.generate(sts, kk)
                    tps.append(res.tokens_generated / (res.total_time / 1e3))
                cell[kk] = tps
            med = {kk: float(np.median(v)) for kk, v in cell.items()}
            ka = lookup(lut, bb).chosen_s
            kf = max(med, key=med.get)
            by_batch[str(bb)] = {
                "adaptive_k": ka, "adaptive_tokens_per_s": round(med[ka], 1),
                "adaptive_spread": [round(min(cell[ka]), 1), round(max(cell[ka]), 1)],
                "best_fixed_k": kf, "best_fixed_tokens_per_s": round(med[kf], 1),
                "best_fixed_spread": [round(min(cell[kf]), 1), round(max(cell[kf]), 1)],
                "adaptive_vs_best_fixed": round(med[ka] / med[kf], 4),
                "k_sweep_median": {str(kk): round(v, 1) for kk, v in sorted(med.items())}}

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

    # ---- config 3 (BASELINE configs[2]): stochastic rejection sampling min(1, p/q) with residual
    # resampling and an ADAPTIVE k TABLE: the same pair in stochastic mode (REAL acceptance of the
    # random-init weights at temperature 1), its own measured b -> k LUT (build_lut mode="measured"),
    # then every (b, k) cell re-timed independently: tokens/s by b, adaptive vs best fixed k
    stoch = None
    if not tp and os.environ.get("SB_SKIP_STOCH", "0") != "1":
        s_sizes = tuple(x for x in (1, 2, 4, 8, 16) if x <= eng.max_batch) if not args.quick else (b,)
        eng_s = SpecEngine(tgt, drf, mode="stochastic", max_batch=max(s_sizes), max_k=8, prompt_len=P,
                           max_new=NEW, seed=rank, autotune=False)
        # (real acceptance is random per batch: 3 batches per (b, k) cell for the profile)
        from paper_2310_18813_b200.policy import SpeculationLUT
        cells = {bb: build_lut(None, trace, s_grid=K_GRID, profiled_sizes=(bb,), mode="measured", sample_size=3 * bb,
                               rng=np.random.default_rng(1), gen_len=NEW, engine=eng_s) for bb in s_sizes}
        lut_s = SpeculationLUT(entries={bb: c.entries[bb] for bb, c in cells.items()}, s_grid=K_GRID,
                               provenance={"mode": "measured", "sample_size": "3 batches per cell"})
        s_by_batch = {}
        acc_s = prop_s = 0
        for bb in s_sizes:
            med, spread = {}, {}
            for kk in K_GRID:
                tps = []
                for r in range(3):
                    sts = [SequenceState(request_id=700000 + 1000 * r + i, target_len=NEW) for i in range(bb)]
                    res = eng_s.generate(sts, kk)
                    tps.append(res.tokens_generated / (res.total_time / 1e3))
                    if kk > 0:
                        log = eng_s.stats.accepted
                        acc_s += int(log[log >= 0].sum())
                        prop_s += int(kk * (log >= 0).sum())
                med[kk] = float(np.median(tps))
                spread[kk] = (round(min(tps), 1), round(max(tps), 1))
            ka = lookup(lut_s, bb).chosen_s
            kf = max(med, key=med.get)
            # real acceptance varies batch to batch: the held-out re-timing of the LUT's k is within the
            # noise of the best fixed k when its best batch reaches the best fixed k's worst one
            s_by_batch[str(bb)] = {"adaptive_k": ka, "adaptive_tokens_per_s": round(med[ka], 1), "best_fixed_k": kf,
                                   "best_fixed_tokens_per_s": round(med[kf], 1),
                                   "adaptive_vs_best_fixed": round(med[ka] / med[kf], 4),
                                   "adaptive_spread": spread[ka], "best_fixed_spread": spread[kf],
                                   "within_batch_noise": spread[ka][1] >= spread[kf][0],
                                   "k_sweep_median": {str(kk): round(v, 1) for kk, v in sorted(med.items())}}
        ks = lookup(lut_s, b).chosen_s
        ms_s = 0.0
        for s in range(2):
            r = eng_s.generate(batch(91000 + s), ks)
            ms_s += r.total_time + eng_s.stats.prefill_ms
        stoch = {"tokens_per_s": 2 * b * NEW / (ms_s / 1e3), "k": ks,
                 "lut": {str(x): v for x, v in lut_s.entries.items()},
                 "acceptance_rate": round(acc_s / max(prop_s, 1), 4),
                 "acceptance": "real (random-init pair, temperature 1): min(1, p/q) + residual resampling",
                 "tokens_per_s_by_batch": s_by_batch,
                 "adaptive_vs_best_fixed_geomean": round(float(np.exp(np.mean(
                     [np.log(v["adaptive_vs_best_fixed"]) for v in s_by_batch.values()]))), 4) if s_by_batch else None,
                 "timing": "decode tokens/s (prefill excluded), median of 3 fresh batches per (b, k) cell"}
        del eng_s
        torch.cuda.empty_cache()

    # ---- roofline of the verify forward (the north_star's roofline object), timed live
    hbm, tf, peak_kind = _peaks()
    ctx_avg = P + NEW // 2
    vb = verify_bytes(tgt.cfg, b, k, ctx_avg)
    v_ms = eng.time_verify(b, k, ctx=ctx_avg, reps=20)
    achieved = vb / (v_ms / 1e3) / 1e9
    verify_by_batch = {}  # north_star: >= 60% of the HBM roofline for verification at b <= 8
    for bb in (sizes if not args.quick else (b,)):
        kb_ = lookup(lut, bb).chosen_s
        ms_ = eng.time_verify(bb, kb_, ctx=ctx_avg, reps=10)
        t_hbm = verify_bytes(tgt.cfg, bb, kb_, ctx_avg) / (hbm * 1e9)
        t_tc = verify_flops(tgt.cfg, bb, kb_, ctx_avg) / (tf * 1e12)
        verify_by_batch[str(bb)] = {"k": kb_, "tokens": bb * (kb_ + 1), "verify_ms": round(ms_, 4),
                                    "frac_hbm": round(t_hbm / (ms_ / 1e3), 4),
                                    "frac_tensor": round(t_tc / (ms_ / 1e3), 4),
                                    "frac_roofline": round(max(t_hbm, t_tc) / (ms_ / 1e3), 4)}
    traffic = None
    tf_path = ROOT / "profiles" / "verify_traffic.json"
    if tf_path.exists():
        tfd = json.loads(tf_path.read_text())
        for e in tfd.get("entries", [tfd]):
            if e.get("b") == b and e.get("k") == k and str(e.get("workload", "")).startswith(TARGET + " "):
                traffic = e["dram_bytes_read_plus_write"]

    # ---- CPU baseline (rank 0, N=1 only): the reference arm's method on a smaller sample
    cpu = None
    if rank == 0 and world == 1 and os.environ.get("SB_SKIP_CPU", "0") != "1":
        try:
            layers = int(os.environ.get("SB_CPU_LAYERS", "8" if TARGET == "llama-2-7b" else "2")) or None
            r = cpu_reference_run(b, 1, 0, layers=layers)
            cpu = {"value": r["value"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
                   "sample": r["sample"]}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        hb = by_batch.get(str(b), {})
        line = {
            "metric": METRIC, "value": value,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong" if tp else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, random prompts)",
            "config": {"workload": workload_str(b),
                       "k": k, "k_source": "adaptive LUT (profiled on this GPU)" if args.k < 0 else "fixed",
                       "lut": {str(kk): v for kk, v in lut.entries.items()},
                       "lut_analytic_from_measured_calibration": {str(kk): v for kk, v in lut_analytic.entries.items()},
                       "acceptance": "injected: TraceSampler(example_trace()) law on device",
                       "parallelism": f"tp{world} (NCCL all-reduce / all-gather)" if tp else f"replicas x{world}",
                       "l2": "inputs (weights >= 13.5 GB) > L2; no flush"},
            "decode_tokens_per_s": jobs * args.steps * b * NEW / (sum(decode_ms) / 1e3) if world == 1 else None,
            "tokens_per_s_by_batch": by_batch,
            "verify_roofline_by_batch": verify_by_batch,
            "best_fixed_k": hb.get("best_fixed_k"),
            "adaptive_vs_best_fixed": hb.get("adaptive_vs_best_fixed"),
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
