"""Wall-clock serving loop (config 5 / SURVEY §8(f)3) on a fake engine: FIFO
batches of at most max_batch formed from what has arrived, one policy
decision per batch, latency = wall finish - release time."""

import time

import numpy as np

from paper_2310_18813_b200.engine import BatchResult
from paper_2310_18813_b200.policy import FixedPolicy
from paper_2310_18813_b200.simulator import ServerConfig, serve_wallclock
from paper_2310_18813_b200.traffic import Request


class _FakeEngine:
    """generate() takes `service_s` of wall time; every request finishes at the end."""

    def __init__(self, service_s=0.004):
        self.service_s = service_s
        self.calls = []

        class _S:
            prefill_ms = 0.0

        self.stats = _S()

    def generate(self, states, k):
        self.calls.append((tuple(s.request_id for s in states), k))
        time.sleep(self.service_s)
        ms = self.service_s * 1e3
        for s in states:
            s.produced = s.target_len
        return BatchResult(batch_size=len(states), spec_len=k, total_time=ms, steps=1,
                           tokens_generated=sum(s.target_len for s in states),
                           per_sequence_finish={s.request_id: ms for s in states})


def test_fifo_batches_and_latency():
    rng = np.random.default_rng(0)
    arrivals = np.cumsum(rng.exponential(0.002, size=40))
    wl = [Request(id=i, arrival=float(t), gen_len=8) for i, t in enumerate(arrivals)]
    eng = _FakeEngine()
    rep = serve_wallclock(wl, ServerConfig(policy=FixedPolicy(3), max_batch=4), eng, time_scale=1.0)
    served = [i for ids, _ in eng.calls for i in ids]
    assert served == list(range(40))  # FIFO, every request exactly once
    assert all(len(ids) <= 4 for ids, _ in eng.calls) and all(k == 3 for _, k in eng.calls)
    assert len(rep.records) == 40
    for r in rep.records:
        assert r.t_b >= r.t_start >= r.t_a - 1e-9
        assert r.latency >= eng.service_s * 0.9
    assert rep.policy == "fixed-3"
    assert abs(rep.avg_latency - np.mean([r.latency for r in rep.records])) < 1e-12
