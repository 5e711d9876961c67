"""Continuous batching on the GPU engine: the formed batch is
no longer held until every sequence finishes (reference engine.py:186-188,
SPEC.md:297) -- finished sequences retire after the iteration that completes
them and waiting requests are admitted into the freed KV slots, and the
speculation length is re-chosen EVERY iteration from the LUT at the current
live batch size (the paper's adaptive policy applied per step instead of per
formed batch).

Mechanics: live sequences occupy rows 0..b-1 of the engine's device state
(tokens, lengths, counters); row r reads / writes KV slot ``engine.slots[r]``.
Retirement compacts the ROW state (a few KB gather on the device) and permutes
the row->slot map; KV slabs never move.  Admission writes the prompt into a
free row, prefills its slot (target + draft) and joins the next iteration.  The
per-(b, k) iteration graphs of :class:`SpecEngine` are replayed unchanged
(they read the slot map and row state from device memory).

Latency is wall-clock (queueing + prefill + decode) exactly as in
:func:`simulator.serve_wallclock`, so the two are directly comparable on the
same trace (``bench.py --workload trace``).
"""

from __future__ import annotations

import time
from collections import deque

import numpy as np
import torch

from .simulator import RequestRecord, SimulationReport, summarize
from .traffic import Request

__all__ = ["serve_continuous"]


def serve_continuous(workload: list[Request], engine, policy, time_scale: float = 1.0, max_batch: int | None = None,
                     group_size: int = 40, clock=None, collect: bool = False, min_admit: int = 1,
                     max_wait: float = 0.0, riding: bool | None = None,
                     compact: bool = False) -> tuple[SimulationReport, dict]:
    """Serve `workload` with continuous batching on `engine` (a SpecEngine).

    `policy.decide(b)` picks k at every iteration for the live batch size b
    (AdaptivePolicy(lut) / FixedPolicy(k)).  Requests need gen_len <= engine.max_new.
    Admission batching: a prefill streams the whole target once, so admitting
    one request at a time is expensive; new requests join only when at least
    `min_admit` can (or the engine is idle, or the oldest has waited
    `max_wait` wall seconds).
    Prefill: with ``riding`` (default: whenever the engine supports it) prompts
    admitted while other rows decode are prefilled INSIDE the next iteration's
    verify forward (sb_decoder_forward_mixed, one weight stream) and decode from
    the iteration after; otherwise each admission runs its own prefill forward.
    Slots: by default a retired row's KV slot is simply freed and the row->slot
    map permuted (no KV moves).  ``compact=True`` keeps row == slot instead: the
    KV slabs of surviving rows in slots >= the new live count are moved into the
    freed low slots by the K5 compaction kernel (sb_kv_compact, target + draft),
    so live KV stays dense in slots [0, b).
    Returns (report, {"mean_live_batch", "mean_k", "iterations", "acceptance_rate",
    "compacted_rows"[, "outputs": {id: tokens}]}).
    """
    if any(nxt.arrival < cur.arrival for cur, nxt in zip(workload, workload[1:])):
        raise ValueError("workload must be sorted by arrival time")
    eng = engine
    B = min(max_batch or eng.max_batch, eng.max_batch)
    P = eng.prompt_len
    dev = eng.dev
    if any(r.gen_len > eng.max_new for r in workload):
        raise ValueError("a request asks for more tokens than the engine's max_new")
    clock = clock or time.perf_counter
    i32 = dict(device=dev, dtype=torch.int32)
    row_req: list[Request | None] = []  # request of each live row
    row_start: list[float] = []
    free_slots = list(range(eng.max_batch))[::-1]
    slot_of_row: list[int] = []
    waiting: deque[Request] = deque()
    records: list[RequestRecord] = []
    nxt, total = 0, len(workload)
    pinned_prompts = torch.zeros(B, P, dtype=torch.int32, pin_memory=True)
    done_host = torch.zeros(eng.max_batch, dtype=torch.int32, pin_memory=True)
    acc_sum = torch.zeros(1, dtype=torch.int64, device=dev)  # accepted drafts over live rows (k > 0 iterations)
    proposed = 0
    k_hist: list[int] = []
    b_hist: list[int] = []
    outputs: dict[int, list[int]] = {}
    prof = {"prefills": 0, "prefill_rows": 0, "ridden_rows": 0, "prefill_s": 0.0, "iter_s": 0.0, "host_s": 0.0,
            "idle_s": 0.0, "compacted_rows": 0}
    if riding is None:
        riding = getattr(eng, "supports_ride", False)
    elif riding and not getattr(eng, "supports_ride", False):
        raise ValueError("this engine's target has no riding-prefill path (llama bf16 unsharded only)")
    if riding:
        eng.tune_riding()  # plans for the mixed token counts (outside the timed replay)
    with torch.cuda.stream(eng.stream):
        eng.iter.zero_()
        eng.finish_iter.fill_(-1)
        t0 = clock()
        while nxt < total or waiting or row_req:
            now = clock() - t0
            while nxt < total and workload[nxt].arrival * time_scale <= now:
                waiting.append(workload[nxt])
                nxt += 1
            if not row_req and not waiting:
                wait = workload[nxt].arrival * time_scale - now
                if wait > 0:
                    time.sleep(min(wait, 0.005))
                    prof["idle_s"] += min(wait, 0.005)
                continue
            # ---- admission into free rows / KV slots
            new_rows = []
            room = B - len(row_req)
            admit = bool(waiting) and room > 0 and (
                not row_req or min(room, len(waiting)) >= min_admit
                or (max_wait > 0 and now - waiting[0].arrival * time_scale >= max_wait))
            while admit and waiting and len(row_req) < B:
                r = waiting.popleft()
                row = len(row_req)
                row_req.append(r)
                slot_of_row.append(free_slots.pop())
                row_start.append(clock() - t0)
                pinned_prompts[len(new_rows)].copy_(torch.from_numpy(np.asarray(eng.prompt_fn(r.id), dtype=np.int32)))
                new_rows.append(row)
            b = len(row_req)
            b_run, ride = b, 0  # rows this iteration decodes / prompts riding along its verify
            if new_rows:
                r0, n = new_rows[0], len(new_rows)  # admitted rows are contiguous at the end
                eng.tokens[r0:r0 + n, :P].copy_(pinned_prompts[:n], non_blocking=True)
                eng.n_tok[r0:r0 + n].fill_(P)
                eng.produced[r0:r0 + n].zero_()
                eng.finish_iter[r0:r0 + n].fill_(-1)
                eng.target_len[r0:r0 + n].copy_(torch.tensor([row_req[i].gen_len for i in new_rows], dtype=torch.int32))
                eng.slots[:b].copy_(torch.tensor(slot_of_row, dtype=torch.int32))
                if riding and r0 > 0 and n <= eng.pf_chunk:
                    # chunked prefill: the prompts ride inside the next verify forward
                    # (one weight stream for both) and decode from the iteration after
                    b_run, ride = r0, n
                    prof["ridden_rows"] += n
                else:
                    tp = clock()
                    _prefill_rows(eng, new_rows)
                    eng.stream.synchronize()  # pinned staging rows are reused next admission
                    prof["prefill_s"] += clock() - tp
                    prof["prefills"] += 1
                    prof["prefill_rows"] += len(new_rows)
            # ---- one speculative iteration at the LUT's k for the live batch size
            k = policy.decide(b_run).chosen_s
            k = min(k, eng.max_k)
            ti = clock()
            # k = 0 iterations keep the draft KV current: the policy may pick k > 0 next
            sync = k == 0 and eng.max_k > 0
            if ride:
                eng._iteration(b_run, k, ride=ride, draft_sync=sync)
            elif eng.use_graphs:
                eng._graph(b, k, draft_sync=sync).replay()
            else:
                eng._iteration(b, k, draft_sync=sync)
            if k > 0:
                acc_sum += eng.accepted[:b_run].sum()
                proposed += k * b_run
            k_hist.append(k)
            b_hist.append(b_run)
            # ---- retirement: rows whose produced reached target_len
            done = (eng.produced[:b] >= eng.target_len[:b]).to(torch.int32)
            done_host[:b].copy_(done, non_blocking=True)
            eng.stream.synchronize()
            prof["iter_s"] += clock() - ti
            fin = done_host[:b].numpy().astype(bool)
            if fin.any():
                t_done = clock() - t0
                keep = [i for i in range(b) if not fin[i]]
                fin_rows = np.nonzero(fin)[0]
                if collect:
                    toks = eng.tokens[torch.as_tensor(fin_rows, device=dev, dtype=torch.long), P:].cpu().numpy()
                for n_, i in enumerate(fin_rows):
                    r = row_req[i]
                    if collect:
                        outputs[r.id] = [int(t) for t in toks[n_, : r.gen_len]]
                    arr = r.arrival * time_scale
                    records.append(RequestRecord(r.id, arr, row_start[i], t_done, t_done - arr, b, k))
                    free_slots.append(slot_of_row[i])
                if keep and keep != list(range(len(keep))):
                    idx = torch.tensor(keep, device=dev, dtype=torch.long)
                    for t in (eng.tokens, eng.n_tok, eng.produced, eng.target_len, eng.finish_iter):
                        t[: len(keep)] = t[idx].clone()
                row_req = [row_req[i] for i in keep]
                row_start = [row_start[i] for i in keep]
                slot_of_row = [slot_of_row[i] for i in keep]
                if compact and keep:
                    n_moved = _compact_slots(eng, slot_of_row, free_slots)
                    prof["compacted_rows"] += n_moved
                if keep:  # the compacted rows keep their KV slots
                    eng.slots[: len(keep)].copy_(torch.tensor(slot_of_row, dtype=torch.int32))
        torch.cuda.synchronize(dev)
        eng.slots.copy_(torch.arange(eng.max_batch, **i32))  # generate() assumes row == slot
    rep = summarize(records, group_size=group_size, policy=f"continuous/{getattr(policy, 'label', 'policy')}")
    extra = {"mean_live_batch": float(np.mean(b_hist)) if b_hist else 0.0,
             "mean_k": float(np.mean(k_hist)) if k_hist else 0.0, "iterations": len(k_hist),
             "acceptance_rate": float(acc_sum.item()) / proposed if proposed else 0.0,
             "wall_s": clock() - t0, **{k_: round(v_, 3) if isinstance(v_, float) else v_ for k_, v_ in prof.items()}}
    if collect:
        extra["outputs"] = outputs
    return rep, extra


def _compact_slots(eng, slot_of_row: list[int], free_slots: list[int]) -> int:
    """Move the KV of live rows whose slot is >= the live count into free slots
    below it (sb_kv_compact on target and draft caches), so row r uses slot r.
    Mutates slot_of_row / free_slots; the row state is already compacted.
    Returns the number of rows moved."""
    b = len(slot_of_row)
    holes = sorted(set(range(b)) - set(slot_of_row))
    movers = [r for r, s in enumerate(slot_of_row) if s >= b]
    assert len(holes) == len(movers)
    if not movers:
        return 0
    dev = eng.dev
    src = torch.tensor([slot_of_row[r] for r in movers], device=dev, dtype=torch.int32)
    dst = torch.tensor(holes, device=dev, dtype=torch.int32)
    rows = torch.tensor(movers, device=dev, dtype=torch.long)
    lens = eng.n_tok[rows].clone()  # every written position (target KV valid to n_tok - 1, draft to n_tok - 3)
    eng.target.kv_compact(eng.kv_t, src, dst, lens)
    if eng.draft is not None:
        eng.draft.kv_compact(eng.kv_d, src, dst, lens)
    for r, h in zip(movers, holes):
        free_slots.append(slot_of_row[r])
        free_slots.remove(h)
        slot_of_row[r] = h
    free_slots.sort(reverse=True)  # pop() hands out the lowest free slot next
    eng.slots[:b].copy_(torch.tensor(slot_of_row, dtype=torch.int32))
    return len(movers)


def _prefill_rows(eng, rows: list[int]) -> None:
    """Prefill the prompts of newly admitted rows (target + draft KV of their slots)."""
    from . import _native as N

    P = eng.prompt_len
    if P < 2:
        return
    q = P - 1
    for c0 in range(0, len(rows), eng.pf_chunk):
        chunk = rows[c0:c0 + eng.pf_chunk]
        nb = len(chunk)
        idx = torch.tensor(chunk, device=eng.dev, dtype=torch.long)
        eng.pf_ids[: nb * q].copy_(eng.tokens[idx, :q].reshape(-1))
        eng.pf_pos[: nb * q].copy_(eng._pf_pos_pattern[: nb * q])
        eng.pf_slots[:nb].copy_(eng.slots[idx])
        eng.target.forward(eng.kv_t, eng.pf_ids, eng.pf_slots, eng.pf_pos, nb, q, None, N.LOGITS_NONE, eng.workspace)
        if eng.draft is not None:
            eng.draft.forward(eng.kv_d, eng.pf_ids, eng.pf_slots, eng.pf_pos, nb, q, None, N.LOGITS_NONE,
                              eng.workspace)
