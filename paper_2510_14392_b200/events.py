"""Event logs in the reference's JSONL format (save_event_log,
engine.cpp:395-451) from the device plan logs.

The device records, per instance, every begin_step (time, duration, predicted
and ground-truth step time, token / context totals), every plan entry in
admission order and every PAB reject.  That is enough to rebuild the whole
EventLog of run_node: arrivals are the enqueued trace rows, and the token
emissions of a step are a replay of its plan entries in plan order over the
requests' progress (complete_step, engine.cpp:204-254).  Within one
timestamp the reference appends completion events (token_emit / request_done
in plan order, then batch_end), then arrivals, then admission rejects, then
batch_start (run_node, engine.cpp:271-283).
"""
from __future__ import annotations

import numpy as np


def _ms(us: int) -> str:
    return "%.3f" % (us / 1000.0)


def event_log_lines(rows, inst, result, counts, steps, entries, rejects, node_id: int = 0):
    """JSONL lines (with trailing newlines) of one instance's EventLog."""
    off, n_arr = int(inst.trace_off), int(result["n_arrived"])
    arrival = rows.arrival_us[off:off + n_arr]
    prompt = rows.prompt_len[off:off + n_arr]
    output = rows.output_len[off:off + n_arr]
    ttft = rows.ttft_us[off:off + n_arr]
    tpot = rows.tpot_us[off:off + n_arr]
    if counts["truncated"]:
        raise ValueError("plan log truncated: raise the log capacities")
    ev = []  # (t, phase, order, line)
    for r in range(n_arr):
        ev.append((int(arrival[r]), 1, r,
                   '{"t_ms":%s,"kind":"arrival","req_id":%d,"arrival_ms":%s,"prompt_tokens":%d,'
                   '"output_tokens":%d,"ttft_slo_ms":%s,"tpot_slo_ms":%s}\n'
                   % (_ms(arrival[r]), r, _ms(arrival[r]), prompt[r], output[r], _ms(ttft[r]),
                      _ms(tpot[r]))))
    for k in range(int(counts["rejects"])):
        rj = rejects[k]
        ev.append((int(rj["t_us"]), 2, k,
                   '{"t_ms":%s,"kind":"admission_reject","req_id":%d,"prompt_tokens":%d,'
                   '"pab_tokens":%d}\n' % (_ms(rj["t_us"]), rj["req"], prompt[rj["req"]],
                                          rj["pab_tokens"])))
    prefilled = np.zeros(max(1, n_arr), np.int64)
    nidx = np.zeros(max(1, n_arr), np.int64)
    for s in range(int(counts["steps"])):
        st = steps[s]
        t0 = int(st["t_us"])
        t1 = t0 + int(st["duration_us"])
        ev.append((t0, 3, s,
                   '{"t_ms":%s,"kind":"batch_start","step":%d,"new_tokens":%d,'
                   '"context_tokens":%d,"predicted_ms":%.6f}\n'
                   % (_ms(t0), s, st["total_new"], st["total_ctx"], st["predicted_ms"])))
        body = []
        for e in entries[int(st["entry_off"]):int(st["entry_off"]) + int(st["n_entries"])]:
            r, take = int(e["req"]), int(e["new_tokens"])
            emit = True
            if prefilled[r] < prompt[r]:
                prefilled[r] += take
                emit = prefilled[r] >= prompt[r]
            if emit:
                body.append('{"t_ms":%s,"kind":"token_emit","req_id":%d,"token_idx":%d}\n'
                            % (_ms(t1), r, nidx[r]))
                nidx[r] += 1
                if nidx[r] >= output[r]:
                    body.append('{"t_ms":%s,"kind":"request_done","req_id":%d}\n' % (_ms(t1), r))
        body.append('{"t_ms":%s,"kind":"batch_end","step":%d,"actual_ms":%.6f}\n'
                    % (_ms(t1), s, st["actual_ms"]))
        ev.append((t1, 0, s, "".join(body)))
    ev.sort(key=lambda x: (x[0], x[1], x[2]))
    lines = [x[3] for x in ev]
    lines.append('{"kind":"log_end","node":%d,"incomplete":%d}\n'
                 % (node_id, 1 if result["incomplete"] else 0))
    return lines


def event_log_jsonl(rows, inst, result, counts, steps, entries, rejects, node_id: int = 0) -> str:
    return "".join(event_log_lines(rows, inst, result, counts, steps, entries, rejects, node_id))
