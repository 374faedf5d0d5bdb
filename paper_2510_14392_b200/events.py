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


def _node_lines(arrivals, prompt, output, arr_us, ttft, tpot, counts, steps, entries, rejects,
                incomplete: bool, node_id: int):
    """EventLog lines of one cluster node.  `arrivals` = [(t, row, rej_before,
    steps_before)] in enqueue order; the tags (-1: not recorded) place an
    arrival among the node's begin_step events of the same instant -- after
    the rejects and batch starts logged before it was enqueued (a rerouted
    arrival can follow the node's own begin at that instant, cluster.cpp:
    222-237).  Within one instant: the step completing (token_emit /
    request_done in plan order, batch_end), then, ordered by (steps begun,
    rejects logged): arrivals, rejects, the batch start."""
    if counts["truncated"]:
        raise ValueError("plan log truncated: raise the log capacities")
    big = 1 << 62
    ev = []
    for k, (t, r, rc, sc) in enumerate(arrivals):
        ev.append((int(t), 1, (int(sc), int(rc), 0, k),
                   '{"t_ms":%s,"kind":"arrival","req_id":%d,"arrival_ms":%s,"prompt_tokens":%d,'
                   '"output_tokens":%d,"ttft_slo_ms":%s,"tpot_slo_ms":%s}\n'
                   % (_ms(t), r, _ms(arr_us[r]), prompt[r], output[r], _ms(ttft[r]),
                      _ms(tpot[r]))))
    for j in range(int(counts["rejects"])):
        rj = rejects[j]
        ev.append((int(rj["t_us"]), 1, (int(rj["step"]), j, 1, 0),
                   '{"t_ms":%s,"kind":"admission_reject","req_id":%d,"prompt_tokens":%d,'
                   '"pab_tokens":%d}\n' % (_ms(rj["t_us"]), rj["req"], prompt[rj["req"]],
                                          rj["pab_tokens"])))
    prefilled, nidx = {}, {}
    for s in range(int(counts["steps"])):
        st = steps[s]
        t0 = int(st["t_us"])
        t1 = t0 + int(st["duration_us"])
        ev.append((t0, 1, (s, big, 2, 0),
                   '{"t_ms":%s,"kind":"batch_start","step":%d,"new_tokens":%d,'
                   '"context_tokens":%d,"predicted_ms":%.6f}\n'
                   % (_ms(t0), s, st["total_new"], st["total_ctx"], st["predicted_ms"])))
        body = []
        for e in entries[int(st["entry_off"]):int(st["entry_off"]) + int(st["n_entries"])]:
            r, take = int(e["req"]), int(e["new_tokens"])
            emit = True
            pf = prefilled.get(r, 0)
            if pf < prompt[r]:
                pf += take
                prefilled[r] = pf
                emit = pf >= prompt[r]
            if emit:
                j = nidx.get(r, 0)
                body.append('{"t_ms":%s,"kind":"token_emit","req_id":%d,"token_idx":%d}\n'
                            % (_ms(t1), r, j))
                nidx[r] = j + 1
                if j + 1 >= output[r]:
                    body.append('{"t_ms":%s,"kind":"request_done","req_id":%d}\n' % (_ms(t1), r))
        body.append('{"t_ms":%s,"kind":"batch_end","step":%d,"actual_ms":%.6f}\n'
                    % (_ms(t1), s, st["actual_ms"]))
        ev.append((t1, 0, (s,), "".join(body)))
    ev.sort(key=lambda x: (x[0], x[1], x[2]))
    lines = [x[3] for x in ev]
    lines.append('{"kind":"log_end","node":%d,"incomplete":%d}\n' % (node_id, 1 if incomplete else 0))
    return lines


def cluster_event_logs(rows, logs, lb_policy: str, nodes: bool = True) -> tuple[list[str], str]:
    """run_cluster's outputs in the reference's JSONL formats: every node's
    save_event_log (engine.cpp:395-451; arrivals = the requests routed to it,
    at their routing times) and save_routing_log (cluster.cpp:114-131, view
    snapshots included).  `logs` is a cluster.ClusterLogs; nodes=False
    returns the routing log only."""
    routes = logs.routes
    node_logs = []
    for i in range(len(logs.counts) if nodes else 0):
        mine = routes[routes["node"] == i]
        arrivals = list(zip(mine["t_us"].tolist(), mine["req"].tolist(),
                            mine["rej_before"].tolist(), mine["steps_before"].tolist()))
        node_logs.append("".join(_node_lines(
            arrivals, rows.prompt_len, rows.output_len, rows.arrival_us, rows.ttft_us,
            rows.tpot_us, logs.counts[i], logs.steps[i], logs.entries[i], logs.rejects[i],
            bool(logs.out.incomplete), i)))
    rl = []
    for k in range(len(routes)):
        e = routes[k]
        snap = ",".join("%.3f" % v for v in logs.snapshots[k])
        rl.append('{"t_ms":%s,"req_id":%d,"node":%d,"policy":"%s","view_snapshot":[%s]}\n'
                  % (_ms(e["t_us"]), e["req"], e["node"], lb_policy, snap))
    return node_logs, "".join(rl)


def event_log_jsonl(rows, inst, result, counts, steps, entries, rejects, node_id: int = 0) -> str:
    return "".join(event_log_lines(rows, inst, result, counts, steps, entries, rejects, node_id))


# ------------------------------------------------------------- replay check

class EventLog:
    """A parsed JSONL event log (EventLog, engine.h:60-72): events as dicts
    with the reference's field names, plus node id and the incomplete flag."""

    def __init__(self, events, node_id: int = 0, incomplete: bool = False):
        self.events = events
        self.node_id = node_id
        self.incomplete = incomplete


_KINDS = ("arrival", "admission_reject", "batch_start", "token_emit", "request_done",
          "batch_end")


def load_event_log(text: str) -> EventLog:
    """load_event_log (engine.cpp:453-520) of a JSONL text: blank lines are
    skipped, ``log_end`` sets node / incomplete, times are ms -> µs with
    llround (time.h:30-32); an unknown kind or bad JSON raises ParseError."""
    import json
    from .batch import ms_to_us
    from .fbgpu import ParseError
    events = []
    node, incomplete = 0, False
    for line_no, line in enumerate(text.split("\n"), 1):
        if not line.strip(" \t\r"):
            continue
        try:
            j = json.loads(line)
        except ValueError as ex:
            raise ParseError(f"event log line {line_no}: {ex}") from None
        kind = j.get("kind", "")
        if kind == "log_end":
            node = int(j.get("node", 0))
            incomplete = int(j.get("incomplete", 0)) != 0
            continue
        if kind not in _KINDS:
            raise ParseError(f"event log line {line_no}: unknown kind '{kind}'")
        e = {"kind": kind, "t": ms_to_us(j.get("t_ms", 0.0))}
        if kind in ("arrival", "admission_reject", "token_emit", "request_done"):
            e["req_id"] = int(j.get("req_id", -1))
        if kind == "arrival":
            e["output_len"] = int(j.get("output_tokens", 0))
        if kind in ("batch_start", "batch_end"):
            e["step"] = int(j.get("step", -1))
        if kind == "token_emit":
            e["token_idx"] = int(j.get("token_idx", -1))
        events.append(e)
    return EventLog(events, node, incomplete)


def replay_check(log: EventLog) -> list[str]:
    """replay_check (engine.cpp:290-393): re-derives the log invariants --
    monotone timestamps, batch bracketing and sequential step ids, token
    indices consecutive from 0, request_done exactly at output_len, no
    activity for rejected requests, every request settled in a complete log.
    Returns the violation messages in the reference's wording and order
    (the final unsettled-request scan walks requests in first-seen order;
    the reference's hash-map order is unspecified, so compare that tail as a
    set)."""
    out = []

    def violation(i, what):
        out.append(f"event {i}: {what}")

    reqs = {}  # id -> [arrived, rejected, done, expected_idx, output_len]

    def req(i):
        r = reqs.get(i)
        if r is None:
            r = reqs[i] = [False, False, False, 0, 0]
        return r

    last_t = None
    in_batch = False
    expected_step = 0
    body = []
    ev = log.events
    for i, e in enumerate(ev):
        if last_t is not None and e["t"] < last_t:
            violation(i, "timestamp decreases")
        last_t = e["t"] if last_t is None else max(last_t, e["t"])
        k = e["kind"]
        if k == "arrival":
            r = req(e["req_id"])
            if r[0]:
                violation(i, "duplicate arrival")
            r[0] = True
            r[4] = e["output_len"]
        elif k == "admission_reject":
            r = req(e["req_id"])
            if not r[0]:
                violation(i, "reject before arrival")
            if r[1]:
                violation(i, "duplicate admission_reject")
            if r[3] > 0 or r[2]:
                violation(i, "reject after request activity")
            r[1] = True
        elif k == "batch_start":
            if in_batch:
                violation(i, "nested batch_start")
            if e["step"] != expected_step:
                violation(i, "non-sequential step id")
            in_batch = True
            body = []
        elif k == "token_emit":
            if not in_batch:
                violation(i, "token_emit outside a batch")
            body.append(i)
            r = req(e["req_id"])
            if not r[0]:
                violation(i, "token_emit for unknown request")
            if r[1]:
                violation(i, "token_emit for rejected request")
            if r[2]:
                violation(i, "token_emit after request_done")
            if e["token_idx"] != r[3]:
                violation(i, f"token index {e['token_idx']} does not continue sequence "
                             f"(expected {r[3]})")
            if e["token_idx"] == r[3]:
                r[3] = e["token_idx"] + 1
        elif k == "request_done":
            if not in_batch:
                violation(i, "request_done outside a batch")
            body.append(i)
            r = req(e["req_id"])
            if not r[0]:
                violation(i, "request_done for unknown request")
            if r[2]:
                violation(i, "duplicate request_done")
            if r[3] != r[4]:
                violation(i, "request_done before all tokens emitted")
            r[2] = True
        elif k == "batch_end":
            if not in_batch:
                violation(i, "batch_end without batch_start")
                continue
            if e["step"] != expected_step:
                violation(i, "batch_end step mismatch")
            for bi in body:
                if ev[bi]["t"] != e["t"]:
                    violation(bi, "in-batch event timestamp differs from batch_end")
            in_batch = False
            expected_step += 1
    if in_batch:
        out.append("log ends inside an open batch")
    if not log.incomplete:
        for rid, r in reqs.items():
            if r[0] and not r[1] and not r[2]:
                out.append(f"request {rid} neither done nor rejected in a complete log")
    return out
